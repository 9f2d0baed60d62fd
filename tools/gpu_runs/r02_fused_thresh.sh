# fused segment kernels vs per-layer kernels at large batch (per segment, each width alone)
for B in 256 512 1024 2048 4096; do
  n=$((25600 / B)); [ $n -lt 6 ] && n=6
  echo "== B=$B fused"; timeout 300 python tools/micro.py $B $n 2>&1 | grep "chain" | head -2
  echo "== B=$B per-layer"; SLIM_NO_FUSED=1 timeout 300 python tools/micro.py $B $n 2>&1 | grep "chain" | head -2
done
