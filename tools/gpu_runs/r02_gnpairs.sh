# GroupNorm in the epilogue for segment 1 (image pairs): parity, batch independence, timing A/B
set -o pipefail
timeout 1200 python -m pytest tests/test_gpu_gn.py -q -x 2>&1 | tail -3
for e in 0 1; do echo "== SLIM_GN_EPI=$e"; SLIM_GN_EPI=$e timeout 300 python tools/micro.py 128 200 gn 2>&1 | grep chain;
  SLIM_GN_EPI=$e timeout 300 python bench.py --norm gn --steps 30 --warmup 5 --energy-seconds 0 --no-cpu 2>/dev/null | tail -1 | cut -c1-120; done
timeout 300 python tools/micro.py 1024 20 gn 2>&1 | grep chain
