python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fused" 2>&1 | tail -15
for m in 0 2 4 8 14; do echo "SLIM_FUSED_SEGS=$m"; SLIM_FUSED_SEGS=$m python tools/micro.py 128 200 2>&1 | grep "r=0.25\|r=0.5"; done
for m in 0 14; do echo "B=8 SLIM_FUSED_SEGS=$m"; SLIM_FUSED_SEGS=$m python tools/micro.py 8 500 2>&1 | grep "r=0.25\|r=0.5"; done
