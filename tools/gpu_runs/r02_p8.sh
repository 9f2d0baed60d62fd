# fused segment 3 at C=128 over clusters of 8 (SLIM_SEGN_P8): bitwise vs per-layer, timing
set -o pipefail
SLIM_SEGN_P8=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fused_segments" 2>&1 | tail -2
for p in 0 1; do echo "== P8=$p"; SLIM_SEGN_P8=$p timeout 300 python tools/micro.py 128 200 2>&1 | grep "r=0.25"; SLIM_SEGN_P8=$p timeout 300 python tools/micro.py 8 400 2>&1 | grep "r=0.25"; SLIM_SEGN_P8=$p timeout 300 python tools/micro.py 256 100 2>&1 | grep "r=0.25"; done
