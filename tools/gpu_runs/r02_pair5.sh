# pair mode with up to 8 half-size B slots in flight
set -o pipefail
for s in 1 2 3; do timeout 300 python tools/pair_check.py $s 1.0 64 2>&1 | tail -1; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "pair_mma or multicast" 2>&1 | tail -2
for p in 0 1; do echo "== PAIR=$p"; SLIM_HALO_PAIR=$p timeout 300 python tools/micro.py 128 200 2>&1 | grep chain; SLIM_HALO_PAIR=$p timeout 300 python tools/micro.py 1024 30 2>&1 | grep chain; done
SLIM_HALO_PAIR=1 timeout 120 python tools/conv_trace.py 1024 1.0 2 2>&1 | tail -10
