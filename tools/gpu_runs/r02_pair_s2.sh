# 2-SM MMA for the stride-2 convs: bitwise tests, timing (SLIM_HALO_PAIR=2: stride-2 convs only)
set -o pipefail
for s in 1 2 3; do SLIM_HALO_PAIR=1 timeout 300 python tools/pair_check.py $s 1.0 64 2>&1 | tail -1; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "pair_mma" 2>&1 | tail -2
for p in 0 2 1; do echo "== PAIR=$p"; SLIM_HALO_PAIR=$p timeout 300 python tools/micro.py 1024 30 2>&1 | grep chain; SLIM_HALO_PAIR=$p timeout 300 python tools/micro.py 128 200 2>&1 | grep -E "r=0.75|r=1.0"; done
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(sys.argv[1], round(d["value"]), round(d["ms_per_step"],4))'
for p in 0 2 0 2; do SLIM_HALO_PAIR=$p timeout 300 python bench.py --steps 30 --warmup 5 --energy-seconds 0 --no-cpu 2>/dev/null | python -c "$P" "pair=$p"; done
