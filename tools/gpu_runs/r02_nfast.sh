# N-fastest tile order: bitwise, timing at B = 128 / 1024 / 4096 (auto pairing on)
set -o pipefail
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tile_order" 2>&1 | tail -2
for n in 0 1; do echo "== NFAST=$n"; for B in 128 1024 4096; do r=$((25600 / B)); [ $r -lt 8 ] && r=8; SLIM_HALO_NFAST=$n timeout 300 python tools/micro.py $B $r 2>&1 | grep -E "r=0.75|r=1.0"; done; done
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(sys.argv[1], round(d["value"]), round(d["ms_per_step"],4))'
for n in 0 1; do SLIM_HALO_NFAST=$n timeout 300 python bench.py --steps 30 --warmup 5 --energy-seconds 0 --no-cpu 2>/dev/null | python -c "$P" "cfg2 nfast=$n"; done
