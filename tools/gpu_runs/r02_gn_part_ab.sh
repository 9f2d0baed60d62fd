# GN CFG2: fused narrow-width segment kernels under SM partitioning (SLIM_FUSED_PART 1 = capped, 2 = uncapped)
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(sys.argv[1], round(d["value"]), round(d["ms_per_step"],4))'
for f in 0 1 2 0 1 2; do SLIM_FUSED_PART=$f timeout 300 python bench.py --norm gn --steps 30 --warmup 5 --energy-seconds 0 --no-cpu 2>/dev/null | python -c "$P" "gn fused_part=$f"; done
