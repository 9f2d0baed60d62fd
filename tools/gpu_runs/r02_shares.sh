# CFG2 SM-share sweep at HEAD (per-width shares r = .25/.5/.75/1)
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(sys.argv[1], round(d["value"]), round(d["ms_per_step"],4))'
for s in auto 0.2,0.3,0.4,0.5 0.15,0.25,0.45,0.6 0.2,0.3,0.45,0.55 0.25,0.35,0.45,0.55 0.1,0.25,0.45,0.65 0.2,0.25,0.4,0.6 0.15,0.3,0.5,0.6 0.3,0.4,0.5,0.6 0.2,0.3,0.5,0.7 auto; do
  timeout 300 python bench.py --steps 40 --warmup 5 --energy-seconds 0 --no-cpu --sm-share $s 2>/dev/null | python -c "$P" "$s"; done
