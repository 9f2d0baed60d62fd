for i in 1 2; do
for env in "X=1" "SLIM_FUSED_PART=0" "SLIM_FUSED_PART=2" "SLIM_FUSED_SEGS=0"; do
  env $env python bench.py --steps 300 --warmup 20 --no-cpu --energy-seconds 0 --width-events 0 --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$env', round(d['value']), round(d['ms_per_step']*1e3,1), 'us')"
done; done
for sp in "0.2,0.3,0.5,0.6" "0.15,0.25,0.5,0.6" "0.25,0.35,0.5,0.6"; do
  SLIM_FUSED_PART=2 python bench.py --steps 300 --warmup 20 --no-cpu --energy-seconds 0 --width-events 0 --e2e-steps 1 --sm-share $sp 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('PART=2 $sp', round(d['value']), round(d['ms_per_step']*1e3,1), 'us')"
done
