for i in 1 2; do
for pr in none wide narrow; do for lo in asc desc; do
  python bench.py --steps 300 --warmup 20 --no-cpu --energy-seconds 0 --width-events 0 --e2e-steps 1 --stream-priority $pr --launch-order $lo 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('prio=$pr order=$lo', round(d['value']), round(d['ms_per_step']*1e3,1), 'us')"
done; done; done
