for pol in slim random; do
  timeout 300 python bench.py --workload stream --policy $pol --steps 1000 --warmup 5 > /tmp/s.json 2>/tmp/s.err
  python -c "
import json;d=json.loads(open('/tmp/s.json').read().strip().splitlines()[-1]);print('$pol', round(d['value']), d['energy_j_per_image'], d['mean_batch_rank0'], d['clocks']['sm_mhz'])" || tail -2 /tmp/s.err
done
