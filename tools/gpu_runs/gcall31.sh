for i in 1 2 3; do
timeout 300 python bench.py --workload stream --executor native --steps 50 --warmup 5 --alg1-shares > /tmp/n.json 2>/tmp/n.err
python -c "
import json;d=json.loads(open('/tmp/n.json').read().strip().splitlines()[-1]);print('native eager shares', round(d['value']), d['batches_per_step_rank0'])" || tail -3 /tmp/n.err
done
