for g in "" "--alg1-graphs"; do for i in 1 2 3; do
timeout 300 python bench.py --workload stream --executor native --steps 20 --warmup 3 $g > /tmp/n.json 2>/dev/null
python -c "
import json;d=json.loads(open('/tmp/n.json').read().strip().splitlines()[-1]);print('native $g', round(d['value']), d['batches_per_step_rank0'])"
done; done
timeout 300 python bench.py --workload stream --executor greedy --steps 20 --warmup 3 > /tmp/n.json 2>/dev/null
python -c "
import json;d=json.loads(open('/tmp/n.json').read().strip().splitlines()[-1]);print('greedy eager', round(d['value']))"
