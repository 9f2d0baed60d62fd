timeout 600 python -m pytest tests/test_gpu_executor.py -x -q 2>&1 | tail -2
for i in 1 2 3; do
timeout 300 python bench.py --workload stream --executor native --steps 50 --warmup 5 > /tmp/n.json 2>/tmp/n.err
python -c "
import json;d=json.loads(open('/tmp/n.json').read().strip().splitlines()[-1]);print('native eager', round(d['value']), d['batches_per_step_rank0'])" || tail -3 /tmp/n.err
done
for i in 1 2; do
timeout 300 python bench.py --workload stream --executor native --steps 50 --warmup 5 --alg1-graphs > /tmp/n.json 2>/tmp/n.err
python -c "
import json;d=json.loads(open('/tmp/n.json').read().strip().splitlines()[-1]);print('native graphs', round(d['value']), d['batches_per_step_rank0'])" || tail -3 /tmp/n.err
done
