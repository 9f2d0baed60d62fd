timeout 600 python -m pytest tests/test_gpu_handoff.py -x -q 2>&1 | tail -2
for i in 1 2; do
timeout 300 python bench.py --workload stream --executor native --steps 20 --warmup 3 > /tmp/n.json 2>/dev/null
python -c "
import json;d=json.loads(open('/tmp/n.json').read().strip().splitlines()[-1]);print('native', round(d['value']), d['batches_per_step_rank0'])"
done
timeout 300 python bench.py --workload handoff --steps 20 --warmup 3 > /tmp/h.json 2>/dev/null
python -c "
import json;d=json.loads(open('/tmp/h.json').read().strip().splitlines()[-1]);print('handoff lanes4', round(d['value']))"
timeout 300 python bench.py --workload stream --steps 20 --warmup 3 > gpurun_out/stream.json 2>/dev/null; cat gpurun_out/stream.json
