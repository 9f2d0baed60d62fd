timeout 600 python -m pytest tests/test_gpu_gn.py -x -q 2>&1 | tail -2
for i in 1 2; do
timeout 300 python bench.py --norm gn --steps 300 --no-cpu --e2e-steps 50 > /tmp/g.json 2>/dev/null
python -c "
import json;d=json.loads(open('/tmp/g.json').read().strip().splitlines()[-1]);print('gn', round(d['value']), round(d['e2e']['value']), d['kernel_time_by_kind_ms_per_step'])"
done
