timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "chunking or max_batch" 2>&1 | tail -2
timeout 600 python bench.py --workload sweep --steps 20 --warmup 3 > /tmp/sw.json 2>/dev/null
python -c "
import json
for l in open('/tmp/sw.json'):
    d=json.loads(l)
    if d['config']['batch']>=512: print(d['config']['batch'], d['config'].get('width'), round(d['value']), round(d.get('tflops',0)))
"
