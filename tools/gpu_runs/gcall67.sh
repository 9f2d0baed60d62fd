timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_handoff.py -x -q -k "stream_executor or handoff" 2>&1 | tail -1
timeout 300 python bench.py --workload stream --steps 200 --warmup 5 > /tmp/s.json 2>/dev/null; tail -c 300 /tmp/s.json
timeout 300 python bench.py --workload handoff --steps 50 --warmup 5 > /tmp/h.json 2>/dev/null
python -c "
import json;d=json.loads(open('/tmp/h.json').read().strip().splitlines()[-1]);print('handoff', round(d['value']))"
