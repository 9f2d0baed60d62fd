timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "stream_executor" 2>&1 | tail -1
for l in 4 8 12 4 8; do
timeout 300 python bench.py --workload stream --lanes $l --steps 200 --warmup 5 > /tmp/s.json 2>/dev/null
python -c "
import json;d=json.loads(open('/tmp/s.json').read().strip().splitlines()[-1]);print('lanes=$l', round(d['value']))"
done
