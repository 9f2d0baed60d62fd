timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "stream_executor" 2>&1 | tail -2
for m in 0 2 3 6; do
SLIM_GN_CAP_MULT=$m timeout 300 python bench.py --norm gn --steps 300 --no-cpu --e2e-steps 20 > /tmp/g.json 2>/dev/null
python -c "
import json;d=json.loads(open('/tmp/g.json').read().strip().splitlines()[-1]);print('gn mult=$m', round(d['value']))"
done
for l in 1 4; do
timeout 300 python bench.py --workload stream --lanes $l --steps 20 --warmup 3 > /tmp/s.json 2>/dev/null
python -c "
import json;d=json.loads(open('/tmp/s.json').read().strip().splitlines()[-1]);print('stream lanes=$l', round(d['value']))"
done
