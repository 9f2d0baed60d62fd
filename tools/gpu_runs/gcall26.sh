timeout 600 python -m pytest tests/test_gpu_gn.py -x -q 2>&1 | tail -2
for sh in none auto; do
timeout 300 python bench.py --norm gn --steps 300 --no-cpu --sm-share $sh > /tmp/g.json 2>/dev/null
python -c "
import json;d=json.loads(open('/tmp/g.json').read().strip().splitlines()[-1]);print('gn share=$sh', round(d['value']), round(d['e2e']['value']))"
done
