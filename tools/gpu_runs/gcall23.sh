for sh in none auto; do
timeout 300 python bench.py --workload stream --executor native --steps 20 --warmup 3 --sm-share $sh > /tmp/n.json 2>/dev/null
python -c "
import json;d=json.loads(open('/tmp/n.json').read().strip().splitlines()[-1]);print('native share=$sh', round(d['value']), d['batches_per_step_rank0'])"
done
for sh in none auto; do
timeout 300 python bench.py --norm gn --steps 300 --no-cpu --sm-share $sh > /tmp/g.json 2>/dev/null
python -c "
import json;d=json.loads(open('/tmp/g.json').read().strip().splitlines()[-1]);print('gn share=$sh', round(d['value']), round(d['e2e']['value']))"
done
timeout 300 python bench.py --widths 0.3 0.6 0.9 --steps 300 --no-cpu > /tmp/u.json 2>/dev/null
python -c "
import json;d=json.loads(open('/tmp/u.json').read().strip().splitlines()[-1]);print('universal auto', round(d['value']), round(d['e2e']['value']))"
