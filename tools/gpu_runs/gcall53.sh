for o in asc desc asc desc; do
  timeout 300 python bench.py --steps 300 --no-cpu --e2e-steps 20 --profile-steps 5 --launch-order $o > /tmp/b.json 2>/tmp/b.err
  python -c "
import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('order=$o', round(d['value']))" || tail -2 /tmp/b.err
done
