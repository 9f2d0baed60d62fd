for sh in auto none "0.25,0.35,0.45,0.55" "0.15,0.25,0.35,0.45" "0.3,0.4,0.5,0.6"; do
  timeout 300 python bench.py --norm gn --steps 300 --no-cpu --e2e-steps 20 --profile-steps 5 --sm-share $sh > /tmp/g.json 2>/dev/null
  python -c "
import json;d=json.loads(open('/tmp/g.json').read().strip().splitlines()[-1]);print('gn share=$sh', round(d['value']))"
done
