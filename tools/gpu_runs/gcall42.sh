for cap in "" "0.2,0.3,0.4,0.55" "0.2,0.3,0.45,0.6" "0.25,0.35,0.45,0.6" "0.15,0.25,0.4,0.55" "0.2,0.3,0.4,0.5" "0.2,0.35,0.5,0.65"; do
  SLIM_GRID_CAP="$cap" timeout 300 python bench.py --steps 300 --no-cpu --e2e-steps 20 --profile-steps 5 > /tmp/b.json 2>/dev/null
  python -c "
import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('cap=[$cap]', round(d['value']))"
done
