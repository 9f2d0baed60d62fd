for sc in "" "1.3,1,1,1" "1,1,0.8,0.6" "1.3,1.1,0.9,0.7" "0.8,1,1.2,1.4" "1.5,1,1,1" "1.2,1.2,1,1"; do
  SLIM_SEG_CAP_SCALE="$sc" timeout 300 python bench.py --steps 300 --no-cpu --e2e-steps 20 --profile-steps 5 > /tmp/b.json 2>/dev/null
  python -c "
import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('segscale=[$sc]', round(d['value']))"
done
