for cap in "" "0.5,0.75,1,1" "0.5,0.5,1,1" "0.25,0.5,0.75,1" "0.35,0.5,0.75,1" "0.5,1,1,1" "0.75,0.75,1,1"; do
  SLIM_GRID_CAP="$cap" timeout 300 python bench.py --steps 300 --no-cpu --e2e-steps 20 --profile-steps 5 > /tmp/b.json 2>/dev/null
  python -c "
import json,sys;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('cap=[$cap]', round(d['value']), {k:round(v) for k,v in d['per_width_images_per_s'].items()})"
done
