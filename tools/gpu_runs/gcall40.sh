for e in "X=1" "SLIM_HALO_NMAX=128" "SLIM_HALO_NMAX=32" "X=2"; do
  env $e timeout 300 python bench.py --steps 300 --no-cpu --e2e-steps 20 --profile-steps 5 > /tmp/b.json 2>/dev/null
  python -c "
import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('[$e]', round(d['value']), {k:round(v) for k,v in d['per_width_images_per_s'].items()})"
done
