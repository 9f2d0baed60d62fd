timeout 600 python -m pytest tests -m gpu -x -q -k "fp32 or f32 or FP32" 2>&1 | tail -2
for sh in auto none; do
timeout 600 python bench.py --dtype fp32 --steps 50 --warmup 3 --no-cpu --sm-share $sh > /tmp/f.json 2>/dev/null
python -c "
import json;d=json.loads(open('/tmp/f.json').read().strip().splitlines()[-1]);print('fp32 share=$sh', round(d['value']), {k:round(v) for k,v in d['per_width_images_per_s'].items()}, round(d['roofline']['frac'],3))"
done
