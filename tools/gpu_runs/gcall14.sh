mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "fp32 or f32 or FP32" > gpurun_out/t14.log 2>&1; echo tests=$?
tail -4 gpurun_out/t14.log
timeout 600 python bench.py --dtype fp32 --steps 50 --warmup 3 --no-cpu > gpurun_out/bench_fp32.json 2> gpurun_out/bench_fp32.err; echo f=$?
tail -3 gpurun_out/bench_fp32.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_fp32.json').read().strip().splitlines()[-1]);print(d['value'],d['per_width_images_per_s'],d['roofline'])"
