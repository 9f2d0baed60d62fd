mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gn.py -x -q > gpurun_out/gn_tests.log 2>&1; echo gn_tests=$?
tail -4 gpurun_out/gn_tests.log
timeout 600 python bench.py --norm gn --steps 300 --no-cpu > gpurun_out/bench_gn.json 2> gpurun_out/bench_gn.err; echo bench=$?
python -c "
import json;d=json.loads(open('gpurun_out/bench_gn.json').read().strip().splitlines()[-1]);print(d['value'],d['per_width_images_per_s'],d['kernel_time_by_kind_ms_per_step'])"
