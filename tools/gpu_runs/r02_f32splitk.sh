# FP32 split-K for the under-filled layers (segments 2-3): parity, layer times, bench line
set -o pipefail
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gn.py tests/test_gpu_universal.py -q -x -k "fp32" 2>&1 | tail -2
timeout 600 python tools/layer_times.py 128 3 bn fp32 2>&1 | grep -E "sum of launches|seg2 L 1|seg3 L 1|seg3 L 3"
SLIM_F32_NO_SPLITK=1 timeout 600 python tools/layer_times.py 128 3 bn fp32 2>&1 | grep -E "sum of launches"
timeout 900 python bench.py --dtype fp32 --steps 10 --warmup 3 --energy-seconds 0 > gpurun_out/r02_fp32b_line.json 2>/dev/null; tail -c 150 gpurun_out/r02_fp32b_line.json; python -c "
import json; d=json.loads(open('gpurun_out/r02_fp32b_line.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'])"
