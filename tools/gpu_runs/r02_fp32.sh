# FP32 mode after the conflict-free A reads: parity, layer times, bench line
set -o pipefail
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gn.py tests/test_gpu_universal.py -q -x -k "fp32" 2>&1 | tail -2
timeout 600 python tools/layer_times.py 128 3 bn fp32 2>&1 | grep -E "sum of launches|seg0 L 1|seg1 L 1|seg2 L 1|seg3 L 1"
timeout 900 python bench.py --dtype fp32 --steps 10 --warmup 3 --energy-seconds 0 > gpurun_out/r02_fp32_line.json 2>/dev/null; tail -c 300 gpurun_out/r02_fp32_line.json
