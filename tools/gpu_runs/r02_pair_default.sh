# 2-SM halo conv on by default from B = 1024: parity (large-batch tests), timing
set -o pipefail
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_step.py -q -x -k "max_batch_4096 or sampled_parity or pair_mma or bench_step or batch_independence" 2>&1 | tail -2
timeout 300 python tools/micro.py 1024 30 2>&1 | grep chain
SLIM_HALO_PAIR=0 timeout 300 python tools/micro.py 1024 30 2>&1 | grep chain
timeout 300 python tools/micro.py 128 200 2>&1 | grep -E "r=1.0"
