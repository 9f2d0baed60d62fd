# 2-CTA MMA microbenchmark; CFG3 sweep with the fused-segment batch limits; fused-limit parity spot check
set -o pipefail
(cd tools/ubench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pair_mma pair_mma.cu && timeout 60 ./pair_mma)
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "batch_independence or max_batch_4096 or fused" 2>&1 | tail -3
timeout 900 python bench.py --workload sweep > gpurun_out/r02_sweep2.json 2> gpurun_out/r02_sweep2.err; tail -c 300 gpurun_out/r02_sweep2.json
for B in 2048 4096; do timeout 300 python tools/micro.py $B 10 2>&1 | grep chain; done
