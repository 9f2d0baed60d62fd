mkdir -p gpurun_out
timeout 600 python bench.py --dtype fp32 --steps 50 --warmup 3 --no-cpu > gpurun_out/bench_fp32.json 2> gpurun_out/bench_fp32.err; echo f=$?
tail -3 gpurun_out/bench_fp32.err; cat gpurun_out/bench_fp32.json
