mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -5 gpurun_out/gpu_tests.log
timeout 300 python bench.py --workload stream --executor greedy --steps 20 --warmup 3 > gpurun_out/greedy.json 2> gpurun_out/greedy.err; echo g=$?
tail -3 gpurun_out/greedy.err; cat gpurun_out/greedy.json
