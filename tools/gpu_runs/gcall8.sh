mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_handoff.py tests/test_gpu_executor.py -x -q > gpurun_out/handoff_tests.log 2>&1; echo tests=$?
tail -25 gpurun_out/handoff_tests.log
timeout 300 python bench.py --workload stream --executor greedy --steps 20 --warmup 3 > gpurun_out/greedy.json 2> gpurun_out/greedy.err; echo g=$?
tail -3 gpurun_out/greedy.err; cat gpurun_out/greedy.json
