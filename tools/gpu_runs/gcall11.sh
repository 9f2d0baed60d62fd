mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -4 gpurun_out/gpu_tests.log
timeout 300 python bench.py --workload handoff --steps 20 --warmup 3 > gpurun_out/handoff.json 2> gpurun_out/handoff.err; echo ho=$?
tail -3 gpurun_out/handoff.err; cat gpurun_out/handoff.json
