mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_executor.py -x -q > gpurun_out/exec_tests.log 2>&1; echo exec_tests=$?
tail -30 gpurun_out/exec_tests.log
