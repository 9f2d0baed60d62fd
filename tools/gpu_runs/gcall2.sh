set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gn.py -x -q > gpurun_out/gn_tests.log 2>&1; echo gn_tests=$?
tail -15 gpurun_out/gn_tests.log
timeout 600 python bench.py --norm gn --steps 300 --no-cpu > gpurun_out/bench_gn.json 2> gpurun_out/bench_gn.err; echo bench=$?
tail -3 gpurun_out/bench_gn.err
cat gpurun_out/bench_gn.json
