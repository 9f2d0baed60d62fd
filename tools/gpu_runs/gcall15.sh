mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
tail -1 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
cat gpurun_out/bench.json
timeout 300 python bench.py --workload cfg1 > gpurun_out/cfg1.json 2> gpurun_out/cfg1.err; echo cfg1=$?
cat gpurun_out/cfg1.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --profile-steps 1 --e2e-steps 1 > gpurun_out/ncu_bench.log 2>&1; echo ncu=$?
