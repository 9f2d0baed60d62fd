mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
cat gpurun_out/bench.json
timeout 300 python bench.py --workload stream --steps 20 --warmup 3 > gpurun_out/stream.json 2>/dev/null; tail -c 400 gpurun_out/stream.json
