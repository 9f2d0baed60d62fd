python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err; tail -c 300 gpurun_out/r02_bench_default.json
python bench.py --steps 300 --warmup 20 --no-cpu > gpurun_out/r02_bench_300.json 2>/dev/null; tail -c 200 gpurun_out/r02_bench_300.json
python bench.py --steps 200 --warmup 20 --no-cpu --norm gn --energy-seconds 1 > gpurun_out/r02_bench_gn.json 2>/dev/null; tail -c 200 gpurun_out/r02_bench_gn.json
python tools/micro.py 128 200 gn 2>&1 | tee gpurun_out/r02_micro_gn.txt
python bench.py --workload cfg1 --steps 2000 --warmup 10 > gpurun_out/r02_cfg1.json 2>/dev/null; cat gpurun_out/r02_cfg1.json
python bench.py --workload sweep --steps 100 --warmup 5 > gpurun_out/r02_sweep.json 2>/dev/null; wc -l gpurun_out/r02_sweep.json
python bench.py --workload stream --steps 50 --warmup 5 > gpurun_out/r02_stream.json 2>/dev/null; tail -c 300 gpurun_out/r02_stream.json
python bench.py --workload stream --policy ppo_frozen --steps 50 --warmup 5 > gpurun_out/r02_stream_ppo.json 2>/dev/null; tail -c 300 gpurun_out/r02_stream_ppo.json
python bench.py --dtype fp32 --steps 20 --warmup 3 --no-cpu --energy-seconds 1 > gpurun_out/r02_bench_fp32.json 2>/dev/null; tail -c 200 gpurun_out/r02_bench_fp32.json
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r02_ref.json; cat gpurun_out/r02_ref.json
