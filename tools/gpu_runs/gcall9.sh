mkdir -p gpurun_out
timeout 600 python bench.py --norm gn > gpurun_out/bench_gn.json 2> gpurun_out/bench_gn.err; echo gn=$?
timeout 600 python bench.py --widths 0.3 0.6 0.9 --steps 300 > gpurun_out/bench_uw.json 2> gpurun_out/bench_uw.err; echo uw=$?
timeout 300 python bench.py --workload handoff --steps 20 --warmup 3 > gpurun_out/handoff.json 2> gpurun_out/handoff.err; echo ho=$?
timeout 600 ncu --set full --clock-control none -k regex:gn_kernel -c 9 -o gpurun_out/r1_gn python tools/profile_chain.py --widths 1.0 --batch 128 --norm gn > gpurun_out/ncu_gn.log 2>&1; echo ncu=$?
ncu -i gpurun_out/r1_gn.ncu-rep --page raw --csv > gpurun_out/r1_gn_raw.csv 2>/dev/null
tail -2 gpurun_out/bench_uw.err gpurun_out/handoff.err
cat gpurun_out/bench_gn.json gpurun_out/bench_uw.json gpurun_out/handoff.json
