# end of round 2: every GPU test, smoke, the bench lines (CFG2 BN / GN / FP32, CFG1, CFG4 stream, CFG3 sweep),
# the ncu launch list of the bench and full captures (B=128 chain per width, B=1024 r=1 chain)
set -o pipefail
NCU=/usr/local/cuda/bin/ncu
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/rf_bench_line.json 2> gpurun_out/rf_bench_line.err; tail -c 200 gpurun_out/rf_bench_line.json; echo
timeout 600 python bench.py --norm gn > gpurun_out/rf_bench_gn_line.json 2>/dev/null
timeout 900 python bench.py --dtype fp32 --steps 10 --warmup 3 > gpurun_out/rf_bench_fp32_line.json 2>/dev/null
timeout 600 python bench.py --workload cfg1 > gpurun_out/rf_cfg1_line.json 2>/dev/null
timeout 600 python bench.py --workload stream > gpurun_out/rf_stream_line.json 2>/dev/null
timeout 900 python bench.py --workload sweep > gpurun_out/rf_sweep.json 2>/dev/null
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/rf_reference_line.json 2>/dev/null
$NCU --set full --clock-control none -k "regex:conv_|fused_kernel|stem_|fc_kernel" -s 18 -c 18 -o /tmp/rf_b4096_r1 python tools/profile_chain.py --widths 1.0 --batch 4096 --reps 2 > gpurun_out/rf_ncu_b4096.log 2>&1
$NCU -i /tmp/rf_b4096_r1.ncu-rep --page raw --csv > gpurun_out/rf_b4096_r1_raw.csv
echo lines rc=$?
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rf_launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --energy-seconds 0 --e2e-steps 1 --profile-steps 1 --width-events 0 > gpurun_out/rf_launch_bench.log 2>&1
echo launches rc=$?
$NCU --set full --clock-control none --import-source on -k "regex:conv_|fused_kernel|stem_|fc_kernel" -s 49 -c 49 \
    -o /tmp/rf_chain_b128 python tools/profile_chain.py --widths 0.25 0.5 0.75 1.0 --batch 128 --reps 2 > gpurun_out/rf_ncu_chain.log 2>&1
echo chain rc=$?
$NCU -i /tmp/rf_chain_b128.ncu-rep --page raw --csv > gpurun_out/rf_chain_b128_raw.csv
$NCU --set full --clock-control none -k "regex:conv_|fused_kernel|stem_|fc_kernel" -s 18 -c 18 -o /tmp/rf_b1024_r1 \
    python tools/profile_chain.py --widths 1.0 --batch 1024 --reps 2 > gpurun_out/rf_ncu_b1024.log 2>&1
echo b1024 rc=$?
$NCU -i /tmp/rf_b1024_r1.ncu-rep --page raw --csv > gpurun_out/rf_b1024_r1_raw.csv
du -sh gpurun_out
