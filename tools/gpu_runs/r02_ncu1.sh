# round-2 ncu evidence: bench launch list, full capture of one B=128 chain per width, B=1024 r=1 chain
# (.ncu-rep files are exported to csv and deleted: gpurun_out must stay under 64 MiB)
NCU=/usr/local/cuda/bin/ncu
python -c "import __graft_entry__ as g; g.build()"
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --energy-seconds 0 --e2e-steps 1 --profile-steps 1 --width-events 0 > gpurun_out/r02_launch_bench.log 2>&1
echo launches rc=$?
# one chain per width at B=128: skip the first repetition's launches (49 of ours)
$NCU --set full --clock-control none --import-source on -k "regex:conv_|fused_kernel|stem_|fc_kernel" -s 49 -c 49 \
    -o /tmp/r02_chain_b128 python tools/profile_chain.py --widths 0.25 0.5 0.75 1.0 --batch 128 --reps 2 > gpurun_out/r02_ncu_chain.log 2>&1
echo chain rc=$?
$NCU -i /tmp/r02_chain_b128.ncu-rep --page raw --csv > gpurun_out/r02_chain_b128_raw.csv
$NCU -i /tmp/r02_chain_b128.ncu-rep --page details --csv > gpurun_out/r02_chain_b128_details.csv
$NCU --set full --clock-control none -k "regex:conv_|fused_kernel|stem_|fc_kernel" -s 18 -c 18 -o /tmp/r02_b1024_r1 \
    python tools/profile_chain.py --widths 1.0 --batch 1024 --reps 2 > gpurun_out/r02_ncu_b1024.log 2>&1
echo b1024 rc=$?
$NCU -i /tmp/r02_b1024_r1.ncu-rep --page raw --csv > gpurun_out/r02_b1024_r1_raw.csv
du -sh gpurun_out; ls -la gpurun_out/
