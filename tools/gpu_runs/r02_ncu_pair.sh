# ncu --set full of the B=1024 r=1 chain with the 2-SM halo conv (SLIM_HALO_PAIR=1)
NCU=/usr/local/cuda/bin/ncu
SLIM_HALO_PAIR=1 $NCU --set full --clock-control none -k "regex:conv_|fused_kernel|stem_|fc_kernel" -s 18 -c 18 -o /tmp/r02_b1024_r1_pair \
    python tools/profile_chain.py --widths 1.0 --batch 1024 --reps 2 > gpurun_out/r02_ncu_b1024_pair.log 2>&1
echo b1024 rc=$?
$NCU -i /tmp/r02_b1024_r1_pair.ncu-rep --page raw --csv > gpurun_out/r02_b1024_r1_pair_raw.csv
