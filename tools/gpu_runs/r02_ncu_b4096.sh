# ncu --set full of the B=4096 r=1 chain (north-star tensor-pipe target at large batch)
NCU=/usr/local/cuda/bin/ncu
$NCU --set full --clock-control none -k "regex:conv_|fused_kernel|stem_|fc_kernel" -s 18 -c 18 -o /tmp/rf_b4096_r1 \
    python tools/profile_chain.py --widths 1.0 --batch 4096 --reps 2 > gpurun_out/rf_ncu_b4096.log 2>&1
echo rc=$?
$NCU -i /tmp/rf_b4096_r1.ncu-rep --page raw --csv > gpurun_out/rf_b4096_r1_raw.csv
