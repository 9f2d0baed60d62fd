mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:gn_kernel -c 9 -o /tmp/r1_gn python tools/profile_chain.py --widths 1.0 --batch 128 --norm gn > gpurun_out/ncu_gn.log 2>&1; echo ncu_gn=$?
ncu -i /tmp/r1_gn.ncu-rep --page raw --csv > gpurun_out/r1_gn_raw.csv 2>/dev/null
