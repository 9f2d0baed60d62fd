mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:conv -c 64 -o /tmp/r1_chain_b128 python tools/profile_chain.py --widths 0.25 0.5 0.75 1.0 --batch 128 > gpurun_out/ncu_chain.log 2>&1; echo ncu=$?
ncu -i /tmp/r1_chain_b128.ncu-rep --page raw --csv > gpurun_out/r1_chain_b128_raw.csv 2>/dev/null; ls -la gpurun_out/r1_chain_b128_raw.csv
