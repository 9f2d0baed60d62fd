set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 600 ncu --set full --clock-control none -k regex:conv -c 20 -o gpurun_out/r1_b1024 python tools/profile_chain.py --widths 1.0 --batch 1024 --reps 1 > gpurun_out/ncu1024.log 2>&1; echo ncu=$?
ncu -i gpurun_out/r1_b1024.ncu-rep --page raw --csv > gpurun_out/r1_b1024_raw.csv 2>/dev/null
tail -3 gpurun_out/gpu_tests.log; cat gpurun_out/smoke.log | tail -2; cat gpurun_out/bench.json
