mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gn.py tests/test_gpu_executor.py -x -q > gpurun_out/t10.log 2>&1; echo tests=$?
tail -15 gpurun_out/t10.log
timeout 300 python bench.py --workload stream --executor native --steps 20 --warmup 3 > gpurun_out/native.json 2> gpurun_out/native.err; echo nat=$?
tail -3 gpurun_out/native.err; cat gpurun_out/native.json
timeout 300 python bench.py --workload handoff --steps 20 --warmup 3 > gpurun_out/handoff.json 2> gpurun_out/handoff.err; echo ho=$?
tail -3 gpurun_out/handoff.err; cat gpurun_out/handoff.json
timeout 600 python bench.py --norm gn --steps 300 --no-cpu > gpurun_out/bench_gn.json 2> gpurun_out/bench_gn.err; echo gn=$?
python -c "
import json;d=json.loads(open('gpurun_out/bench_gn.json').read().strip().splitlines()[-1]);print(d['value'],d['per_width_images_per_s'],d['kernel_time_by_kind_ms_per_step'])"
timeout 600 ncu --set full --clock-control none -k regex:gn_kernel -c 9 -o gpurun_out/r1_gn python tools/profile_chain.py --widths 1.0 --batch 128 --norm gn > gpurun_out/ncu_gn.log 2>&1; echo ncu=$?
ncu -i gpurun_out/r1_gn.ncu-rep --page raw --csv > gpurun_out/r1_gn_raw.csv 2>/dev/null
