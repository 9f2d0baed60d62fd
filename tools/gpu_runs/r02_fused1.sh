set -x
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fused or segment0 or chain or batch or graph or closed or nan" 2>&1 | tail -8
python tools/micro.py 128 200 2>&1 | tail -6
SLIM_NO_FUSED=1 python tools/micro.py 128 200 2>&1 | tail -6
python tools/micro.py 8 500 2>&1 | tail -6
python bench.py --workload cfg1 --steps 2000 --warmup 10 2>&1 | tail -1
SLIM_NO_FUSED=1 python bench.py --workload cfg1 --steps 2000 --warmup 10 2>&1 | tail -1
python bench.py --steps 200 --warmup 20 --no-cpu --width-events 0 > gpurun_out/b_fused.json 2>gpurun_out/b_fused.err; tail -c 600 gpurun_out/b_fused.json
SLIM_NO_FUSED=1 python bench.py --steps 200 --warmup 20 --no-cpu --width-events 0 > gpurun_out/b_nofused.json 2>&1; tail -c 300 gpurun_out/b_nofused.json
python bench.py --steps 200 --warmup 20 --no-cpu --width-events 1 > gpurun_out/b_fused_ev.json 2>&1
