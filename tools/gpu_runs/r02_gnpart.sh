python -m pytest tests/test_gpu_gn.py -m gpu -x -q 2>&1 | tail -6
python tools/micro.py 128 200 gn 2>&1 | tail -5
SLIM_GN_NO_PART=1 python tools/micro.py 128 200 gn 2>&1 | tail -5
python bench.py --steps 200 --warmup 20 --no-cpu --norm gn --energy-seconds 0 --width-events 0 --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('gn part', round(d['value']), round(d['ms_per_step']*1e3,1))"
SLIM_GN_NO_PART=1 python bench.py --steps 200 --warmup 20 --no-cpu --norm gn --energy-seconds 0 --width-events 0 --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('gn old', round(d['value']), round(d['ms_per_step']*1e3,1))"
