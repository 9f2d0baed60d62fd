python -m pytest tests/test_gpu_gn.py -m gpu -q -x 2>&1 | tail -3
python tools/micro.py 128 200 gn 2>&1 | tail -4
SLIM_NO_FUSED_GN=1 python tools/micro.py 128 200 gn 2>&1 | tail -4
python tools/micro.py 8 300 gn 2>&1 | tail -4
python bench.py --steps 200 --warmup 20 --no-cpu --norm gn --energy-seconds 0 --width-events 0 --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('gn step', round(d['value']), round(d['ms_per_step']*1e3,1), {k:round(v['images_per_s_alone']) for k,v in d['per_width'].items()})"
SLIM_NO_FUSED_GN=1 python bench.py --steps 200 --warmup 20 --no-cpu --norm gn --energy-seconds 0 --width-events 0 --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('gn step nofused', round(d['value']), round(d['ms_per_step']*1e3,1))"
