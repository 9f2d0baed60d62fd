# PDL on/off A/B: CFG2 step, each chain alone; FP32 128x64 kernel for every layer (A/B)
for p in 1 0 1 0; do SLIM_PDL=$p timeout 300 python bench.py --steps 30 --warmup 5 --energy-seconds 0 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pdl', $p, round(d['value']), round(d['ms_per_step'],4))"; done
for p in 1 0; do echo "== PDL=$p"; SLIM_PDL=$p timeout 300 python tools/micro.py 128 200 2>&1 | grep chain; done
for g in 0 1; do timeout 600 python tools/layer_times.py 128 3 bn fp32 2>&1 | grep -E "sum of launches"; done
SLIM_F32_GEMM128=1 timeout 600 python tools/layer_times.py 128 3 bn fp32 2>&1 | grep -E "sum of launches"
