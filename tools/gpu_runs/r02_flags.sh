# tile-granular dependencies (SLIM_TILE_FLAGS): bitwise tests, parity, timing A/B
set -o pipefail
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "segment_parity_all or chain_parity or composition or batch_independence or sampled_parity or graph_mode or max_batch_4096" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_bench_step.py tests/test_gpu_parity.py -q -x -k "bench_step or stream_executor or native_stream or sm_share" 2>&1 | tail -3
for f in 1 0 1 0; do SLIM_TILE_FLAGS=$f timeout 300 python bench.py --steps 30 --warmup 5 --energy-seconds 0 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('flags', $f, round(d['value']), round(d['ms_per_step'],4))"; done
for f in 1 0; do echo "== FLAGS=$f"; SLIM_TILE_FLAGS=$f timeout 300 python tools/micro.py 128 200 2>&1 | grep chain; SLIM_TILE_FLAGS=$f timeout 300 python tools/micro.py 1024 30 2>&1 | grep chain; done
