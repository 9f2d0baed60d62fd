python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fused or segment0 or batch or graph or closed or nan or chain" 2>&1 | tail -3
for e in X=1 SLIM_SEG0_CLUSTER=0; do echo $e; env $e python bench.py --workload cfg1 --steps 2000 --warmup 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['us_per_call'],2), 'us', round(d['ratio_to_launch_floor'],2), 'x floor', d['gpu_launches_per_call'])"; env $e python tools/micro.py 8 500 2>&1 | grep "r=0.25\|r=0.5"; done
python tools/fused_trace.py 8 0.25
