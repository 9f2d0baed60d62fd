# HEAD verification: all GPU tests, smoke, default bench line; CFG2 with the 2-SM halo conv (A/B); GN line
set -o pipefail
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/r02v2_bench_line.json 2> gpurun_out/r02v2_bench_line.err; tail -c 300 gpurun_out/r02v2_bench_line.json; echo
for p in 0 1 0 1; do SLIM_HALO_PAIR=$p timeout 300 python bench.py --steps 30 --warmup 5 --energy-seconds 0 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pair', $p, round(d['value']), round(d['ms_per_step'],4))"; done
timeout 600 python bench.py --norm gn > gpurun_out/r02v2_bench_gn_line.json 2>/dev/null; tail -c 200 gpurun_out/r02v2_bench_gn_line.json
