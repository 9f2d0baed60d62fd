# re-entry: verify HEAD on a fresh box (build, all GPU tests, smoke, default bench line, micro)
set -o pipefail
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/r02v_bench_line.json 2> gpurun_out/r02v_bench_line.err; tail -c 600 gpurun_out/r02v_bench_line.json
timeout 300 python tools/micro.py 128 200 2>&1 | tee gpurun_out/r02v_micro128.txt
timeout 300 python tools/micro.py 1024 30 2>&1 | tee gpurun_out/r02v_micro1024.txt
