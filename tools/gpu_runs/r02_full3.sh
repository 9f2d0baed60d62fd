python -m pytest tests -m gpu -q 2>&1 | tail -4
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/r02_bench_line.json 2> gpurun_out/r02_bench_line.err; tail -c 1500 gpurun_out/r02_bench_line.json
python tools/micro.py 128 200 2>&1 | tee gpurun_out/r02_micro128_final.txt
