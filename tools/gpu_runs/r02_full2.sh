python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python tools/micro.py 128 200 2>&1 | tee gpurun_out/micro128.txt
python tools/micro.py 8 500 2>&1 | tee gpurun_out/micro8.txt
python bench.py --steps 200 --warmup 20 --no-cpu > gpurun_out/b3.json 2>gpurun_out/b3.err; tail -c 400 gpurun_out/b3.json
