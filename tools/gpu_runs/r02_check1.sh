set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python bench.py --steps 20 --warmup 5 > gpurun_out/b1.json 2> gpurun_out/b1.err; tail -2 gpurun_out/b1.err
python bench.py --steps 200 --warmup 20 --no-cpu > gpurun_out/b2.json 2> gpurun_out/b2.err; tail -2 gpurun_out/b2.err
python bench.py --workload stream --steps 20 --warmup 3 > gpurun_out/s1.json 2>gpurun_out/s1.err; tail -2 gpurun_out/s1.err
python bench.py --workload stream --policy ppo_frozen --steps 20 --warmup 3 > gpurun_out/s2.json 2>gpurun_out/s2.err; tail -2 gpurun_out/s2.err
python bench.py --workload stream --repeat-stream --steps 20 --warmup 3 > gpurun_out/s3.json 2>gpurun_out/s3.err
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/ref.json
