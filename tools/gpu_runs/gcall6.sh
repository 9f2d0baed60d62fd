mkdir -p gpurun_out
timeout 300 python bench.py --workload stream --steps 20 --warmup 3 > gpurun_out/stream.json 2> gpurun_out/stream.err; echo s=$?
timeout 300 python bench.py --workload stream --executor greedy --steps 20 --warmup 3 > gpurun_out/greedy.json 2> gpurun_out/greedy.err; echo g=$?
timeout 300 python bench.py --workload stream --executor greedy --q-th 64 --n-new 4 --steps 20 --warmup 3 > gpurun_out/greedy2.json 2> gpurun_out/greedy2.err; echo g2=$?
tail -3 gpurun_out/greedy.err
cat gpurun_out/stream.json gpurun_out/greedy.json gpurun_out/greedy2.json
