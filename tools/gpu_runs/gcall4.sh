mkdir -p gpurun_out
python tools/layer_times.py 128 20 gn > gpurun_out/layer_times_gn.txt 2>&1
python tools/micro.py 128 200 gn > gpurun_out/micro_gn.txt 2>&1
python tools/micro.py 128 200 bn > gpurun_out/micro_bn.txt 2>&1
cat gpurun_out/micro_gn.txt gpurun_out/micro_bn.txt; grep -A40 "r=1.0" gpurun_out/layer_times_gn.txt
