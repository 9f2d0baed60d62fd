python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fused" 2>&1 | tail -3
SLIM_FUSED_SEGS=14 python tools/fused_trace2.py 8 3 0.25
python tools/micro.py 128 200 2>&1 | tee gpurun_out/micro128_r02.txt
python tools/micro.py 8 500 2>&1 | tee gpurun_out/micro8_r02.txt
SLIM_NO_FUSED=1 python tools/micro.py 128 200 2>&1 | tee gpurun_out/micro128_nofused.txt
SLIM_NO_FUSED=1 python tools/micro.py 8 500 2>&1 | tee gpurun_out/micro8_nofused.txt
