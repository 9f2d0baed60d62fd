python tools/fused_trace.py 8 0.25
python tools/fused_trace.py 8 0.5
python tools/fused_trace.py 128 0.25
python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -4
