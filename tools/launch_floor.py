"""Calibrate the per-kernel floor on this box: N tiny kernels captured in one CUDA graph."""
import time
import torch

t = torch.zeros(1, device="cuda")
big = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
t0 = time.time()
while time.time() - t0 < 1.0:          # warm the clocks for ~1 s
    big.add_(1)
torch.cuda.synchronize()
N = 200
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        t.add_(1)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for _ in range(N):
            t.add_(1)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    g.replay()
b.record()
torch.cuda.synchronize()
print(f"graph of {N} tiny kernels: {a.elapsed_time(b) / (10 * N) * 1e3:.2f} us per kernel")
x = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
a.record()
for _ in range(100):
    x.zero_()
b.record()
torch.cuda.synchronize()
print(f"64 MiB memset: {a.elapsed_time(b) / 100 * 1e3:.1f} us  ({64 * 2**20 / (a.elapsed_time(b) / 100 * 1e-3) / 1e9:.0f} GB/s)")
