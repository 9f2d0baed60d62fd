"""Per-CTA phase timestamps of one conv launch (diagnostic; SLIM_CONV_TRACE=1).
Runs segment `seg` at width r, prints the stamps of its LAST conv launch."""
import ctypes
import os
import sys

os.environ["SLIM_CONV_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2510_09018_b200 as slim  # noqa: E402

B, r, seg = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])
net = slim.SlimNet(synth.make_weights(), synth.make_bn(), max_batch=B)
lib = slim.load_library()
lib.slimdbg_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
x = torch.from_numpy(synth.make_images(B)).to(torch.bfloat16).cuda()
h = x
for s in range(seg):
    h = net.forward(s, h, r, r)
for _ in range(20):
    out = net.forward(seg, h, r, r)
torch.cuda.synchronize()
buf = np.zeros(4096 * 8, np.uint64)
lib.slimdbg_trace(net.ctx, buf.ctypes.data, buf.size)
t = buf.reshape(-1, 8)[:148].astype(np.int64)
t = t[t[:, 0] > 0]
base = t[:, 0].min()
names = ["entry", "prologue", "producer_done", "mma_done", "epi_done", "stores_done", "exit"]
print(f"B={B} r={r} seg={seg} ctas={len(t)}")
for i, n in enumerate(names):
    col = t[:, i] - base
    print(f"{n:14s} min {col.min()/1e3:7.2f} med {np.median(col)/1e3:7.2f} max {col.max()/1e3:7.2f} us")
