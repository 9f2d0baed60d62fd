"""Per-tile %globaltimer stamps of the stem kernel's CTA 0 (diagnostic; SLIM_CONV_TRACE=1)."""
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

B, r = int(sys.argv[1]), float(sys.argv[2])
net = slim.SlimNet(synth.make_weights(), synth.make_bn(), max_batch=B)
lib = slim.load_library()
lib.slimdbg_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
x = torch.from_numpy(synth.make_images(B)).to(torch.bfloat16).cuda()
os.environ.pop("SLIM_CONV_TRACE")
for _ in range(10):
    net.forward(0, x, r, r)   # stem + convs; the convs overwrite the trace -> read it right after a stem-only run
torch.cuda.synchronize()
buf = np.zeros(4096, np.uint64)
lib.slimdbg_trace(net.ctx, buf.ctypes.data, buf.size)
d = buf[3584:3584 + 320].astype(np.int64)
t0 = d[256]
print(f"B={B} r={r}: prologue done {(d[257] - t0) / 1e3:.2f} us, exit {(d[258] - t0) / 1e3:.2f} us")
names = ["halo issued", "A built", "MMA issued", "stored"]
for ti in range(8):
    row = [f"{names[k]}={(d[k * 64 + ti] - t0) / 1e3:6.2f}" for k in range(4) if d[k * 64 + ti]]
    if row:
        print(f"tile {ti}: " + "  ".join(row))
