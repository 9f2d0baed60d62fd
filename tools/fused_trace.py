"""Phase stamps of the fused segment-0 kernel (diagnostic; SLIM_CONV_TRACE=1): CTA 0's thread 0
(epilogue) and the MMA warp, us since kernel entry.   python tools/fused_trace.py [B] [r]"""
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

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
r = float(sys.argv[2]) if len(sys.argv) > 2 else 0.25
net = slim.SlimNet(synth.make_weights(), synth.make_bn(), max_batch=max(B, 16))
lib = slim.load_library()
lib.slimdbg_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
x = torch.from_numpy(synth.make_images(B)).to(torch.bfloat16).cuda()
for _ in range(20):
    net.forward(0, x, r, r)
torch.cuda.synchronize()
buf = np.zeros(4096 * 8, np.uint64)
lib.slimdbg_trace(net.ctx, buf.ctypes.data, buf.size)
t = buf[8192:8192 + 32].astype(np.int64)
base = t[0]
names = ["entry", "prologue", "pdl", "img", "stem0", "stem1", "L0", "L1", "L2", "L3"]
print(f"B={B} r={r} epilogue thread: " + " ".join(f"{n}={(v - base) / 1e3:.2f}" for n, v in zip(names, t[:16]) if v))
print("MMA warp: " + " ".join(f"{n}={(v - base) / 1e3:.2f}" for n, v in zip(names, t[16:32]) if v))
