"""Phase stamps of the fused segment-s kernel (diagnostic; SLIM_CONV_TRACE=1), us since entry.
    SLIM_FUSED_SEGS=14 python tools/fused_trace2.py B seg r"""
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

B, seg, r = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
net = slim.SlimNet(synth.make_weights(), synth.make_bn(), max_batch=max(B, 16))
lib = slim.load_library()
lib.slimdbg_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
H = 32 >> (seg - 1)
C = synth.active_channels(r, synth.BASE_CHANNELS[seg - 1])
x = torch.from_numpy(np.abs(synth.make_images(B * H * H * C // 3072 + 1).reshape(-1))[:B * H * H * C]
                     .reshape(B, H, H, C)).to(torch.bfloat16).cuda()
for _ in range(10):
    net.forward(seg, x, r, r)
torch.cuda.synchronize()
buf = np.zeros(4096 * 8, np.uint64)
lib.slimdbg_trace(net.ctx, buf.ctypes.data, buf.size)
t = buf[8192 + 64:8192 + 64 + 48].astype(np.int64)
base = t[0]
fmt = lambda v: " ".join(f"{(x - base) / 1e3:.2f}" for x in v if x)
print(f"B={B} seg={seg} r={r}\n epilogue: {fmt(t[:16])}\n mma:      {fmt(t[16:32])}\n producer: {fmt(t[32:48])}")
