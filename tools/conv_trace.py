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
# per-tile detail of CTA 0 (halo kernel only): roles A(0) MMA(1) EPI(2), 4 points each
d = buf[2048:2048 + 4 * 256].astype(np.int64).reshape(4, 64, 4)
if d.any():
    t0 = buf.reshape(-1, 8)[0, 1].astype(np.int64)
    labels = {0: ["A:start", "A:res_slot", "A:a_slot", "-"], 1: ["M:start", "M:tmem", "M:a_full", "M:commit"],
              2: ["E:t_full", "E:rd_done", "E:res_ok", "E:store"], 3: ["M:mma0", "M:mma_end", "M:c_a", "M:c_t"]}
    for ti in range(8):
        row = []
        for role in (0, 1, 3, 2):
            for pt in range(4):
                v = d[role, ti, pt]
                if v:
                    row.append(f"{labels[role][pt]}={(v - t0) / 1e3:6.2f}")
        if row:
            print(f"tile {ti}: " + " ".join(row))
w = buf[2048:2048 + 148 * 8].astype(np.int64).reshape(148, 8)
w = w[w[:, 2] > 0]
if len(w):
    med = np.median(w, axis=0) / 1e3
    print(f"median per-CTA waits (us): A-prod empty {med[0]:.2f}  B-prod empty {med[1]:.2f}  MMA full {med[2]:.2f}  "
          f"MMA tmem-empty {med[3]:.2f}  epi t_full {med[4]:.2f}  (n={len(w)})")
