"""Per-launch device times of the bench chain (slim_profile_*, CUDA events per launch, no PDL).

    python tools/layer_times.py [B] [reps] [bn|gn] [bf16|fp32]
"""
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_2510_09018_b200 as slim  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
norm = sys.argv[3] if len(sys.argv) > 3 else "bn"
dtype = sys.argv[4] if len(sys.argv) > 4 else "bf16"
net = slim.SlimNet(synth.make_weights(), synth.make_bn(), max_batch=B, norm=norm, dtype=dtype)
x = torch.from_numpy(synth.make_images(B)).to(torch.bfloat16 if dtype == "bf16" else torch.float32).cuda()
for r in (0.25, 0.5, 0.75, 1.0):
    for _ in range(5):
        net.forward_chain(x, (r,) * 4)
    torch.cuda.synchronize()
    slim.slim_profile_begin(net.ctx, reps * 40)
    for _ in range(reps):
        net.forward_chain(x, (r,) * 4)
    recs = slim.slim_profile_end(net.ctx)
    agg = defaultdict(lambda: [0.0, 0, 0.0, 0.0])
    order = []
    for rec in recs:
        k = (rec["seg"], rec["layer"], rec["kind"])
        if k not in agg:
            order.append(k)
        a = agg[k]
        a[0] += rec["ms"]
        a[1] += 1
        a[2] = rec["flops"]
        a[3] = rec["bytes"]
    tot = sum(agg[k][0] / agg[k][1] for k in order)
    print(f"r={r}: sum of launches {tot * 1e3:.1f} us")
    for k in order:
        ms, n, fl, by = agg[k]
        us = ms / n * 1e3
        print(f"  seg{k[0]} L{k[1]:2d} {k[2]:10s} {us:7.2f} us  {fl / us * 1e-6:7.1f} TFLOP/s  {by / us * 1e-3:7.1f} GB/s")
