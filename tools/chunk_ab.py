"""A/B of the chain chunking at large batches: images/s of forward_chain (graph replay, L2 flushed
before each replay) for B in (2048, 4096) and each width; run with SLIM_CHAIN_CHUNK=0 for 'off'."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2510_09018_b200 as slim  # noqa: E402

net = slim.SlimNet(synth.make_weights(), synth.make_bn(), max_batch=4096)
slim.slim_set_graph_mode(net.ctx, True)
x = torch.from_numpy(synth.make_images(4096)).to(torch.bfloat16).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
tag = os.environ.get("SLIM_CHAIN_CHUNK", "default")
for B in (2048, 4096):
    for r in (0.25, 0.5, 0.75, 1.0):
        xb = x[:B]
        for _ in range(3):
            net.forward_chain(xb, (r,) * 4)
        tot = 0.0
        for _ in range(30):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            net.forward_chain(xb, (r,) * 4)
            b.record()
            torch.cuda.synchronize()
            tot += a.elapsed_time(b)
        print(f"chunk={tag} B={B} r={r}: {B * 30 / (tot / 1e3):,.0f} images/s")
