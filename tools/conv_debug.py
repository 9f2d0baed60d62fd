"""Per-launch event timings of one chain (profiling mode) -- used with SLIM_CONV_DEBUG to isolate
TMA vs MMA vs epilogue costs of the conv kernel.  Diagnostic only (results are garbage in debug modes)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2510_09018_b200 as slim  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
r = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
net = slim.SlimNet(synth.make_weights(), synth.make_bn(), max_batch=B)
x = torch.from_numpy(synth.make_images(B)).to(torch.bfloat16).cuda()
for _ in range(3):
    net.forward_chain(x, (r,) * 4)
slim.slim_profile_begin(net.ctx, 400)
for _ in range(5):
    net.forward_chain(x, (r,) * 4)
recs = slim.slim_profile_end(net.ctx)
n = 18
avg = [sum(recs[i + k * n]["ms"] for k in range(5)) / 5 for i in range(n)]
print(os.environ.get("SLIM_CONV_DEBUG", "0"), " ".join(f"{recs[i]['kind'][:4]}{recs[i]['seg']}:{avg[i]*1e3:.1f}" for i in range(n)),
      f"| total {sum(avg)*1e3:.1f} us")
