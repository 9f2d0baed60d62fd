"""CFG2 step (4 widths x B=128) with each width's batch split over S instances (own stream each,
Alg. 1 scale-up instances of the same key), SM shares per width scaled by `scale`.  Prints
images/s of the device-timed concurrent step (graph replay, L2 flushed before every step).

    python tools/split_instances.py S scale
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2510_09018_b200 as slim  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 2
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
B, W, K = 128, (0.25, 0.5, 0.75, 1.0), 300
b = B // S
net = slim.SlimNet(synth.make_weights(), synth.make_bn(), max_batch=B)
for r in W:
    slim.slim_set_sm_share(net.ctx, r, min(1.0, (0.1 + 0.45 * r) * scale))
slim.slim_set_graph_mode(net.ctx, True)
inst = [(r, j) for r in W for j in range(S)]
xs = {k: torch.from_numpy(synth.make_images(b, offset=i)).to(torch.bfloat16).cuda() for i, k in enumerate(inst)}
lg = {k: torch.empty(b, 100, device="cuda") for k in inst}
wsb = max(slim.slim_chain_workspace_bytes(net.ctx, (r,) * 4, b) for r in W)
ws = {k: torch.empty(wsb, dtype=torch.uint8, device="cuda") for k in inst}
st = {k: torch.cuda.Stream() for k in inst}
main = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def step():
    ev = torch.cuda.Event()
    ev.record(main)
    for k in inst:
        st[k].wait_event(ev)
        slim.slim_forward_chain(net.ctx, (k[0],) * 4, b, xs[k], lg[k], ws[k], wsb, st[k])
    for k in inst:
        main.wait_stream(st[k])


for _ in range(10):
    step()
torch.cuda.synchronize()
tot = 0.0
for _ in range(K):
    flush.zero_()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(main)
    step()
    e.record(main)
    torch.cuda.synchronize()
    tot += a.elapsed_time(e)
print(f"S={S} scale={scale}: {len(W) * B * K / (tot / 1e3):,.0f} images/s ({tot / K * 1e3:.1f} us/step)")
