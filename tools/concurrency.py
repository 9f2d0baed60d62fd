"""Sequential vs concurrent (one stream per width instance) execution of the CFG2 step."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2510_09018_b200 as slim  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
W = (0.25, 0.5, 0.75, 1.0)
net = slim.SlimNet(synth.make_weights(), synth.make_bn(), max_batch=B)
slim.slim_set_graph_mode(net.ctx, True)
xs = {r: torch.from_numpy(synth.make_images(B, offset=i)).to(torch.bfloat16).cuda() for i, r in enumerate(W)}
lg = {r: torch.empty(B, 100, device="cuda") for r in W}
wsb = max(slim.slim_chain_workspace_bytes(net.ctx, (r,) * 4, B) for r in W)
ws = {r: torch.empty(wsb, dtype=torch.uint8, device="cuda") for r in W}
streams = {r: torch.cuda.Stream() for r in W}
main = torch.cuda.current_stream()


def seq():
    for r in W:
        slim.slim_forward_chain(net.ctx, (r,) * 4, B, xs[r], lg[r], ws[r], wsb, main)


def conc():
    ev = torch.cuda.Event()
    ev.record(main)
    for r in W:
        streams[r].wait_event(ev)
        slim.slim_forward_chain(net.ctx, (r,) * 4, B, xs[r], lg[r], ws[r], wsb, streams[r])
    for r in W:
        main.wait_stream(streams[r])


def t(fn, n=200):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(main)
    for _ in range(n):
        fn()
    b.record(main)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


ts, tc = t(seq), t(conc)
print(f"B={B}: sequential {ts:.1f} us/step ({4 * B / ts * 1e6:,.0f} img/s), concurrent {tc:.1f} us/step "
      f"({4 * B / tc * 1e6:,.0f} img/s)")
