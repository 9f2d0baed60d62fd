"""Throughput of each segment (and of trivial kernels) with warm clocks: N back-to-back
calls bracketed by one CUDA-event pair, so per-call time excludes event overheads.

    python tools/micro.py [B] [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2510_09018_b200 as slim  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
N = int(sys.argv[2]) if len(sys.argv) > 2 else 200
graph = os.environ.get("GRAPH", "1") == "1"
net = slim.SlimNet(synth.make_weights(), synth.make_bn(), max_batch=B, norm=sys.argv[3] if len(sys.argv) > 3 else "bn")
slim.slim_set_graph_mode(net.ctx, graph)
x = torch.from_numpy(synth.make_images(B)).to(torch.bfloat16).cuda()
st = torch.cuda.current_stream()


def timeit(fn, n=N):
    for _ in range(10):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3   # us


# warm the clocks
buf = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
for _ in range(50):
    buf.add_(1)
t = torch.zeros(1, device="cuda")
print(f"empty-ish torch kernel: {timeit(lambda: t.add_(1)):.2f} us")
for r in (0.25, 0.5, 0.75, 1.0):
    ins = {0: x}
    outs = {}
    h = x
    line = []
    for s in range(4):
        shp = net.segment_out_shape(s, r, B)
        o = torch.empty(shp, dtype=torch.float32 if s == 3 else torch.bfloat16, device="cuda")
        wsb = slim.slim_forward_workspace_bytes(net.ctx, s, r, r, B)
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        hin = h
        us = timeit(lambda: slim.slim_forward_ws(net.ctx, s, r, r, B, hin, o, ws, wsb, st))
        line.append(f"seg{s}:{us:6.1f}")
        h = o
    logits = torch.empty(B, 100, device="cuda")
    wsb = slim.slim_chain_workspace_bytes(net.ctx, (r,) * 4, B)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    us = timeit(lambda: slim.slim_forward_chain(net.ctx, (r,) * 4, B, x, logits, ws, wsb, st))
    print(f"r={r}: " + " ".join(line) + f"  chain:{us:6.1f} us  -> {B / us * 1e6:,.0f} img/s")
