"""Host cost of the eager enqueue path (no graphs): microseconds of host time per slim_forward_ws
call per segment / width at a small batch (GPU work stays short, so the launch queue never fills),
and per slim_stream_run call.  Usage: python tools/host_overhead.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
import paper_2510_09018_b200 as slim
from paper_2510_09018_b200.stream import NativeStreamExecutor
from paper_2510_09018_b200.router import TABLE_TUPLES

net = slim.SlimNet(synth.make_weights(), synth.make_bn(), max_batch=256)
slim.slim_set_graph_mode(net.ctx, False)
cfg = net.cfg
B = 8
wsb = max(slim.slim_forward_workspace_bytes(net.ctx, s, 1.0, 1.0, 256) for s in range(4))
ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
buf_in = torch.zeros(256 * 32 * 32 * 64, dtype=torch.bfloat16, device="cuda")
buf_out = torch.zeros(256 * 32 * 32 * 64, dtype=torch.bfloat16, device="cuda")
lib = slim.load_library()
st = torch.cuda.current_stream().cuda_stream
for s in range(4):
    for r in (0.25, 1.0):
        for b in (B, 128):
            ts = []
            l0 = slim.slim_launch_count(net.ctx)
            for it in range(60):
                t0 = time.perf_counter()
                rc = lib.slim_forward_ws(net.ctx, s, r, r, b, buf_in.data_ptr(), buf_out.data_ptr(), ws.data_ptr(), wsb, st)
                ts.append(time.perf_counter() - t0)
                assert rc == 0, rc
                if it % 5 == 4:
                    torch.cuda.synchronize()
            n_l = (slim.slim_launch_count(net.ctx) - l0) / 60
            print(f"seg{s} r={r} B={b}: host {1e6 * np.median(ts[10:]):.1f} us/call, {n_l:.0f} launches/call")
rng = np.random.default_rng(0)
for lanes in (1, 8):
    nx = NativeStreamExecutor(net, n_max=1024, B_max=256, lanes=lanes)
    x = torch.from_numpy(synth.make_images(1024, offset=3)).to(torch.bfloat16).cuda()
    for k in range(12):
        tup = np.asarray(TABLE_TUPLES, np.float32)[rng.integers(0, len(TABLE_TUPLES), 1024)]
        nx.run(x, tup)
        torch.cuda.synchronize()   # host time alone: no GPU back-pressure
    print(f"slim_stream_run lanes={lanes}: host {1e6 * np.median(nx.host_s[2:]):.0f} us/call "
          f"(pack {1e6 * np.median(nx.pack_s[2:]):.0f} us), {nx.last_n_batches} batches, {nx.last_launches} launches")
    nx.close()
