"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

Runs every kernel family at CFG1-like sizes through the C-ABI: the stem, the halo / per-tap /
split-K conv kernels (whichever the env switches select), the fused pool, FC, gather/scatter,
GroupNorm and the FP32 SIMT path.  Parity is checked elsewhere (tests/); this only drives the
kernels so the sanitizer sees every launch.  Usage (one env variant per process, the switches
are read once per process):

    SLIM_SPLITK_FORCE=1 compute-sanitizer --tool memcheck python tools/sanitize_workload.py [bn|gn|fp32]
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2510_09018_b200 as slim  # noqa: E402


def main(mode: str = "bn"):
    w, bn = synth.make_weights(), synth.make_bn()
    kw = dict(max_batch=16)
    if mode == "gn":
        kw["norm"] = "gn"
    if mode == "fp32":
        kw["dtype"] = "fp32"
    net = slim.SlimNet(w, bn, **kw)
    adt = net.act_dtype
    x = torch.from_numpy(synth.make_images(9, offset=5)).to(adt).cuda()
    for tup in ((0.25, 0.25, 0.25, 0.25), (1.0, 1.0, 1.0, 1.0), (0.25, 0.75, 0.5, 1.0)):
        net.forward_chain(x, tup)
    # single segments incl. CFG1 (seg 0, r=0.25, B=8)
    net.forward(0, x[:8].contiguous(), 0.25, 0.25)
    h = net.forward(0, x, 0.5, 0.5)
    h = net.forward(1, h, 0.5, 1.0)
    # packer + gather + launch + scatter
    if mode == "bn":
        reqs = [(i, 0, 0.25, 0.25, i) for i in range(5)]
        descs, order = slim.slim_pack(net.cfg, reqs, 16)
        ws_b = slim.slim_forward_workspace_bytes(net.ctx, 0, 0.25, 0.25, 5)
        ws = torch.empty(max(ws_b, 1), dtype=torch.uint8, device="cuda")
        slab = torch.empty(5, 32, 32, 3, dtype=adt, device="cuda")
        out = torch.empty(5, 32, 32, 16, dtype=adt, device="cuda")
        idx = torch.from_numpy(order[:5].astype(np.int32)).cuda()
        slim.slim_launch(net.ctx, descs[0], idx, x, 32 * 32 * 3 * 2, slab, out, ws, ws_b)
        dst = torch.zeros(9, 32, 32, 16, dtype=adt, device="cuda")
        slim.slim_scatter(net.ctx, out, idx, 5, 32 * 32 * 16 * 2, dst, 32 * 32 * 16 * 2)
    # graph replay path
    slim.slim_set_graph_mode(net.ctx, True)
    net.forward_chain(x, (0.5, 0.25, 1.0, 0.75))
    net.forward_chain(x, (0.5, 0.25, 1.0, 0.75))
    torch.cuda.synchronize()
    st = slim.slim_last_error(net.ctx)
    net.close()
    print(f"sanitize workload {mode} done, status {st}")
    assert st == 0


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "bn")
