"""Independent float64 PyTorch reference of the SlimResNet forward (test-only).

Written from SURVEY.md §8(c) O2-O8 with library routines only
(torch.nn.functional.conv2d / batch_norm / relu / avg_pool2d / linear, NCHW),
explicitly TRUNCATING the shared weights to the active prefix before calling the
library.  It shares no code with oracle/ and is used to pin the oracle
("special cases that reduce to a library routine").
"""
from __future__ import annotations

import torch
import torch.nn.functional as F

from synth import active_channels


def _w(weights, name, c_out, c_in):
    w = torch.from_numpy(weights[name]).double()          # KRSC
    return w[:c_out, :, :, :c_in].permute(0, 3, 1, 2).contiguous()   # -> [Cout, Cin, kh, kw]


def _bn(y, st, eps):
    c = y.shape[1]
    t = lambda a: torch.as_tensor(a[:c]).double()
    return F.batch_norm(y, t(st["mean"]), t(st["var"]), t(st["gamma"]), t(st["beta"]),
                        training=False, eps=eps)


def _bn_batch(y, st, eps):
    """Training-mode BN: normalises with this batch's per-channel statistics (biased variance)
    -- the library's statement of what O10's calibrated statistics must reproduce."""
    c = y.shape[1]
    t = lambda a: torch.as_tensor(a[:c]).double()
    return F.batch_norm(y, None, None, t(st["gamma"]), t(st["beta"]), training=True, eps=eps)


def _gn(y, st, eps, group_channels=16):
    c = y.shape[1]
    t = lambda a: torch.as_tensor(a[:c]).double()
    return F.group_norm(y, c // group_channels, t(st["gamma"]), t(st["beta"]), eps=eps)


def segment(weights, bn, widths, s, x_nchw, r_prev, r, base=(64, 128, 256, 512), blocks=(2, 2, 2, 2),
            eps=1e-5, head=True, norm="bn"):
    wi = [abs(q - r) < 1e-6 for q in widths].index(True)
    _bn = {"gn": _gn, "bn_batch": _bn_batch}.get(norm, globals()["_bn"])
    C = active_channels(r, base[s])
    h = x_nchw
    if s == 0:
        h = F.relu(_bn(F.conv2d(h, _w(weights, "stem", C, h.shape[1]), stride=1, padding=1), bn["stem"][wi], eps))
    for b in range(blocks[s]):
        down = s > 0 and b == 0
        st = 2 if down else 1
        cin = h.shape[1]
        t = F.relu(_bn(F.conv2d(h, _w(weights, f"s{s}b{b}c1", C, cin), stride=st, padding=1),
                       bn[f"s{s}b{b}c1"][wi], eps))
        u = _bn(F.conv2d(t, _w(weights, f"s{s}b{b}c2", C, C), stride=1, padding=1), bn[f"s{s}b{b}c2"][wi], eps)
        if down:
            sc = _bn(F.conv2d(h, _w(weights, f"s{s}b{b}sc", C, cin), stride=2, padding=0),
                     bn[f"s{s}b{b}sc"][wi], eps)
        else:
            sc = h
        h = F.relu(u + sc)
    if s == 3 and head:
        p = F.avg_pool2d(h, kernel_size=h.shape[-1]).flatten(1)
        fw = torch.from_numpy(weights["fc_w"]).double()[:, :C]
        fb = torch.from_numpy(weights["fc_b"]).double()
        return F.linear(p, fw, fb)
    return h


def chain(weights, bn, widths, x_nhwc, r_per_seg, **kw):
    h = torch.from_numpy(x_nhwc).double().permute(0, 3, 1, 2).contiguous()
    h = segment(weights, bn, widths, 0, h, None, r_per_seg[0], **kw)
    for s in range(1, 4):
        h = segment(weights, bn, widths, s, h, r_per_seg[s - 1], r_per_seg[s], **kw)
    return h.numpy()


def to_nhwc(t):
    return t.permute(0, 2, 3, 1).contiguous().numpy()
