"""Pins of the oracle's GroupNorm variant ("Group Normalization instead of Batch
Normalization"; reading R16: 16 channels per group).

* brute force -- literal loops over (n, g) on a tiny tensor (catches a wrong reduction
                 axis, unbiased variance, a dropped eps, gamma/beta on the wrong index)
* library     -- torch.nn.functional.group_norm float64 (NCHW), per layer and for
                 whole GN segments / chains on explicitly truncated weights
* invariants  -- per-(image, group) affine invariance, output moments, group-aligned
                 slicing, batch independence (GN has no cross-image term)
"""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
import synth
from tests import torch_ref

W4 = synth.WIDTHS


def _params(c, g):
    return {"gamma": g.uniform(0.5, 1.5, c), "beta": g.uniform(-0.1, 0.1, c)}


def test_groupnorm_brute_force():
    g = np.random.default_rng(3)
    y = g.standard_normal((2, 3, 3, 32)) * 2.0 + 0.7
    p = _params(48, g)                               # longer than c: only the prefix is read
    got = oracle.groupnorm(y, p, 16, 1e-5)
    B, H, W, C = y.shape
    ref = np.zeros_like(y)
    for n in range(B):
        for grp in range(C // 16):
            vals = [float(y[n, h, w, c]) for h in range(H) for w in range(W) for c in range(16 * grp, 16 * grp + 16)]
            mu = sum(vals) / len(vals)
            var = sum((v - mu) ** 2 for v in vals) / len(vals)
            for h in range(H):
                for w in range(W):
                    for c in range(16 * grp, 16 * grp + 16):
                        ref[n, h, w, c] = (y[n, h, w, c] - mu) / math.sqrt(var + 1e-5) * p["gamma"][c] + p["beta"][c]
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("C", [16, 48, 64, 384])
def test_groupnorm_matches_torch(C):
    g = np.random.default_rng(C)
    y = g.standard_normal((3, 4, 4, C)) * 3.0 - 1.0
    p = _params(C, g)
    got = oracle.groupnorm(y, p)
    ref = F.group_norm(torch.from_numpy(y).permute(0, 3, 1, 2), C // 16, torch.from_numpy(p["gamma"]),
                       torch.from_numpy(p["beta"]), eps=1e-5).permute(0, 2, 3, 1).numpy()
    np.testing.assert_allclose(got, ref, rtol=1e-10, atol=1e-10)


def test_groupnorm_invariants():
    g = np.random.default_rng(11)
    y = g.standard_normal((2, 8, 8, 64))
    ones = {"gamma": np.ones(64), "beta": np.zeros(64)}
    z = oracle.groupnorm(y, ones, 16, 0.0)
    zg = z.reshape(2, 8, 8, 4, 16)
    np.testing.assert_allclose(zg.mean(axis=(1, 2, 4)), 0.0, atol=1e-12)          # zero mean per (n, g)
    np.testing.assert_allclose((zg ** 2).mean(axis=(1, 2, 4)), 1.0, rtol=1e-12)   # unit variance per (n, g)
    # per-(image, group) affine y -> a*y + b (a > 0) leaves GN unchanged (eps = 0)
    a = g.uniform(0.5, 3.0, (2, 1, 1, 4, 1))
    b = g.standard_normal((2, 1, 1, 4, 1))
    y2 = (y.reshape(2, 8, 8, 4, 16) * a + b).reshape(y.shape)
    np.testing.assert_allclose(oracle.groupnorm(y2, ones, 16, 0.0), z, atol=1e-11)
    # a group sees only its own channels: the first groups of a wider tensor normalise alike
    np.testing.assert_allclose(oracle.groupnorm(y, ones, 16)[..., :32], oracle.groupnorm(y[..., :32], ones, 16),
                               atol=1e-14)
    # no cross-image term: image 1 alone == image 1 in the batch
    np.testing.assert_allclose(oracle.groupnorm(y[1:], ones, 16), oracle.groupnorm(y, ones, 16)[1:], atol=0)
    with pytest.raises(AssertionError):
        oracle.groupnorm(y[..., :24], ones, 16)   # 24 channels do not hold whole 16-channel groups


@pytest.fixture(scope="module")
def net():
    return synth.make_weights(), synth.make_bn()


@pytest.mark.parametrize("s,r_prev,r", [(0, None, 0.25), (0, None, 1.0), (1, 1.0, 0.5), (2, 0.25, 0.75), (3, 0.5, 1.0)])
def test_gn_segment_matches_torch(net, s, r_prev, r):
    weights, bn = net
    g = np.random.default_rng(5)
    H = 32 >> max(s - 1, 0) if s else 32
    c_in = 3 if s == 0 else synth.active_channels(r_prev, synth.BASE_CHANNELS[s - 1])
    x = g.standard_normal((2, H, H, c_in))
    if s:
        x = np.maximum(x, 0)
    m = oracle.Model(weights, bn, norm="gn")
    got = m.segment(s, x, r_prev, r)
    ref = torch_ref.segment(weights, bn, W4, s, torch.from_numpy(x).permute(0, 3, 1, 2).contiguous(), r_prev, r,
                            norm="gn")
    ref = ref.numpy() if s == 3 else torch_ref.to_nhwc(ref)
    np.testing.assert_allclose(got, ref, rtol=1e-9, atol=1e-9)


@pytest.mark.parametrize("tup", [(1.0, 0.75, 0.5, 0.25), (0.25, 0.25, 0.25, 0.25)])
def test_gn_chain_matches_torch(net, tup):
    weights, bn = net
    x = synth.make_images(2, offset=3)
    got = oracle.Model(weights, bn, norm="gn").chain(x, tup)
    ref = torch_ref.chain(weights, bn, W4, x, tup, norm="gn")
    np.testing.assert_allclose(got, ref, rtol=1e-9, atol=1e-9)
    # GN is not BN: the two variants differ on the same weights (negative control)
    assert np.abs(got - oracle.Model(weights, bn).chain(x, tup)).max() > 1e-3
