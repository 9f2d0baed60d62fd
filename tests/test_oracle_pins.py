"""Pins of the CPU oracle against things other than itself (run with -m "not gpu").

Each test names what it pins and why a plausible oracle bug (dropped term,
wrong sign/index, transposed operand, wrong BN set, wrong slice) fails it:

* brute force   -- literal nested loops in pure Python on tiny tensors (O2, O7)
* library       -- torch.nn.functional float64 on explicitly truncated weights (O2-O8)
* closed form   -- centre-tap delta kernels + unit BN: seg0 = 4*relu(x), each later
                   segment = 4*h[::2, ::2] (SURVEY §8(c) "Closed form")
* invariants    -- slicing == truncation, NaN prefix isolation, BN-width selection
                   (with a negative control), batch independence.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from tests import torch_ref

W4 = synth.WIDTHS


@pytest.fixture(scope="module")
def net():
    return synth.make_weights(), synth.make_bn()


# ------------------------------------------------------------------ brute force
def _brute_conv(x, w, c_out, s, p):
    B, H, W, c_in = x.shape
    _, k, _, _ = w.shape
    Ho = (H + 2 * p - k) // s + 1
    Wo = (W + 2 * p - k) // s + 1
    y = [[[[0.0] * c_out for _ in range(Wo)] for _ in range(Ho)] for _ in range(B)]
    for n in range(B):
        for oh in range(Ho):
            for ow in range(Wo):
                for co in range(c_out):
                    acc = 0.0
                    for kh in range(k):
                        for kw in range(k):
                            ih, iw = s * oh + kh - p, s * ow + kw - p
                            if 0 <= ih < H and 0 <= iw < W:
                                for ci in range(c_in):
                                    acc += float(x[n, ih, iw, ci]) * float(w[co, kh, kw, ci])
                    y[n][oh][ow][co] = acc
    return np.array(y)


@pytest.mark.parametrize("k,s,p,H", [(3, 1, 1, 5), (3, 2, 1, 6), (3, 2, 1, 5), (1, 2, 0, 6), (1, 1, 0, 4)])
def test_conv_matches_brute_force(k, s, p, H):
    g = np.random.default_rng(7)
    x = g.standard_normal((2, H, H, 3))
    w = g.standard_normal((4, k, k, 5))          # full width Cin=5 > c_in=3, Cout=4 > c_out=2
    got = oracle.conv2d(x, w, c_out=2, stride=s, pad=p)
    ref = _brute_conv(x, w, 2, s, p)
    assert got.shape == ref.shape
    np.testing.assert_allclose(got, ref, rtol=1e-13, atol=1e-13)


def test_conv_asymmetric_taps_detect_transpose():
    """A kernel non-symmetric in (kh,kw) and a non-square-patterned input: a kh/kw swap fails."""
    x = np.arange(1 * 4 * 4 * 1, dtype=np.float64).reshape(1, 4, 4, 1)
    w = np.zeros((1, 3, 3, 1)); w[0, 0, 2, 0] = 1.0   # tap (kh=0, kw=2): y[oh,ow] = x[oh-1, ow+1]
    y = oracle.conv2d(x, w, 1, 1, 1)[0, :, :, 0]
    X = x[0, :, :, 0]
    for oh in range(4):
        for ow in range(4):
            exp = X[oh - 1, ow + 1] if (oh - 1 >= 0 and ow + 1 < 4) else 0.0
            assert y[oh, ow] == exp


def test_head_matches_brute_force(net):
    weights, bn = net
    m = oracle.Model(weights, bn)
    g = np.random.default_rng(3)
    h = g.standard_normal((2, 4, 4, 128))
    got = m.head(h, 0.25)
    for n in range(2):
        for k in range(100):
            acc = float(weights["fc_b"][k])
            for c in range(128):
                pc = sum(h[n, i, j, c] for i in range(4) for j in range(4)) / 16.0
                acc += pc * float(weights["fc_w"][k, c])
            assert math.isclose(got[n, k], acc, rel_tol=1e-12, abs_tol=1e-12)


def test_bn_matches_formula_by_hand():
    y = np.array([[[[2.0, -1.0]]]])
    st = dict(mean=np.array([1.0, 0.5]), var=np.array([3.0, 0.0]), gamma=np.array([2.0, -1.0]),
              beta=np.array([0.5, 0.25]))
    z = oracle.batchnorm(y, st, eps=1.0)
    assert z[0, 0, 0, 0] == pytest.approx((2 - 1) / 2.0 * 2 + 0.5)
    assert z[0, 0, 0, 1] == pytest.approx((-1 - 0.5) / 1.0 * -1 + 0.25)


# ------------------------------------------------------------------ library routine
@pytest.mark.parametrize("k,s,p", [(3, 1, 1), (3, 2, 1), (1, 2, 0)])
def test_conv_matches_torch_float64(k, s, p):
    g = np.random.default_rng(11)
    x = g.standard_normal((3, 10, 10, 24))
    w = g.standard_normal((40, k, k, 32))
    got = oracle.conv2d(x, w, c_out=16, stride=s, pad=p)
    ref = torch.nn.functional.conv2d(torch.from_numpy(x).permute(0, 3, 1, 2),
                                     torch.from_numpy(w[:16, :, :, :24]).permute(0, 3, 1, 2),
                                     stride=s, padding=p).permute(0, 2, 3, 1).numpy()
    np.testing.assert_allclose(got, ref, rtol=1e-11, atol=1e-11)


@pytest.mark.parametrize("tup", [(1.0, 1.0, 1.0, 1.0), (0.25, 0.25, 0.25, 0.25), (1.0, 0.75, 0.5, 0.25),
                                 (0.5, 0.25, 1.0, 0.75)])
def test_chain_matches_torch_float64(net, tup):
    """r=1 equals the unsliced network; any tuple equals the library net on truncated weights."""
    weights, bn = net
    x = synth.make_images(2)
    got = oracle.Model(weights, bn).chain(x, tup)
    ref = torch_ref.chain(weights, bn, W4, x, tup)
    np.testing.assert_allclose(got, ref, rtol=1e-9, atol=1e-9 * np.abs(ref).max())


def test_segment_outputs_match_torch(net):
    weights, bn = net
    m = oracle.Model(weights, bn)
    x = synth.make_images(2, offset=1)
    h = m.segment(0, x, None, 0.5)
    ref = torch_ref.to_nhwc(torch_ref.segment(weights, bn, W4, 0,
                                              torch.from_numpy(x).double().permute(0, 3, 1, 2), None, 0.5))
    np.testing.assert_allclose(h, ref, rtol=1e-10, atol=1e-10)
    h2 = m.segment(1, h, 0.5, 0.75)
    ref2 = torch_ref.to_nhwc(torch_ref.segment(weights, bn, W4, 1, torch.from_numpy(h).permute(0, 3, 1, 2),
                                               0.5, 0.75))
    np.testing.assert_allclose(h2, ref2, rtol=1e-10, atol=1e-10)


# ------------------------------------------------------------------ closed form
def _delta_net(base=(64, 128, 256, 512), var_fill=0.25 - 1e-5, var_dtype=np.float64):
    """var+eps == 0.25 to 1 ulp in fp64 (float32 stats would add a 1e-7 relative term per BN)."""
    weights, bn = {}, {}
    for sp in synth.layer_specs(base):
        w = np.zeros((sp["cout"], sp["k"], sp["k"], sp["cin"]), np.float32)
        c = sp["k"] // 2
        for i in range(min(sp["cout"], sp["cin"])):
            w[i, c, c, i] = 1.0
        weights[sp["name"]] = w
        bn[sp["name"]] = [dict(gamma=np.full(synth.active_channels(r, sp["cout"]), 0.5, np.float32),
                               beta=np.zeros(synth.active_channels(r, sp["cout"]), np.float32),
                               mean=np.zeros(synth.active_channels(r, sp["cout"]), np.float32),
                               var=np.full(synth.active_channels(r, sp["cout"]), var_fill, var_dtype))
                          for r in synth.WIDTHS]
    weights["fc_w"] = synth.make_weights()["fc_w"]
    weights["fc_b"] = np.zeros(100, np.float32)
    return weights, bn


@pytest.mark.parametrize("tup", [(0.25, 0.25, 0.25, 0.25), (1.0, 0.5, 0.75, 0.25)])
def test_closed_form_delta_network(tup):
    """Centre-tap delta kernels, BN scale 0.5/sqrt(0.25)=1: every block maps h>=0 to 2h.
    seg0 -> 4*relu(x) on channels<3, 0 elsewhere; seg s>0 -> 4*h[::2, ::2]; head pools exactly."""
    weights, bn = _delta_net()
    m = oracle.Model(weights, bn)
    x = synth.make_images(2, offset=2)
    rx = np.maximum(x.astype(np.float64), 0)
    h = m.segment(0, x, None, tup[0])
    exp = np.zeros(h.shape); exp[..., :3] = 4 * rx
    np.testing.assert_allclose(h, exp, rtol=1e-12, atol=1e-12)
    for s in range(1, 4):
        h = m.segment(s, h, tup[s - 1], tup[s], head=False)
        exp = np.zeros(h.shape); exp[..., :3] = 4 ** (s + 1) * rx[:, ::2 ** s, ::2 ** s, :]
        np.testing.assert_allclose(h, exp, rtol=1e-12, atol=1e-12)
    logits = m.head(h, tup[3])
    c3 = h.shape[-1]
    pooled = np.zeros((2, c3)); pooled[:, :3] = 256 * rx[:, ::8, ::8, :].mean(axis=(1, 2))
    np.testing.assert_allclose(logits, pooled @ weights["fc_w"][:, :c3].astype(np.float64).T,
                               rtol=1e-12, atol=1e-12)


# ------------------------------------------------------------------ invariants
@pytest.mark.parametrize("r", [0.25, 0.75])
def test_slicing_equals_truncation(net, r):
    """oracle(W, r) == oracle on explicitly truncated copies run as a full-width net (bitwise)."""
    weights, bn = net
    wi = W4.index(r)
    base = tuple(synth.active_channels(r, C) for C in synth.BASE_CHANNELS)
    tw, tb = {}, {}
    for sp in synth.layer_specs():
        co = synth.active_channels(r, sp["cout"])
        ci = sp["cin"] if sp["kind"] == "stem" else synth.active_channels(r, sp["cin"])
        tw[sp["name"]] = weights[sp["name"]][:co, :, :, :ci].copy()
        tb[sp["name"]] = [bn[sp["name"]][wi]]
    tw["fc_w"] = weights["fc_w"][:, :base[3]].copy()
    tw["fc_b"] = weights["fc_b"]
    x = synth.make_images(2, offset=3)
    a = oracle.Model(weights, bn).chain(x, (r,) * 4)
    b = oracle.Model(tw, tb, widths=(1.0,), base=base).chain(x, (1.0,) * 4)
    assert np.array_equal(a, b)


def test_nan_prefix_isolation(net):
    """Entries outside the active prefix are never read: NaN there changes nothing (bitwise)."""
    weights, bn = net
    r_prev, r = 0.5, 0.25
    poisoned = synth.nan_poison_weights(weights, r_prev, r)
    x = synth.make_images(2, offset=4)
    m = oracle.Model(weights, bn)
    h0 = m.segment(0, x, None, r_prev)
    a = m.segment(1, h0, r_prev, r)
    b = oracle.Model(poisoned, bn).segment(1, h0, r_prev, r)
    assert np.isfinite(b).all() and np.array_equal(a, b)


def test_bn_width_selection_with_negative_control(net):
    """Each switchable BN selects exactly its own width's statistics (north_star invariant)."""
    weights, bn = net
    m = oracle.Model(weights, bn)
    x = synth.make_images(2, offset=5)
    a = m.segment(0, x, None, 0.25)
    ref = torch_ref.to_nhwc(torch_ref.segment(weights, bn, W4, 0,
                                              torch.from_numpy(x).double().permute(0, 3, 1, 2), None, 0.25))
    np.testing.assert_allclose(a, ref, rtol=1e-10, atol=1e-10)
    # negative control: the 0.5-width statistics on the same 16-channel prefix differ by >> tolerance
    bad = m.segment(0, x, None, 0.25, bn_width=0.5)
    assert oracle.per_image_rel_err(bad, a).min() > 0.05


def test_batch_independence(net):
    weights, bn = net
    m = oracle.Model(weights, bn)
    x = synth.make_images(3, offset=6)
    full = m.chain(x, (0.5, 0.25, 0.25, 0.5))
    for i in range(3):
        one = m.chain(x[i:i + 1], (0.5, 0.25, 0.25, 0.5))
        assert np.array_equal(one[0], full[i])


def test_width_channels_rule():
    assert [oracle.channels(r, 64) for r in W4] == [16, 32, 48, 64]
    assert [oracle.channels(r, 512) for r in W4] == [128, 256, 384, 512]
    assert oracle.channels(0.3, 64) == 20          # ceil(19.2)


def test_empty_batch():
    y = oracle.conv2d(np.zeros((0, 8, 8, 16)), np.zeros((16, 3, 3, 16)), 16, 1, 1)
    assert y.shape == (0, 8, 8, 16)
