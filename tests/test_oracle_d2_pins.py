"""Pins of the oracle pieces behind the D2 argmax check (reading #13)
and of the parity checker itself (VERDICT r01 next #1c), run with -m "not gpu".

* per_image_rel_err   -- a hand-computed two-image case that a max over the batch axis or a
                         batch-wide denominator gets wrong
* fast conv == plain  -- the vectorised oracle conv is bitwise the one-output-at-a-time loop nest
                         and bitwise the pure-Python brute force (zero-padding identity)
* O10 calibrate_bn    -- inference with the calibrated statistics == torch float64 training-mode
                         BN (batch statistics) on the calibration set (library routine)
* NCM head            -- closed form: prototype k scores 4||f_k - m|| on class k and is top-1
* fixture             -- tests/golden/d2_model.npz regenerates (tuple 0) bit for bit
"""
import os
import sys

import numpy as np
import pytest
import torch

import oracle
import synth
from tests import torch_ref
from tests.test_oracle_pins import _brute_conv

W4 = synth.WIDTHS


def test_per_image_rel_err_hand_computed():
    """Image 0: ref (1, -4), got (1.5, -4) -> 0.5/4 = 0.125.  Image 1: ref (100, 0), got (100, 1)
    -> 1/100 = 0.01.  Reducing over the batch axis instead gives per-logit values (0.5/100, 1/4)
    and a batch-wide denominator max|ref| = 100 gives (0.005, 0.01): both fail the asserts."""
    ref = np.array([[1.0, -4.0], [100.0, 0.0]])
    got = np.array([[1.5, -4.0], [100.0, 1.0]])
    err = oracle.per_image_rel_err(got, ref)
    assert err.shape == (2,)
    assert err[0] == 0.125 and err[1] == 0.01
    # a 4-d segment output: per image over ALL of its H*W*C elements
    r4 = np.zeros((2, 2, 2, 3)); r4[0, 1, 0, 2] = -8.0; r4[1, 0, 1, 1] = 2.0
    g4 = r4.copy(); g4[0, 0, 0, 0] = 1.0; g4[1, 1, 1, 2] = -0.5
    assert list(oracle.per_image_rel_err(g4, r4)) == [1.0 / 8.0, 0.5 / 2.0]


@pytest.mark.parametrize("B,H,ci,co,k,s,p,cif,cof", [
    (3, 8, 5, 7, 3, 1, 1, 9, 9), (2, 9, 16, 32, 3, 2, 1, 16, 40), (2, 8, 13, 11, 1, 2, 0, 20, 20),
    (2, 8, 32, 48, 3, 1, 1, 64, 64), (2, 7, 3, 16, 3, 1, 1, 3, 16), (2, 16, 64, 128, 3, 2, 1, 64, 128),
    (2, 8, 32, 32, 1, 2, 0, 32, 32), (1, 5, 16, 16, 3, 2, 1, 16, 16), (1, 4, 512, 512, 3, 1, 1, 512, 512)])
def test_fast_conv_is_bitwise_plain(B, H, ci, co, k, s, p, cif, cof):
    g = np.random.default_rng(B * 1000 + H * 10 + k)
    x = g.standard_normal((B, H, H, ci))
    w = g.standard_normal((cof, k, k, cif))
    w[co:] = np.nan                      # never read
    w[..., ci:] = np.nan
    a = oracle.conv2d(x, w, co, s, p)
    b = oracle.conv2d(x, w, co, s, p, plain=True)
    assert np.isfinite(a).all() and np.array_equal(a, b)


@pytest.mark.parametrize("k,s,p,H,co", [(3, 1, 1, 5, 16), (3, 2, 1, 8, 16), (1, 2, 0, 8, 16), (3, 1, 1, 4, 2)])
def test_fast_conv_is_bitwise_brute_force(k, s, p, H, co):
    """Same summation order as the pure-Python brute force (kh, kw, ci; padding terms omitted
    there, added as exact zeros in the fast path): bitwise equal."""
    g = np.random.default_rng(5)
    x = g.standard_normal((1, H, H, 3))
    w = g.standard_normal((co, k, k, 3))
    assert np.array_equal(oracle.conv2d(x, w, co, s, p), _brute_conv(x, w, co, s, p))


@pytest.mark.parametrize("tup", [(0.25, 0.25, 0.25, 0.25), (0.5, 0.25, 0.25, 0.5)])
def test_calibrate_bn_matches_torch_training_mode(tup):
    """O10: with the calibrated statistics, inference-mode BN on the calibration set is the
    library's training-mode BN (batch statistics, biased variance) on that set, layer after layer."""
    weights, bn = synth.make_weights(), synth.make_bn()
    x, _, _ = synth.make_prototype_images(24, sigma=0.1, offset=5)
    m = oracle.Model(weights, bn)
    bn_t = m.calibrate_bn(x, tup)
    got = oracle.Model(weights, bn_t).chain(x, tup)
    ref = torch_ref.chain(weights, bn, W4, x, tup, norm="bn_batch")
    # calibrated statistics are stored in float32: ~1e-7 relative per BN
    np.testing.assert_allclose(got, ref, rtol=2e-5, atol=2e-5 * np.abs(ref).max())
    # the statistics of widths the tuple does not use, and self.bn, are untouched
    for name, per_w in bn.items():
        for wi in range(4):
            s_ = int(name[1]) if name != "stem" else 0
            if W4[wi] != tup[s_]:
                assert bn_t[name][wi]["mean"] is per_w[wi]["mean"]
    assert m.bn is bn


def test_ncm_head_closed_form():
    """W[k] = 4 u_k, u_k = (f_k - m)/||f_k - m||, b = -m W^T: prototype k's logits are 4 (f_k - m).u_j,
    so class k scores 4||f_k - m|| (Cauchy-Schwarz maximum) and is top-1; W is zero past c3."""
    g = np.random.default_rng(9)
    f = g.standard_normal((100, 48)) + 3.0
    W, b = oracle.ncm_head(f, 100, 64)
    assert W.shape == (100, 64) and b.shape == (100,)
    assert (W[:, 48:] == 0).all()
    logits = f @ W[:, :48].astype(np.float64).T + b
    m = f.mean(axis=0)
    assert (logits.argmax(axis=1) == np.arange(100)).all()
    np.testing.assert_allclose(np.diag(logits), 4 * np.linalg.norm(f - m, axis=1), rtol=2e-2)
    np.testing.assert_allclose(np.linalg.norm(W, axis=1), 4.0, rtol=1e-2)
    assert np.array_equal(synth.round_bf16(W), W) and np.array_equal(synth.round_bf16(b), b)


def test_d2_fixture_regenerates_tuple0():
    """tests/golden/d2_model.npz was written by make_d2_fixture.py from oracle/ only: tuple 0 rebuilt
    here matches bit for bit, and the stored head classifies the clean prototypes correctly."""
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    import make_d2_fixture as mk
    from tests import d2_fixture
    weights, bn = synth.make_weights(), synth.make_bn()
    x_cal, _, protos = synth.make_prototype_images(mk.N_CAL, sigma=mk.SIGMA, offset=0)
    fresh = mk.build_tuple(0, weights, bn, x_cal, protos)
    stored = d2_fixture._npz()
    for k, v in fresh.items():
        assert np.array_equal(stored[k], v), k
    w_t, bn_t = d2_fixture.model(0)
    logits = oracle.Model(w_t, bn_t).chain(protos, synth.TABLE_TUPLES[0])
    assert (logits.argmax(axis=1) == np.arange(100)).all()
