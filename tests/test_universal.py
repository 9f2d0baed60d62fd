"""Universal widths ("universally slimmable") on CPU:
the oracle at widths whose channel counts are not multiples of 16 against torch float64 on
explicitly truncated weights, the kernel channel-padding rule, and config validation."""
import ctypes

import numpy as np
import pytest

import oracle
import synth
import paper_2510_09018_b200 as slim
from tests import torch_ref

UW = (0.25, 0.3, 0.5, 0.6, 0.75, 0.9, 1.0)


def test_act_channels_rule():
    for C in (64, 128, 256, 512):
        for r in np.linspace(0.05, 1.0, 40):
            c = slim.slim_channels(float(r), C)
            ca = slim.slim_act_channels(float(r), C)
            assert c == int(np.ceil(np.float32(r) * np.float64(C) - 1e-9))
            assert c <= ca <= C and ca % 16 == 0 and (ca <= 128 or ca % 64 == 0)
            assert ca - c < (16 if ca <= 128 else 64)
    for C in (64, 128, 256, 512):   # the paper's set: no padding
        for r in synth.WIDTHS:
            assert slim.slim_act_channels(r, C) == slim.slim_channels(r, C)
    assert [slim.slim_channels(r, 64) for r in (0.3, 0.6, 0.9)] == [20, 39, 58]
    assert [slim.slim_act_channels(r, 64) for r in (0.3, 0.6, 0.9)] == [32, 48, 64]
    assert slim.slim_act_channels(0.9, 512) == 512 and slim.slim_act_channels(0.3, 512) == 192


def test_universal_config_is_accepted_before_the_device():
    lib = slim.load_library()
    h = ctypes.c_void_p()
    cfg = slim.default_config(widths=UW)
    # validation passes; without a GPU the call then fails on the device (not EUNSUPPORTED)
    import torch
    if not torch.cuda.is_available():
        assert lib.slim_create(0, ctypes.byref(cfg), ctypes.byref(h)) == slim.SLIM_ECUDA
    gn = slim.default_config(widths=UW, norm="gn")   # 20 channels hold no whole 16-channel groups
    assert lib.slim_create(0, ctypes.byref(gn), ctypes.byref(h)) == slim.SLIM_EUNSUPPORTED


@pytest.mark.parametrize("tup", [(0.3, 0.6, 0.9, 0.3), (0.9, 0.25, 0.6, 1.0)])
def test_oracle_universal_chain_matches_torch(tup):
    weights, bn = synth.make_weights(), synth.make_bn(widths=UW)
    x = synth.make_images(2, offset=17)
    got = oracle.Model(weights, bn, widths=UW).chain(x, tup)
    ref = torch_ref.chain(weights, bn, UW, x, tup)
    np.testing.assert_allclose(got, ref, rtol=1e-9, atol=1e-9)
