"""GPU parity at universal widths: channel counts c = ceil(r*C) that
are not multiples of 16 run on kernels padded to c_act = slim_act_channels(r, C); the
padded channels must be exact zeros and the first c must match the fp64 oracle
(per image max|d| <= tau * max|oracle|, tau 2e-2 bf16 / 1e-4 FP32)."""
import numpy as np
import pytest
import torch

import oracle
import synth
import paper_2510_09018_b200 as slim

pytestmark = pytest.mark.gpu

UW = (0.25, 0.3, 0.5, 0.6, 0.75, 0.9, 1.0)
TAU_BF16, TAU_FP32 = 2e-2, 1e-4


@pytest.fixture(scope="module")
def params():
    return synth.make_weights(), synth.make_bn(widths=UW)


@pytest.fixture(scope="module")
def net(params):
    n = slim.SlimNet(*params, widths=UW, max_batch=64)
    yield n
    n.close()


@pytest.fixture(scope="module")
def ref(params):
    return oracle.Model(*params, widths=UW)


def _input(seg, r_prev, B, seed):
    """(device input of c_act channels, zero padded; oracle input of c channels)."""
    if seg == 0:
        x = synth.make_images(B, offset=seed)
        return torch.from_numpy(x).to(torch.bfloat16).cuda(), x
    H = 32 >> (seg - 1)
    C = synth.BASE_CHANNELS[seg - 1]
    c, ca = slim.slim_channels(r_prev, C), slim.slim_act_channels(r_prev, C)
    g = np.random.default_rng(3000 + seed)
    x = synth.round_bf16(np.abs(g.standard_normal((B, H, H, c), dtype=np.float32)))
    xp = np.zeros((B, H, H, ca), np.float32)
    xp[..., :c] = x
    return torch.from_numpy(xp).to(torch.bfloat16).cuda(), x


def _check(got, exp, tau, what):
    err = oracle.per_image_rel_err(got, exp)
    assert np.isfinite(got).all(), what
    assert err.max() <= tau, f"{what}: worst per-image rel err {err.max():.3e}"


@pytest.mark.parametrize("seg,r_prev,r", [(0, None, 0.3), (0, None, 0.6), (0, None, 0.9), (1, 0.3, 0.6),
                                          (1, 0.9, 0.3), (2, 0.6, 0.9), (2, 0.25, 0.3), (3, 0.9, 0.6),
                                          (3, 0.3, 0.9), (3, 1.0, 0.3)])
def test_universal_segment(net, ref, seg, r_prev, r):
    xd, x = _input(seg, r_prev, 9, seg)
    got = net.forward(seg, xd, r_prev if seg else r, r).float().cpu().numpy()
    exp = ref.segment(seg, x, r_prev, r)
    if seg < 3:
        c = slim.slim_channels(r, synth.BASE_CHANNELS[seg])
        assert got.shape[-1] == slim.slim_act_channels(r, synth.BASE_CHANNELS[seg])
        assert (got[..., c:] == 0).all(), "padded channels must be exact zeros"
        got = got[..., :c]
    _check(got, exp, TAU_BF16, f"universal seg{seg} ({r_prev}->{r})")


@pytest.mark.parametrize("tup", [(0.3, 0.6, 0.9, 0.3), (0.9, 0.9, 0.9, 0.9), (0.6, 0.3, 1.0, 0.9),
                                 (0.25, 0.5, 0.75, 1.0)])
def test_universal_chain(net, ref, tup):
    x = synth.make_images(33, offset=12)
    got = net.forward_chain(torch.from_numpy(x).to(torch.bfloat16).cuda(), tup).cpu().numpy()
    _check(got, ref.chain(x, tup), TAU_BF16, f"universal chain {tup}")


def test_universal_batch_independence_bitwise(net):
    x = torch.from_numpy(synth.make_images(16, offset=4)).to(torch.bfloat16).cuda()
    a = net.forward_chain(x, (0.9, 0.3, 0.6, 1.0)).cpu()
    b = net.forward_chain(x[:5].contiguous(), (0.9, 0.3, 0.6, 1.0)).cpu()
    torch.testing.assert_close(b, a[:5], rtol=0, atol=0)


def test_universal_fp32_mode(params):
    n = slim.SlimNet(*params, widths=UW, max_batch=8, dtype="fp32")
    x = synth.make_images(3, offset=6)
    tup = (0.3, 0.9, 0.6, 0.3)
    got = n.forward_chain(torch.from_numpy(x).cuda(), tup).cpu().numpy()
    n.close()
    _check(got, oracle.Model(*params, widths=UW).chain(x, tup), TAU_FP32, "universal fp32 chain")
