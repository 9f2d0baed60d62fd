"""GPU parity of the GroupNorm variant ("Group Normalization instead of Batch
Normalization"; reading R16: 16 channels per group)
through the C-ABI (slim_config.norm = SLIM_NORM_GN) against the fp64 oracle
(oracle.Model(norm="gn")).  Same tolerance rule as tests/test_gpu_parity.py:
per image max|GPU - oracle| <= tau * max|oracle|, tau 2e-2 (bf16), 1e-4 (FP32 mode).
"""
import numpy as np
import pytest
import torch

import oracle
import synth
import paper_2510_09018_b200 as slim

pytestmark = pytest.mark.gpu

TAU_BF16 = 2e-2
TAU_FP32 = 1e-4
W4 = synth.WIDTHS


def _dev(a, dtype=torch.bfloat16):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dtype).cuda()


@pytest.fixture(scope="module")
def params():
    return synth.make_weights(), synth.make_bn()


@pytest.fixture(scope="module")
def net(params):
    n = slim.SlimNet(*params, max_batch=256, norm="gn")
    yield n
    n.close()


@pytest.fixture(scope="module")
def ref(params):
    return oracle.Model(*params, norm="gn")


def _seg_input(seg, r_prev, B, seed):
    if seg == 0:
        return synth.make_images(B, offset=seed)
    H = 32 >> (seg - 1)
    C = synth.active_channels(r_prev, synth.BASE_CHANNELS[seg - 1])
    g = np.random.default_rng(2000 + seed)
    return synth.round_bf16(np.abs(g.standard_normal((B, H, H, C), dtype=np.float32)))


def _check(got, exp, tau, what):
    err = oracle.per_image_rel_err(got, exp)
    assert np.isfinite(got).all(), f"{what}: non-finite output"
    assert err.max() <= tau, f"{what}: worst per-image rel err {err.max():.3e} > {tau}"
    return err


@pytest.mark.parametrize("r", W4)
def test_gn_segment0(net, ref, r):
    x = _seg_input(0, None, 9, 0)
    got = net.forward(0, _dev(x), r, r).float().cpu().numpy()
    _check(got, ref.segment(0, x, None, r), TAU_BF16, f"GN seg0 r={r}")


@pytest.mark.parametrize("seg", [1, 2, 3])
@pytest.mark.parametrize("r_prev,r", [(0.25, 0.25), (1.0, 1.0), (0.5, 0.75), (0.75, 0.25), (0.25, 1.0)])
def test_gn_segment(net, ref, seg, r_prev, r):
    x = _seg_input(seg, r_prev, 9, seg)
    got = net.forward(seg, _dev(x), r_prev, r).float().cpu().numpy()
    _check(got, ref.segment(seg, x, r_prev, r), TAU_BF16, f"GN seg{seg} ({r_prev}->{r})")


@pytest.mark.parametrize("tup", synth.TABLE_TUPLES)
def test_gn_chain_table_tuples(net, ref, tup):
    x = synth.make_images(9, offset=21)
    got = net.forward_chain(_dev(x), tup).cpu().numpy()
    exp = ref.chain(x, tup)
    _check(got, exp, TAU_BF16, f"GN chain {tup}")
    # argmax agrees wherever the oracle's top-2 margin exceeds the tolerance band
    top2 = np.sort(exp, 1)[:, -2:]
    band = 2 * TAU_BF16 * np.abs(exp).max(1)
    assert ((got.argmax(1) == exp.argmax(1)) | (top2[:, 1] - top2[:, 0] < band)).all()


@pytest.mark.parametrize("r", W4)
def test_gn_chain_bench_batch_sampled(net, ref, r):
    """B=128 (the bench configuration); 4 sampled images checked one by one (GN has no cross-image term)."""
    x = synth.make_images(128, offset=5)
    got = net.forward_chain(_dev(x), (r,) * 4).cpu().numpy()
    idx = [0, 37, 90, 127]
    _check(got[idx], ref.chain(x[idx], (r,) * 4), TAU_BF16, f"GN chain r={r} B=128")


def test_gn_batch_independence_bitwise(net):
    x = synth.make_images(130, offset=8)
    tup = (0.5, 1.0, 0.25, 0.75)
    full = net.forward_chain(_dev(x), tup).cpu().numpy()
    for B in (1, 7):
        part = net.forward_chain(_dev(x[:B]), tup).cpu().numpy()
        np.testing.assert_array_equal(part, full[:B])


def test_gn_differs_from_bn(params):
    """Negative control: the GN context really normalises per group (BN context differs)."""
    x = synth.make_images(4, offset=2)
    with_gn = slim.SlimNet(*params, max_batch=8, norm="gn")
    with_bn = slim.SlimNet(*params, max_batch=8)
    a = with_gn.forward_chain(_dev(x), (1.0,) * 4).cpu().numpy()
    b = with_bn.forward_chain(_dev(x), (1.0,) * 4).cpu().numpy()
    with_gn.close()
    with_bn.close()
    assert np.abs(a - b).max() > 1e-2


@pytest.mark.parametrize("tup", [(1.0, 0.75, 0.5, 0.25), (0.25, 0.5, 0.75, 1.0)])
def test_gn_fp32_mode(params, tup):
    net32 = slim.SlimNet(*params, max_batch=16, norm="gn", dtype="fp32")
    x = synth.make_images(5, offset=13)
    got = net32.forward_chain(_dev(x, torch.float32), tup).cpu().numpy()
    net32.close()
    _check(got, oracle.Model(*params, norm="gn").chain(x, tup), TAU_FP32, f"GN fp32 chain {tup}")


def test_gn_graph_replay_equals_eager(params):
    x = _dev(synth.make_images(16, offset=4))
    tup = (0.75, 0.25, 1.0, 0.5)
    n = slim.SlimNet(*params, max_batch=16, norm="gn")
    eager = n.forward_chain(x, tup).clone()
    slim.slim_set_graph_mode(n.ctx, True)
    g1 = n.forward_chain(x, tup).clone()
    g2 = n.forward_chain(x, tup).clone()
    n.close()
    torch.testing.assert_close(g1, eager, rtol=0, atol=0)
    torch.testing.assert_close(g2, eager, rtol=0, atol=0)


@pytest.mark.parametrize("blocks", [(1, 1, 1, 1), (2, 1, 1, 3)])
def test_gn_other_depths_pool_paths(blocks):
    """Depths where the last block of segment 3 is (or is not) the down-sampling block: the fused
    average pool of the last GN lands in a free workspace buffer (chain), and the unfused head runs
    when the only candidate is the caller's input (slim_forward of segment 3)."""
    w = synth.make_weights(blocks=blocks)
    bn = synth.make_bn(blocks=blocks)
    n = slim.SlimNet(w, bn, max_batch=16, norm="gn", blocks_per_seg=blocks)
    ref = oracle.Model(w, bn, blocks=blocks, norm="gn")
    x = synth.make_images(9, offset=41)
    tup = (0.5, 1.0, 0.25, 0.75)
    got = n.forward_chain(_dev(x), tup).cpu().numpy()
    _check(got, ref.chain(x, tup), TAU_BF16, f"GN chain blocks={blocks}")
    h = _seg_input(3, 0.25, 5, 3)
    got3 = n.forward(3, _dev(h), 0.25, 0.75).cpu().numpy()
    _check(got3, ref.segment(3, h, 0.25, 0.75), TAU_BF16, f"GN seg3 blocks={blocks}")
    n.close()


def test_gn_statistics_partials_path_parity():
    """The opt-in GroupNorm path (SLIM_GN_PART=1): the halo conv writes per-(image, tile, group) statistics
    partials and the GN becomes an elementwise pass over them -- same network within tolerance of the
    oracle, bitwise batch independent."""
    import os, subprocess, sys
    code = (
        "import numpy as np, torch, synth, oracle, paper_2510_09018_b200 as slim\n"
        "w, bn = synth.make_weights(), synth.make_bn()\n"
        "net = slim.SlimNet(w, bn, max_batch=64, norm='gn')\n"
        "ref = oracle.Model(w, bn, norm='gn')\n"
        "x = synth.make_images(20, offset=37)\n"
        "xd = torch.from_numpy(x).to(torch.bfloat16).cuda()\n"
        "worst = 0.0\n"
        "for t in ((1.0, 1.0, 1.0, 1.0), (0.25, 0.75, 0.5, 1.0), (0.5, 0.5, 0.25, 0.25)):\n"
        "    got = net.forward_chain(xd, t)\n"
        "    sub = net.forward_chain(xd[3:7].contiguous(), t)\n"
        "    assert torch.equal(got[3:7], sub)\n"
        "    worst = max(worst, float(oracle.per_image_rel_err(got[:3].cpu().numpy(), ref.chain(x[:3], t)).max()))\n"
        "print(worst)\n"
    )
    out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, SLIM_GN_PART="1"), capture_output=True,
                         text=True, timeout=600, cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert out.returncode == 0, out.stderr[-2000:]
    assert float(out.stdout.strip().splitlines()[-1]) <= 2e-2


def test_fused_segment0_gn_parity_and_cluster_bitwise():
    """GroupNorm inside the fused segment-0 kernel (two-pass statistics over the fp32 raw output, one
    fixed merge tree): within tolerance of the oracle for r = 0.25 / 0.5, and the 8-CTA cluster variant
    (small batches) bit-identical to the one-CTA-per-image variant."""
    import os, subprocess, sys, tempfile
    code = (
        "import sys, numpy as np, torch, synth, paper_2510_09018_b200 as slim\n"
        "w, bn = synth.make_weights(), synth.make_bn()\n"
        "net = slim.SlimNet(w, bn, max_batch=16, norm='gn')\n"
        "x = torch.from_numpy(synth.make_images(9, offset=71)).to(torch.bfloat16).cuda()\n"
        "o = [net.forward(0, x, r, r).view(torch.int16).cpu().numpy() for r in (0.25, 0.5)]\n"
        "np.savez(sys.argv[1], o0=o[0], o1=o[1])\n"
    )
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with tempfile.TemporaryDirectory() as d:
        res = {}
        for name, cl in (("p8", "8"), ("p1", "0")):
            out = subprocess.run([sys.executable, "-c", code, os.path.join(d, name + ".npz")],
                                 env=dict(os.environ, SLIM_SEG0_CLUSTER=cl), capture_output=True, text=True,
                                 timeout=300, cwd=root)
            assert out.returncode == 0, out.stderr[-2000:]
            res[name] = np.load(os.path.join(d, name + ".npz"))
        for k in ("o0", "o1"):
            assert np.array_equal(res["p8"][k], res["p1"][k]), k
    w, bn = synth.make_weights(), synth.make_bn()
    ref = oracle.Model(w, bn, norm="gn")
    x = synth.make_images(9, offset=71)
    for k, r in (("o0", 0.25), ("o1", 0.5)):
        got = (res["p8"][k].astype(np.int32).astype(np.uint32) << 16).view(np.float32)
        err = oracle.per_image_rel_err(got[:3], ref.segment(0, x[:3], None, r))
        assert err.max() <= 2e-2, (r, err.max())


@pytest.mark.parametrize("seg", [1, 2, 3])
def test_fused_segments_gn_parity(seg):
    """GroupNorm inside the fused segment-1..3 kernels (statistics per image of the unit, channel slices over
    the cluster): every (r_prev, r) the fused kernel takes against the oracle, ragged unit counts, and
    bitwise batch independence (an image's statistics never depend on its slot in the unit)."""
    w, bn = synth.make_weights(), synth.make_bn()
    net = slim.SlimNet(w, bn, max_batch=16, norm="gn")
    ref = oracle.Model(w, bn, norm="gn")
    H = 32 >> (seg - 1)
    worst = 0.0
    for rp in synth.WIDTHS:
        C = synth.active_channels(rp, synth.BASE_CHANNELS[seg - 1])
        g = np.random.default_rng(900 + seg)
        x = synth.round_bf16(np.abs(g.standard_normal((11, H, H, C), dtype=np.float32)))
        xd = torch.from_numpy(x).to(torch.bfloat16).cuda()
        for r in (0.25, 0.5):
            got = net.forward(seg, xd, rp, r)
            sub = net.forward(seg, xd[3:6].contiguous(), rp, r)
            assert torch.equal(got[3:6], sub), (rp, r)
            gotn = got.float().cpu().numpy()
            err = oracle.per_image_rel_err(gotn[[0, 4, 10]], ref.segment(seg, x[[0, 4, 10]], rp, r))
            worst = max(worst, float(err.max()))
    net.close()
    assert worst <= 2e-2, worst


def test_gn_epilogue_image_pairs_opt_in():
    """SLIM_GN_PAIRS=1: segment 1's GroupNorm in the conv epilogue with one CTA taking both M tiles of an
    image (statistics over the two TMEM-resident accumulators) -- within tolerance of the oracle for every
    (r_prev, r) it accepts, and bitwise batch independent."""
    import os, subprocess, sys
    code = (
        "import numpy as np, torch, synth, oracle, paper_2510_09018_b200 as slim\n"
        "w, bn = synth.make_weights(), synth.make_bn()\n"
        "net = slim.SlimNet(w, bn, max_batch=32, norm='gn')\n"
        "ref = oracle.Model(w, bn, norm='gn')\n"
        "worst = 0.0\n"
        "for rp in synth.WIDTHS:\n"
        "    C = synth.active_channels(rp, synth.BASE_CHANNELS[0])\n"
        "    g = np.random.default_rng(7)\n"
        "    x = synth.round_bf16(np.abs(g.standard_normal((9, 32, 32, C), dtype=np.float32)))\n"
        "    xd = torch.from_numpy(x).to(torch.bfloat16).cuda()\n"
        "    for r in synth.WIDTHS:\n"
        "        got = net.forward(1, xd, rp, r).float().cpu().numpy()\n"
        "        err = oracle.per_image_rel_err(got, ref.segment(1, x, rp, r))\n"
        "        worst = max(worst, float(err.max()))\n"
        "        one = net.forward(1, xd[4:5].contiguous(), rp, r).float().cpu().numpy()\n"
        "        assert np.array_equal(one[0], got[4]), (rp, r)\n"
        "print(worst)\n"
    )
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SLIM_GN_PAIRS="1", SLIM_NO_FUSED="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    assert float(out.stdout.strip().splitlines()[-1]) <= TAU_BF16
