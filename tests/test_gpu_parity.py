"""GPU parity: the CUDA path (through the C-ABI) against the fp64 CPU oracle.

Tolerance (north_star; reading D4): per image, max|GPU - oracle| <= tau * max|oracle|
over that image's output elements, tau = 2e-2 in bf16 mode, 1e-4 in FP32 mode.
Bit-exact checks where the arithmetic is exact (closed form, prefix isolation,
batch independence, chain = composition of segments).
Inputs: seeded synthetic (synth/), shapes of the paper's workload (CIFAR-100-shaped
32x32x3 images); batch sizes span several M-tiles with a ragged tail.
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
    w, bn = params
    n = slim.SlimNet(w, bn, max_batch=512)
    yield n
    n.close()


@pytest.fixture(scope="module")
def ref(params):
    return oracle.Model(*params)


def _seg_input(seg, r_prev, B, seed):
    """bf16-representable input of segment `seg`: images for seg 0, else a non-negative
    post-ReLU-like activation [B, H_{s-1}, H_{s-1}, c_{s-1}(r_prev)]."""
    if seg == 0:
        return synth.make_images(B, offset=seed)
    H = 32 >> (seg - 1)
    C = synth.active_channels(r_prev, synth.BASE_CHANNELS[seg - 1])
    g = np.random.default_rng(1000 + seed)
    return synth.round_bf16(np.abs(g.standard_normal((B, H, H, C), dtype=np.float32)))


def _check(got, exp, tau, what):
    err = oracle.per_image_rel_err(got, exp)
    assert np.isfinite(got).all(), f"{what}: non-finite output"
    assert err.max() <= tau, f"{what}: worst per-image rel err {err.max():.3e} > {tau} (median {np.median(err):.2e})"
    return err


# ------------------------------------------------------------------ per segment, every (r_prev, r)
@pytest.mark.parametrize("r", W4)
def test_segment0_parity(net, ref, r):
    x = _seg_input(0, None, 9, 0)
    got = net.forward(0, _dev(x), r, r).float().cpu().numpy()
    _check(got, ref.segment(0, x, None, r), TAU_BF16, f"seg0 r={r}")


@pytest.mark.parametrize("seg", [1, 2, 3])
@pytest.mark.parametrize("r_prev", W4)
@pytest.mark.parametrize("r", W4)
def test_segment_parity_all_width_pairs(net, ref, seg, r_prev, r):
    B = 9   # seg2: 2 images per M-tile, seg3: 8 -> ragged last tile
    x = _seg_input(seg, r_prev, B, seg)
    got = net.forward(seg, _dev(x), r_prev, r).float().cpu().numpy()
    _check(got, ref.segment(seg, x, r_prev, r), TAU_BF16, f"seg{seg} ({r_prev}->{r})")


# ------------------------------------------------------------------ whole chain
@pytest.mark.parametrize("tup", synth.TABLE_TUPLES)
def test_chain_parity_table_tuples(net, ref, tup):
    """The 8 width tuples of PAPER.md Tables I-II, full chain + head, logits per image."""
    x = synth.make_images(12, offset=7)
    got = net.forward_chain(_dev(x), tup).cpu().numpy()
    _check(got, ref.chain(x, tup), TAU_BF16, f"chain {tup}")


def test_chain_equals_composition_bitwise(net):
    x = _dev(synth.make_images(10, offset=8))
    tup = (1.0, 0.5, 0.25, 0.75)
    a = net.forward_chain(x, tup)
    h = net.forward(0, x, tup[0], tup[0])
    for s in range(1, 4):
        h = net.forward(s, h, tup[s - 1], tup[s])
    torch.cuda.synchronize()
    assert torch.equal(a, h)


def test_batch_independence_bitwise(net):
    x = synth.make_images(130, offset=9)
    tup = (0.5, 0.75, 1.0, 0.25)
    full = net.forward_chain(_dev(x), tup).cpu()
    for idx in ([0], [129], list(range(37, 44))):
        part = net.forward_chain(_dev(x[idx]), tup).cpu()
        assert torch.equal(part, full[idx]), idx


def test_sampled_parity_at_bench_size(net, ref):
    """B=128 (CFG2, the bench config) at every width; 6 sampled images through the oracle
    (batch independence makes a sample exact)."""
    x = synth.make_images(128, offset=10)
    pick = [0, 1, 63, 64, 126, 127]
    for r in W4:
        got = net.forward_chain(_dev(x), (r,) * 4).cpu().numpy()[pick]
        _check(got, ref.chain(x[pick], (r,) * 4), TAU_BF16, f"B=128 r={r}")


# ------------------------------------------------------------------ invariants
def test_nan_prefix_isolation_bitwise(params):
    """Weights outside the active prefix are NaN: output finite and bitwise unchanged
    (the prefix is selected by TMA bounds, not read-and-masked)."""
    w, bn = params
    r_prev, r = 0.5, 0.25
    clean = slim.SlimNet(w, bn, max_batch=16, segments=(1,))
    dirty = slim.SlimNet(synth.nan_poison_weights(w, r_prev, r), bn, max_batch=16, segments=(1,))
    x = _dev(_seg_input(1, r_prev, 5, 11))
    a = clean.forward(1, x, r_prev, r)
    b = dirty.forward(1, x, r_prev, r)
    torch.cuda.synchronize()
    assert torch.isfinite(b.float()).all()
    assert torch.equal(a, b)
    clean.close()
    dirty.close()


def test_bn_width_selection_negative_control(net, ref):
    x = synth.make_images(4, offset=12)
    got = net.forward(0, _dev(x), 0.25, 0.25).float().cpu().numpy()
    _check(got, ref.segment(0, x, None, 0.25), TAU_BF16, "bn select")
    wrong = ref.segment(0, x, None, 0.25, bn_width=0.5)
    assert oracle.per_image_rel_err(got, wrong).min() > 5 * TAU_BF16


def _delta_params():
    weights, bn = {}, {}
    for sp in synth.layer_specs():
        wt = np.zeros((sp["cout"], sp["k"], sp["k"], sp["cin"]), np.float32)
        c = sp["k"] // 2
        for i in range(min(sp["cout"], sp["cin"])):
            wt[i, c, c, i] = 1.0
        weights[sp["name"]] = wt
        bn[sp["name"]] = [dict(gamma=np.full(n, 0.5, np.float32), beta=np.zeros(n, np.float32),
                               mean=np.zeros(n, np.float32), var=np.full(n, np.float32(0.25 - 1e-5), np.float32))
                          for n in (synth.active_channels(r, sp["cout"]) for r in W4)]
    weights["fc_w"] = synth.make_weights()["fc_w"]
    weights["fc_b"] = np.zeros(100, np.float32)
    return weights, bn


def test_closed_form_delta_network_bitwise():
    """Centre-tap delta kernels, BN folding to exactly s=1, t=0: seg0 = 4*relu(x) on channels<3,
    each later segment = 4*h[::2, ::2] -- powers of two, exact in bf16, so bitwise."""
    net = slim.SlimNet(*_delta_params(), max_batch=16)
    x = synth.make_images(3, offset=13)
    rx = np.maximum(x, 0)
    tup = (0.75, 0.25, 1.0, 0.5)
    h = net.forward(0, _dev(x), tup[0], tup[0])
    exp = np.zeros(tuple(h.shape), np.float32)
    exp[..., :3] = 4 * rx
    assert np.array_equal(h.float().cpu().numpy(), exp)
    for s in (1, 2):
        h = net.forward(s, h, tup[s - 1], tup[s])
        exp = np.zeros(tuple(h.shape), np.float32)
        exp[..., :3] = 4 ** (s + 1) * rx[:, ::2 ** s, ::2 ** s, :]
        assert np.array_equal(h.float().cpu().numpy(), exp), s
    net.close()


# ------------------------------------------------------------------ error paths
def test_error_paths(net):
    x = _dev(synth.make_images(2, offset=14))
    with pytest.raises(slim.SlimError, match="EINVAL"):
        net.forward(0, x, 0.3, 0.3)                    # width not in the set
    with pytest.raises(slim.SlimError, match="EINVAL"):
        slim.slim_forward(net.ctx, 0, 0.25, 0.25, 10_000, x, x)   # B > B_max
    with pytest.raises(slim.SlimError, match="EINVAL"):
        slim.slim_forward(net.ctx, 4, 0.25, 0.25, 2, x, x)        # seg out of range
    with pytest.raises(slim.SlimError, match="EINVAL"):
        slim.slim_forward(net.ctx, 0, 0.25, 0.25, 0, x, x)        # empty batch
    with pytest.raises(slim.SlimError, match="EINVAL"):
        slim.slim_forward(net.ctx, 0, 0.25, 0.25, 2, x.data_ptr() + 2, x)   # input not 16-B aligned
    assert slim.slim_last_error(net.ctx) == 0


def test_not_loaded(params):
    w, bn = params
    n = slim.SlimNet(w, bn, max_batch=4, segments=(0,))
    x = _dev(_seg_input(1, 0.25, 2, 15))
    with pytest.raises(slim.SlimError, match="ENOTLOADED"):
        n.forward(1, x, 0.25, 0.25)
    slim.slim_unload_segment(n.ctx, 0)
    with pytest.raises(slim.SlimError, match="ENOTLOADED"):
        n.forward(0, _dev(synth.make_images(2)), 0.25, 0.25)
    n.close()


# ------------------------------------------------------------------ packer + gather launch
def test_pack_gather_launch_matches_direct(net, ref):
    """Requests scattered in a pool, grouped by key (s, w_req, w_prev), gathered by the K8
    kernel and run; each output equals the direct forward of the same images."""
    rng = np.random.default_rng(16)
    n = 23
    seg = 1
    keys = [(0.5, 0.25), (1.0, 0.25), (0.5, 0.75)]
    pool_np = _seg_input(1, 1.0, n, 16)                       # pool rows sized for the widest r_prev
    reqs = []
    for i in range(n):
        wr, wp = keys[rng.integers(0, 3)]
        reqs.append((i, seg, wr, wp, i))
    descs, order = slim.slim_pack(net.cfg, reqs, 8)
    C_full = synth.BASE_CHANNELS[0]
    row_bytes = 32 * 32 * C_full * 2
    for d in descs:
        idx = order[d["first"]:d["first"] + d["batch"]]
        cin = synth.active_channels(d["r_prev"], C_full)
        # the pool holds each request's activation at its own width r_prev (dense prefix per row)
        pool = np.zeros((n, 32, 32, C_full), np.float32)
        pool.reshape(n, -1)[:, :32 * 32 * cin] = pool_np[..., :cin].reshape(n, -1)
        pool_d = _dev(pool)
        slots = torch.from_numpy(idx.astype(np.int32)).cuda()
        slab = torch.empty(d["batch"], 32, 32, cin, dtype=torch.bfloat16, device="cuda")
        out = torch.empty(net.segment_out_shape(seg, d["r"], d["batch"]), dtype=torch.bfloat16, device="cuda")
        ws_b = slim.slim_forward_workspace_bytes(net.ctx, seg, d["r_prev"], d["r"], d["batch"])
        ws = torch.empty(ws_b, dtype=torch.uint8, device="cuda")
        slim.slim_launch(net.ctx, d, slots, pool_d, row_bytes, slab, out, ws, ws_b)
        direct = net.forward(seg, _dev(pool_np[idx][..., :cin]), d["r_prev"], d["r"])
        torch.cuda.synchronize()
        assert torch.equal(out, direct)


# ------------------------------------------------------------------ graph mode + profiling
def test_graph_mode_bitwise_and_launch_count(params):
    w, bn = params
    n = slim.SlimNet(w, bn, max_batch=32)
    x = _dev(synth.make_images(20, offset=17))
    tup = (0.25, 1.0, 0.75, 0.5)
    a = n.forward_chain(x, tup).clone()
    c0 = slim.slim_launch_count(n.ctx)
    n.forward_chain(x, tup)
    per_chain = slim.slim_launch_count(n.ctx) - c0
    # segment 0 at r = 0.25 is one fused kernel (stem + both blocks); then 2 convs x 6 blocks + head
    assert per_chain == 1 + 4 * 3 + 1
    slim.slim_set_graph_mode(n.ctx, True)
    logits = torch.empty_like(a)
    for _ in range(3):
        n.forward_chain(x, tup, logits=logits)
        torch.cuda.synchronize()
        assert torch.equal(logits, a)
    c1 = slim.slim_launch_count(n.ctx)
    n.forward_chain(x, tup, logits=logits)
    assert slim.slim_launch_count(n.ctx) - c1 == per_chain
    n.close()


def test_profile_records_cover_every_launch(net):
    x = _dev(synth.make_images(16, offset=18))
    slim.slim_profile_begin(net.ctx, 64)
    net.forward_chain(x, (1.0,) * 4)
    recs = slim.slim_profile_end(net.ctx)
    assert len(recs) == 18
    kinds = [r["kind"] for r in recs]
    assert kinds[0] == "stem" and kinds[-1] == "head" and kinds.count("conv_umma") == 16
    assert all(r["ms"] > 0 for r in recs)
    # sliced FLOPs of the r=1 chain: 1110.94 MFLOP per image
    total = sum(r["flops"] for r in recs) / 16
    assert abs(total / 1e6 - 1110.94) / 1110.94 < 2e-3


# ------------------------------------------------------------------ FP32 mode (TF32 off)
@pytest.fixture(scope="module")
def net32(params):
    w, bn = params
    n = slim.SlimNet(w, bn, max_batch=64, dtype="fp32")
    yield n
    n.close()


@pytest.mark.parametrize("tup", [(1.0, 1.0, 1.0, 1.0), (0.25, 0.25, 0.25, 0.25), (1.0, 0.75, 0.5, 0.25),
                                 (0.5, 0.25, 1.0, 0.75)])
def test_fp32_chain_parity(net32, ref, tup):
    """FP32 storage + FFMA accumulation (SIMT kernels, no TF32): <= 1e-4 per image (north_star)."""
    x = synth.make_images(9, offset=19)
    got = net32.forward_chain(_dev(x, torch.float32), tup).cpu().numpy()
    _check(got, ref.chain(x, tup), TAU_FP32, f"fp32 chain {tup}")


@pytest.mark.parametrize("seg,r_prev,r", [(0, None, 0.75), (1, 0.25, 1.0), (2, 1.0, 0.5), (3, 0.5, 0.25)])
def test_fp32_segment_parity(net32, ref, seg, r_prev, r):
    x = _seg_input(seg, r_prev if r_prev else 0.25, 5, 20)
    got = net32.forward(seg, _dev(x, torch.float32), r_prev if seg else r, r).cpu().numpy()
    _check(got, ref.segment(seg, x, r_prev, r), TAU_FP32, f"fp32 seg{seg}")


# ------------------------------------------------------------------ request stream (CFG4)
@pytest.mark.parametrize("lanes", [1, 4, 8])
def test_stream_executor_matches_per_request_chain(net, lanes):
    """Mixed-width stream: key batching per segment + gather/scatter; each request's logits are
    bitwise the chain of its own tuple (batch independence makes grouping invisible); lanes = 4
    runs a segment's batches concurrently on one stream per width."""
    from paper_2510_09018_b200.stream import StreamExecutor
    from paper_2510_09018_b200.router import TABLE_TUPLES
    rng = np.random.default_rng(21)
    n = 61
    tup = np.asarray([TABLE_TUPLES[i] for i in rng.integers(0, len(TABLE_TUPLES), n)], np.float32)
    x = synth.make_images(n, offset=21)
    ex = StreamExecutor(net, n_max=64, B_max=8, lanes=lanes)
    got = ex.run(_dev(x), tup).clone()
    torch.cuda.synchronize()
    assert max(max(b) for b in ex.last_batches) <= 8
    for t in set(map(tuple, tup.tolist())):
        idx = [i for i in range(n) if tuple(tup[i].tolist()) == t]
        ref_l = net.forward_chain(_dev(x[idx]), t)
        assert torch.equal(got[idx], ref_l), t


@pytest.mark.parametrize("lanes", [1, 8])
def test_native_stream_executor_matches_python_and_chain(net, lanes):
    """slim_stream_run (the C++ sequencer) on three consecutive fresh streams (the staging buffers
    alternate and are reused): bitwise the Python executor's logits and each tuple's own chain;
    n = 1 and a single-key stream are the degenerate cases."""
    from paper_2510_09018_b200.stream import NativeStreamExecutor, StreamExecutor
    from paper_2510_09018_b200.router import TABLE_TUPLES
    nx = NativeStreamExecutor(net, n_max=64, B_max=8, lanes=lanes)
    px = StreamExecutor(net, n_max=64, B_max=8, lanes=lanes)
    px.cache_plans = False
    for seed, n in ((22, 61), (23, 64), (24, 1)):
        rng = np.random.default_rng(seed)
        tup = np.asarray([TABLE_TUPLES[i] for i in rng.integers(0, len(TABLE_TUPLES), n)], np.float32)
        x = _dev(synth.make_images(n, offset=seed))
        got = nx.run(x, tup).clone()
        want = px.run(x, tup).clone()
        torch.cuda.synchronize()
        assert torch.equal(got, want), (seed, n)
        assert nx.last_n_batches == sum(len(b) for b in px.last_batches)
        for t in set(map(tuple, tup.tolist())):
            idx = [i for i in range(n) if tuple(tup[i].tolist()) == t]
            assert torch.equal(got[idx], net.forward_chain(x[idx], t)), t
    tup = np.tile(np.asarray([[0.5, 0.25, 1.0, 0.75]], np.float32), (40, 1))
    x = _dev(synth.make_images(40, offset=25))
    got = nx.run(x, tup).clone()
    torch.cuda.synchronize()
    assert nx.last_n_batches == 4 * 5                     # 40 requests, B_max 8, one key per segment
    assert torch.equal(got, net.forward_chain(x, (0.5, 0.25, 1.0, 0.75)))
    with pytest.raises(slim.SlimError):                  # a width outside cfg.widths: rejected before any launch
        nx.run(x, np.full((40, 4), 0.3, np.float32))
    nx.close()


def test_cluster_multicast_path_parity(params, ref):
    """The A-tile multicast variant (cluster of CTAs sharing an M tile; off by default, SLIM_MC_MAX)
    computes the same results: run it through a subprocess with the env var set."""
    import subprocess, sys, os
    code = (
        "import numpy as np, torch, synth, oracle, paper_2510_09018_b200 as slim\n"
        "w, bn = synth.make_weights(), synth.make_bn()\n"
        "net = slim.SlimNet(w, bn, max_batch=64)\n"
        "x = synth.make_images(40, offset=23)\n"
        "got = net.forward_chain(torch.from_numpy(x).to(torch.bfloat16).cuda(), (1.0, 1.0, 1.0, 1.0)).cpu().numpy()\n"
        "err = oracle.per_image_rel_err(got[:4], oracle.Model(w, bn).chain(x[:4], (1.0,) * 4))\n"
        "print(err.max())\n"
    )
    env = dict(os.environ, SLIM_MC_MAX="4")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert out.returncode == 0, out.stderr[-2000:]
    assert float(out.stdout.strip().splitlines()[-1]) <= TAU_BF16


def _seg123_outputs_under_env(tmp_path, variants):
    """Every segment 1-3 output for all (r_prev, r) at B = 13 and 64 (per-layer kernels), once per env
    variant, each run in its own process (the knobs are read once); the oracle checks a sample."""
    import subprocess, sys, os
    code = (
        "import sys, numpy as np, torch, synth, oracle, paper_2510_09018_b200 as slim\n"
        "w, bn = synth.make_weights(), synth.make_bn()\n"
        "net = slim.SlimNet(w, bn, max_batch=64)\n"
        "W = synth.WIDTHS\n"
        "outs = {}\n"
        "for seg in (1, 2, 3):\n"
        "    H = 32 >> (seg - 1)\n"
        "    for rp in W:\n"
        "        C = synth.active_channels(rp, synth.BASE_CHANNELS[seg - 1])\n"
        "        g = np.random.default_rng(91 + seg)\n"
        "        x = synth.round_bf16(np.abs(g.standard_normal((64, H, H, C), dtype=np.float32)))\n"
        "        xd = torch.from_numpy(x).to(torch.bfloat16).cuda()\n"
        "        for r in W:\n"
        "            for B in (13, 64):\n"
        "                outs[f'{seg}_{rp}_{r}_{B}'] = net.forward(seg, xd[:B].contiguous(), rp, r).float().cpu().numpy()\n"
        "        if rp == 1.0:\n"
        "            ref = oracle.Model(w, bn).segment(seg, x[:3], rp, 1.0)\n"
        "            err = oracle.per_image_rel_err(outs[f'{seg}_{rp}_1.0_13'][:3], ref)\n"
        "            assert err.max() <= 2e-2, (seg, err.max())\n"
        "np.savez(sys.argv[1], **outs)\n"
    )
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = []
    for i, var in enumerate(variants):
        f = str(tmp_path / f"v{i}.npz")
        env = dict(os.environ, SLIM_NO_FUSED="1", **var)
        out = subprocess.run([sys.executable, "-c", code, f], env=env, capture_output=True, text=True, timeout=600,
                             cwd=root)
        assert out.returncode == 0, out.stderr[-2000:]
        res.append(np.load(f))
    return res


@pytest.mark.parametrize("bmc", [2, 4])
def test_halo_weight_multicast_bitwise(bmc, tmp_path):
    """Streamed-weight multicast (clusters of bmc CTAs share each B stage, SLIM_HALO_BMC): every
    segment 1-3 output for all (r_prev, r) at B = 13 and 64 is bitwise the unclustered kernel's (same
    MMA order; only who loads the weights changes), and the oracle agrees on a sample."""
    base, mc = _seg123_outputs_under_env(tmp_path, [dict(SLIM_HALO_BMC="1", SLIM_HALO_PAIR="0"),
                                                    dict(SLIM_HALO_BMC=str(bmc), SLIM_HALO_PAIR="0")])
    for k in base.files:
        assert np.array_equal(base[k], mc[k]), k


def test_halo_pair_mma_bitwise(tmp_path):
    """2-SM MMA (cta_group::2, SLIM_HALO_PAIR): a CTA pair issues one M = 256 MMA per k-step with each
    CTA holding half of every weight stage.  Every segment 1-3 output for all (r_prev, r) at B = 13 and
    64 is bitwise the one-CTA kernel's (each output row's K order is unchanged), and the oracle agrees
    on a sample -- so the choice cannot break batch independence."""
    one, two = _seg123_outputs_under_env(tmp_path, [dict(SLIM_HALO_PAIR="0"), dict(SLIM_HALO_PAIR="1")])
    for k in one.files:
        assert np.array_equal(one[k], two[k]), k


def test_splitk_cluster_path_parity():
    """The split-K conv (cluster of CTAs over K, fp32 partials reduced through DSMEM; chosen by a
    cost model, forced here with SLIM_SPLITK_FORCE) matches the oracle on segments 1-3 for every
    (r_prev, r), including the projection shortcut and the fused pool, and stays bitwise batch
    independent (fixed rank-order reduction)."""
    import subprocess, sys, os
    code = (
        "import numpy as np, torch, synth, oracle, paper_2510_09018_b200 as slim\n"
        "w, bn = synth.make_weights(), synth.make_bn()\n"
        "net = slim.SlimNet(w, bn, max_batch=128)\n"
        "ref = oracle.Model(w, bn)\n"
        "W = synth.WIDTHS\n"
        "worst = 0.0\n"
        "for seg in (1, 2, 3):\n"
        "    H = 32 >> (seg - 1)\n"
        "    for rp in W:\n"
        "        C = synth.active_channels(rp, synth.BASE_CHANNELS[seg - 1])\n"
        "        g = np.random.default_rng(77 + seg)\n"
        "        x = synth.round_bf16(np.abs(g.standard_normal((9, H, H, C), dtype=np.float32)))\n"
        "        xd = torch.from_numpy(x).to(torch.bfloat16).cuda()\n"
        "        for r in W:\n"
        "            got = net.forward(seg, xd, rp, r)\n"
        "            sub = net.forward(seg, xd[2:5].contiguous(), rp, r)\n"
        "            assert torch.equal(got[2:5], sub), ('batch independence', seg, rp, r)\n"
        "            err = oracle.per_image_rel_err(got.float().cpu().numpy(), ref.segment(seg, x, rp, r))\n"
        "            worst = max(worst, float(err.max()))\n"
        "print(worst)\n"
    )
    env = dict(os.environ, SLIM_SPLITK_FORCE="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert out.returncode == 0, out.stderr[-2000:]
    assert float(out.stdout.strip().splitlines()[-1]) <= TAU_BF16


@pytest.mark.parametrize("env", [
    "SLIM_NO_HALO=1",                      # every conv through the per-tap kernel (+ split-K where chosen)
    "SLIM_HALO_NO_S2=1 SLIM_HALO_NO_PROJ=1 SLIM_HALO_NO_SMALL=1",   # halo only for large stride-1 layers
    "SLIM_HALO_X3=1",                      # three shifted boxes, one accumulator (opt-in variant)
    "SLIM_HALO_X3=2",                      # two boxes, two accumulators (opt-in variant)
    "SLIM_HALO_STAGES=1 SLIM_HALO_EPI1=1",  # one accumulator stage, one epilogue group
    "SLIM_HALO_NARROW=1",                  # 16/32-channel operand boxes
    "SLIM_NPROD=1",                        # one TMA producer in the per-tap kernel
    "SLIM_HALO_SMALL=1",                   # compact two-CTA-per-SM variant for narrow layers
])
def test_kernel_variant_parity(env):
    """Every kernel variant / fallback a runtime switch can select computes the same network:
    chains at a mixed width tuple and at r=1 against the oracle (subprocess: the switches are
    read once per process)."""
    import subprocess, sys, os
    code = (
        "import numpy as np, torch, synth, oracle, paper_2510_09018_b200 as slim\n"
        "w, bn = synth.make_weights(), synth.make_bn()\n"
        "net = slim.SlimNet(w, bn, max_batch=64)\n"
        "ref = oracle.Model(w, bn)\n"
        "x = synth.make_images(10, offset=31)\n"
        "xd = torch.from_numpy(x).to(torch.bfloat16).cuda()\n"
        "worst = 0.0\n"
        "for t in ((1.0, 1.0, 1.0, 1.0), (0.25, 0.75, 0.5, 1.0)):\n"
        "    got = net.forward_chain(xd, t).cpu().numpy()\n"
        "    worst = max(worst, float(oracle.per_image_rel_err(got[:3], ref.chain(x[:3], t)).max()))\n"
        "print(worst)\n"
    )
    e = dict(os.environ)
    for kv in env.split():
        k, v = kv.split("=")
        e[k] = v
    out = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True, timeout=600,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert out.returncode == 0, out.stderr[-2000:]
    assert float(out.stdout.strip().splitlines()[-1]) <= TAU_BF16, env


def test_sm_share_is_bit_exact(params):
    """SM partitioning (slim_set_sm_share) only changes which CTA computes which tile: bit-exact."""
    w, bn = params
    n = slim.SlimNet(w, bn, max_batch=64)
    x = _dev(synth.make_images(64, offset=31))
    tup = (0.25, 1.0, 0.5, 0.75)
    full = n.forward_chain(x, tup).clone()
    for r, sh in ((0.25, 0.05), (1.0, 0.2), (0.5, 0.33), (0.75, 0.6)):
        slim.slim_set_sm_share(n.ctx, r, sh)
    slim.slim_set_graph_mode(n.ctx, True)
    part = n.forward_chain(x, tup).clone()
    part2 = n.forward_chain(x, tup).clone()
    with pytest.raises(slim.SlimError):
        slim.slim_set_sm_share(n.ctx, 0.3, 0.5)
    with pytest.raises(slim.SlimError):
        slim.slim_set_sm_share(n.ctx, 0.5, 0.0)
    n.close()
    torch.testing.assert_close(part, full, rtol=0, atol=0)
    torch.testing.assert_close(part2, full, rtol=0, atol=0)


@pytest.mark.parametrize("r", [0.25, 1.0])
def test_max_batch_4096(params, ref, r):
    """CFG3's largest batch (B = 4096, the default B_max): 48 sampled images against the oracle, and
    512 sampled images bit-identical to the same images run as a batch of 512 (batch independence
    carries the oracle check to every image)."""
    w, bn = params
    n = slim.SlimNet(w, bn)                       # default config: B_max = 4096
    B = 4096
    x = synth.make_images(B, offset=77)
    xd = _dev(x)
    got = n.forward_chain(xd, (r,) * 4)
    g = np.random.default_rng(int(r * 100))
    idx = np.sort(g.choice(B, 512, replace=False))
    sub = n.forward_chain(xd[torch.from_numpy(idx).cuda()].contiguous(), (r,) * 4)
    torch.testing.assert_close(got[torch.from_numpy(idx).cuda()], sub, rtol=0, atol=0)
    pick = idx[:48]
    _check(got[torch.from_numpy(pick).cuda()].cpu().numpy(), ref.chain(x[pick], (r,) * 4), TAU_BF16,
           f"B=4096 r={r}")
    n.close()



@pytest.mark.parametrize("B", [1, 8, 130])
def test_fused_segment0_bitwise_equals_per_layer(B):
    """Segment 0 at the narrow widths runs as one fused kernel (kernels_fused.cu); the same arithmetic
    as the per-layer stem + halo convs (SLIM_NO_FUSED=1), bit for bit, and within tolerance of the oracle."""
    import subprocess, sys, os
    code = (
        "import sys, numpy as np, torch, synth, paper_2510_09018_b200 as slim\n"
        "w, bn = synth.make_weights(), synth.make_bn()\n"
        f"B = {B}\n"
        "net = slim.SlimNet(w, bn, max_batch=max(B, 16))\n"
        "x = torch.from_numpy(synth.make_images(B, offset=61)).to(torch.bfloat16).cuda()\n"
        "outs = [net.forward(0, x, r, r).view(torch.int16).cpu().numpy() for r in (0.25, 0.5)]\n"
        "logits = net.forward_chain(x, (0.25, 0.5, 0.25, 0.5)).cpu().numpy()\n"
        "np.savez(sys.argv[1], o0=outs[0], o1=outs[1], logits=logits)\n"
    )
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        res = {}
        for name, extra in (("fused", {}), ("layers", {"SLIM_NO_FUSED": "1"})):
            out = subprocess.run([sys.executable, "-c", code, os.path.join(d, name + ".npz")],
                                 env=dict(os.environ, **extra), capture_output=True, text=True, timeout=300, cwd=root)
            assert out.returncode == 0, out.stderr[-2000:]
            res[name] = np.load(os.path.join(d, name + ".npz"))
        for k in ("o0", "o1", "logits"):
            assert np.array_equal(res["fused"][k], res["layers"][k]), k
    x = synth.make_images(B, offset=61)
    ref = oracle.Model(synth.make_weights(), synth.make_bn())
    exp = ref.segment(0, x[:4], None, 0.25)
    got = res["fused"]["o0"][:4].astype(np.int32).astype(np.uint32) << 16
    _check(got.view(np.float32), exp, TAU_BF16, "fused seg0 r=0.25")


@pytest.mark.parametrize("seg", [1, 2, 3])
def test_fused_segments_bitwise_equal_per_layer(seg):
    """Segments 1-3 at the narrow widths as one fused kernel (kernels_fused.cu, forced on for every
    segment with SLIM_FUSED_SEGS=14): bit-identical to the per-layer halo kernels (SLIM_NO_FUSED=1) for
    every (r_prev, r) the fused kernel takes, ragged unit counts included, and within tolerance of the
    oracle."""
    import subprocess, sys, os, tempfile
    code = (
        "import sys, numpy as np, torch, synth, paper_2510_09018_b200 as slim\n"
        "w, bn = synth.make_weights(), synth.make_bn()\n"
        f"seg = {seg}\n"
        "net = slim.SlimNet(w, bn, max_batch=64)\n"
        "res = {}\n"
        "for B in (1, 9, 64):\n"
        "    H = 32 >> (seg - 1)\n"
        "    for rp in synth.WIDTHS:\n"
        "        C = synth.active_channels(rp, synth.BASE_CHANNELS[seg - 1])\n"
        "        g = np.random.default_rng(700 + seg + B)\n"
        "        x = synth.round_bf16(np.abs(g.standard_normal((B, H, H, C), dtype=np.float32)))\n"
        "        xd = torch.from_numpy(x).to(torch.bfloat16).cuda()\n"
        "        for r in (0.25, 0.5):\n"
        "            o = net.forward(seg, xd, rp, r)\n"
        "            res[f'{B}_{rp}_{r}'] = (o.view(torch.int16) if o.dtype == torch.bfloat16 else o.view(torch.int32)).cpu().numpy()\n"
        "np.savez(sys.argv[1], **res)\n"
    )
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with tempfile.TemporaryDirectory() as d:
        out = {}
        for name, extra in (("fused", {"SLIM_FUSED_SEGS": "14"}), ("layers", {"SLIM_NO_FUSED": "1"})):
            p = subprocess.run([sys.executable, "-c", code, os.path.join(d, name + ".npz")],
                               env=dict(os.environ, **extra), capture_output=True, text=True, timeout=600, cwd=root)
            assert p.returncode == 0, p.stderr[-3000:]
            out[name] = dict(np.load(os.path.join(d, name + ".npz")))
        bad = [k for k in out["fused"] if not np.array_equal(out["fused"][k], out["layers"][k])]
        assert not bad, f"fused != per-layer for {bad[:8]} ({len(bad)} of {len(out['fused'])})"
    # the fused result against the oracle (one configuration per segment)
    ref = oracle.Model(synth.make_weights(), synth.make_bn())
    H = 32 >> (seg - 1)
    C = synth.active_channels(0.5, synth.BASE_CHANNELS[seg - 1])
    g = np.random.default_rng(700 + seg + 9)
    x = synth.round_bf16(np.abs(g.standard_normal((9, H, H, C), dtype=np.float32)))
    got = out["fused"]["9_0.5_0.25"]
    got = got.view(np.float32) if seg == 3 else (got.astype(np.int32).astype(np.uint32) << 16).view(np.float32)
    _check(got[:3], ref.segment(seg, x[:3], 0.5, 0.25), TAU_BF16, f"fused seg{seg}")


@pytest.mark.parametrize("blocks", [(1, 1, 1, 1), (2, 1, 1, 3)])
def test_other_depths(blocks):
    """BasicBlocks per segment other than (2, 2, 2, 2): with one block in segment 3 its only block is the
    down-sampling one, so the network's last conv carries the projection and cannot pool in its
    epilogue (the head pools); chain and segment 3 within tolerance of the oracle."""
    w = synth.make_weights(blocks=blocks)
    bn = synth.make_bn(blocks=blocks)
    n = slim.SlimNet(w, bn, max_batch=16, blocks_per_seg=blocks)
    oref = oracle.Model(w, bn, blocks=blocks)
    x = synth.make_images(9, offset=43)
    tup = (0.5, 1.0, 0.25, 0.75)
    xd = torch.from_numpy(x).to(torch.bfloat16).cuda()
    got = n.forward_chain(xd, tup).cpu().numpy()
    err = oracle.per_image_rel_err(got, oref.chain(x, tup))
    assert err.max() <= TAU_BF16, err.max()
    n.close()


def test_tile_flags_bitwise(tmp_path):
    """Opt-in tile-granular dependencies between a segment's halo convs (SLIM_TILE_FLAGS=1: block 1's convs
    wait per tile on counters the previous conv releases after each tile's TMA store, instead of on the
    whole previous grid): every segment output bitwise equal to the default PDL ordering."""
    one, two = _seg123_outputs_under_env(tmp_path, [dict(SLIM_TILE_FLAGS="0"), dict(SLIM_TILE_FLAGS="1")])
    for k in one.files:
        assert np.array_equal(one[k], two[k]), k


def test_fp32_split_k_batch_independence_bitwise(net32):
    """FP32 mode's split-K (under-filled layers of segments 2-3: K ranges per split, partials reduced in
    split order) picks its split count from the layer shape and max_batch only, so an image's logits are
    bitwise the same in a batch of 1, 7 or 16 (max_batch 64: segments 2-3 split)."""
    x = synth.make_images(16, offset=23)
    tup = (1.0, 0.5, 1.0, 0.25)
    full = net32.forward_chain(_dev(x, torch.float32), tup).cpu().numpy()
    for B in (1, 7):
        part = net32.forward_chain(_dev(x[:B], torch.float32), tup).cpu().numpy()
        assert np.array_equal(part, full[:B]), B


def test_halo_tile_order_bitwise(tmp_path):
    """N-fastest tile order (SLIM_HALO_NFAST=1; the n_tiles tiles of an M tile on neighbouring CTAs), with
    and without the 2-SM pairing: every segment 1-3 output bitwise the default order's."""
    base, nf, nfp = _seg123_outputs_under_env(tmp_path, [dict(SLIM_HALO_NFAST="0", SLIM_HALO_PAIR="0"),
                                                         dict(SLIM_HALO_NFAST="1", SLIM_HALO_PAIR="0"),
                                                         dict(SLIM_HALO_NFAST="1", SLIM_HALO_PAIR="1")])
    for k in base.files:
        assert np.array_equal(base[k], nf[k]), k
        assert np.array_equal(base[k], nfp[k]), k
