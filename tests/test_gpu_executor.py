"""GPU: the Alg. 1 executor (native scheduler decisions + libslim kernels on per-instance
streams) returns, for every request of a mixed-width
stream, exactly the logits of that request's chain.  Bit-exact: every kernel is
batch-independent (tests/test_gpu_parity.py), so batch composition cannot change a bit."""
import numpy as np
import pytest
import torch

import synth
import paper_2510_09018_b200 as slim
from paper_2510_09018_b200.executor import GreedyExecutor

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def net():
    n = slim.SlimNet(synth.make_weights(), synth.make_bn(), max_batch=256)
    yield n
    n.close()


def _stream(n, seed):
    g = np.random.default_rng(seed)
    tuples = np.asarray(synth.TABLE_TUPLES, np.float32)[g.integers(0, len(synth.TABLE_TUPLES), n)]
    x = torch.from_numpy(synth.make_images(n, offset=seed)).to(torch.bfloat16).cuda()
    return x, tuples


def _expected(net, x, tuples):
    exp = torch.empty(x.shape[0], 100, dtype=torch.float32, device=x.device)
    for t in {tuple(map(float, r)) for r in tuples}:
        idx = torch.from_numpy(np.nonzero((tuples == np.asarray(t, np.float32)).all(1))[0]).cuda()
        exp[idx] = net.forward_chain(x[idx].contiguous(), t)
    return exp


@pytest.mark.parametrize("B_max,Q_th,N_new", [(32, 64, 2), (7, 4, 3), (256, 512, 1)])
def test_executor_matches_per_request_chain(net, B_max, Q_th, N_new):
    x, tuples = _stream(300, 11)
    ex = GreedyExecutor(net, n_max=300, B_max=B_max, Q_th=Q_th, N_new=N_new)
    got = ex.run(x, tuples).clone()
    torch.testing.assert_close(got, _expected(net, x, tuples), rtol=0, atol=0)
    assert ex.stats["batches"] >= 4 * len({tuple(r) for r in tuples[:, :1]})
    assert max(ex.stats["batch_sizes"]) <= B_max
    assert ex.sched.queue_len() == 0 and all(not i["busy"] for i in ex.sched.instances())


def test_executor_vram_cap_serialises_and_offload_reloads(net):
    """M_max admits only ~one instance at a time: batches wait for busy instances (requeue,
    l.9), idle instances are unloaded (t_idle = 0) and their segments offloaded and
    reloaded -- the results do not change."""
    x, tuples = _stream(120, 5)
    big = max(slim.slim_segment_bytes(net.cfg, s, 1.0, 1.0) for s in range(4))
    base = torch.cuda.memory_allocated()
    ex = GreedyExecutor(net, n_max=120, B_max=16, offload=True, t_idle_s=0.0, M_max_bytes=float(1.5 * big),
                        vram_fn=lambda: 0)
    got = ex.run(x, tuples).clone()
    for s in range(4):            # leave the shared net fully loaded for the other tests
        if not net.segment_loaded(s):
            net.load_segment(s)
    torch.testing.assert_close(got, _expected(net, x, tuples), rtol=0, atol=0)
    assert ex.stats["unloaded"] > 0 and ex.stats["seg_reloads"] > 0
    assert torch.cuda.memory_allocated() >= base


@pytest.mark.parametrize("B_max,Q_th,N_new", [(32, 64, 2), (5, 3, 4), (256, 512, 1)])
def test_native_executor_matches_per_request_chain(net, B_max, Q_th, N_new):
    x, tuples = _stream(300, 17)
    ex = slim.NativeExecutor(net, n_max=300, B_max=B_max, Q_th=Q_th, N_new=N_new)
    got = ex.run(x, tuples).clone()
    got2 = ex.run(x, tuples).clone()          # instances persist across runs
    ex.close()
    exp = _expected(net, x, tuples)
    torch.testing.assert_close(got, exp, rtol=0, atol=0)
    torch.testing.assert_close(got2, exp, rtol=0, atol=0)


def test_native_executor_vram_cap_and_unload(net):
    x, tuples = _stream(100, 3)
    big = max(slim.slim_segment_bytes(net.cfg, s, 1.0, 1.0) for s in range(4))
    # one instance's buffers: slab + out (16 rows of the widest activation row) + the widest workspace
    per_inst = 2 * 16 * 32 * 32 * 64 * 2 + max(slim.slim_forward_workspace_bytes(net.ctx, s, 1.0, 1.0, 16)
                                               for s in range(4))
    ex = slim.NativeExecutor(net, n_max=100, B_max=16, t_idle_s=0.0, M_max_bytes=float(1.2 * (big + per_inst)))
    got = ex.run(x, tuples).clone()
    st = ex.stats
    ex.close()
    torch.testing.assert_close(got, _expected(net, x, tuples), rtol=0, atol=0)
    assert st["unloaded"] > 0 and st["batches"] >= 4


def test_native_executor_open_loop_arrivals(net):
    """Open loop (Poisson arrivals): same bits as the closed loop; every request completes after it
    arrives, and requests arriving late cannot finish before they arrive."""
    x, tuples = _stream(200, 23)
    g = np.random.default_rng(4)
    arrivals = np.cumsum(g.exponential(1.0 / 50_000.0, 200))       # ~4 ms trace
    ex = slim.NativeExecutor(net, n_max=200, B_max=32)
    got = ex.run(x, tuples, arrivals=arrivals).clone()
    lat, done = ex.latency.copy(), ex.done.copy()
    with pytest.raises(slim.SlimError):
        ex.run(x, tuples, arrivals=arrivals[::-1].copy())          # arrivals must be ascending
    ex.close()
    torch.testing.assert_close(got, _expected(net, x, tuples), rtol=0, atol=0)
    assert (lat > 0).all() and (done >= arrivals).all()
    assert done.max() >= arrivals[-1]
