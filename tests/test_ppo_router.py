"""Frozen PPO router forward (Eqs. 1-7) on CPU.

Pins: the MLP against torch.nn float64 modules (library), Eq. 5's mixture at eps = 0 / 1
and its schedule's clamp, Eq. 6 against a direct product of the three categorical
probabilities, sampling frequencies against the probabilities (seeded), Eq. 1's layout
from telemetry records, and Eq. 7 on hand-computed numbers."""
import math

import numpy as np
import torch

from paper_2510_09018_b200 import ppo_router as pr


def _router(N=4, **kw):
    return pr.FrozenRouter(pr.FrozenRouter.init(N), **kw)


def test_state_vector_layout_eq1():
    rec = np.array([[3, 400.0, 0.5, 0, 0, 0, 0, 0], [7, 500.0, 0.9, 0, 0, 0, 0, 1]], np.float32)
    s = pr.state_from_telemetry(rec, q_fifo=11, c_done=20)
    np.testing.assert_array_equal(s, [11, 20, 3, 400, 0.5, 7, 500, np.float32(0.9)])


def test_mlp_matches_torch_modules():
    r = _router(N=3)
    p = r.p
    s = np.random.default_rng(0).standard_normal(2 + 3 * 3)
    trunk = torch.nn.Sequential(torch.nn.Linear(11, 64), torch.nn.Tanh(), torch.nn.Linear(64, 64), torch.nn.Tanh()).double()
    with torch.no_grad():
        trunk[0].weight.copy_(torch.from_numpy(p["W1"]))
        trunk[0].bias.copy_(torch.from_numpy(p["b1"]))
        trunk[2].weight.copy_(torch.from_numpy(p["W2"]))
        trunk[2].bias.copy_(torch.from_numpy(p["b2"]))
        h = trunk(torch.from_numpy(s))
        got = r.forward(s)
        for i, k in enumerate(("srv", "w", "g")):
            ref = torch.nn.functional.linear(h, torch.from_numpy(p[f"W_{k}"]), torch.from_numpy(p[f"b_{k}"]))
            np.testing.assert_allclose(got[i], ref.numpy(), rtol=1e-12, atol=1e-12)
        v = torch.nn.functional.linear(h, torch.from_numpy(p["W_v"]), torch.from_numpy(p["b_v"]))
        assert abs(got[3] - float(v)) < 1e-12


def test_eq5_mixture_and_schedule():
    r = _router(N=5, eps_min=0.0, eps_max=1.0, t_dec=100.0)
    s = np.linspace(-1, 1, 17)
    l_srv = r.forward(s)[0]
    soft = np.exp(l_srv - l_srv.max()) / np.exp(l_srv - l_srv.max()).sum()
    np.testing.assert_allclose(r.probs(s, 0.0)[0], np.full(5, 0.2), atol=1e-15)      # eps = 1: uniform
    np.testing.assert_allclose(r.probs(s, 100.0)[0], soft, rtol=1e-12)               # eps = 0: softmax
    np.testing.assert_allclose(r.probs(s, 25.0)[0], 0.25 * soft + 0.75 / 5, rtol=1e-12)   # eps_25 = 0.75
    assert pr.epsilon(1e9, 0.05, 0.5, 10.0) == 0.05                                   # clamped at eps_min
    assert abs(pr.epsilon(5.0, 0.05, 0.5, 10.0) - 0.275) < 1e-15
    for p in r.probs(s, 10.0):
        assert abs(p.sum() - 1.0) < 1e-12 and (p > 0).all()


def test_eq6_joint_log_prob_and_sampling():
    r = _router(N=4)
    s = np.array([40.0, 7.0] + [1, 300, 0.3, 5, 500, 0.9, 0, 200, 0.1, 2, 250, 0.5])
    p_srv, p_w, p_g = r.probs(s, 3.0)
    for a in [(0, 0, 0), (3, 2, 1), (1, 3, 2)]:
        assert abs(r.log_prob(s, 3.0, a) - math.log(p_srv[a[0]] * p_w[a[1]] * p_g[a[2]])) < 1e-12
    g = np.random.default_rng(5)
    n = 20000
    counts = np.zeros(4)
    wcount = {w: 0 for w in r.widths}
    for _ in range(n):
        srv, w, grp, lp = r.act(s, 3.0, g)
        counts[srv] += 1
        wcount[w] += 1
        assert grp in r.groups
    assert np.abs(counts / n - p_srv).max() < 0.015
    assert np.abs(np.array([wcount[w] for w in r.widths]) / n - p_w).max() < 0.015
    srv, w, grp, lp = r.act(s, 3.0, g, greedy=True)
    assert srv == int(np.argmax(p_srv)) and w == r.widths[int(np.argmax(p_w))]


def test_replicated_decisions_are_identical():
    """Every rank holds the same frozen weights and seed: identical actions from identical state."""
    s = np.arange(14, dtype=np.float64)
    a = [_router().act(s, 1.0, np.random.default_rng(9)) for _ in range(2)]
    assert a[0] == a[1]


def test_eq7_reward():
    r = pr.reward(p_acc=0.7, latency_s=0.2, mean_power_w=100.0, utils=[0.2, 0.6], alpha=1.0, beta=2.0,
                  gamma=0.01, delta=3.0, bonus=0.5)
    assert abs(r - (0.7 - 0.4 - 0.2 - 3.0 * 0.04 + 0.5)) < 1e-12
