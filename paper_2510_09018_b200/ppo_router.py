"""Frozen-policy forward of the paper's factored PPO router (Eqs. 1-7;
SURVEY §8(f) NEXT-3) -- host-side control, numpy float64.

PPO *training* is out of scope (the reward weights alpha..delta and the network sizes are
unstated); what the serving path needs is the policy's forward pass on the
gathered telemetry, replicated on every rank:

* Eq. 1  state  s_t = [q_fifo, c_done, (q_i, P_i, U_i) for each of N servers]
* Eq. 3  (l_srv, l_w, l_g, V) = MLP_theta(s_t)   -- one shared trunk, four linear heads
* Eq. 4  pi(a|s) = pi_srv * pi_w * pi_g, each Cat(softmax(l))
* Eq. 5  server head mixed with uniform exploration:
         pi~_srv = (1 - eps_t) pi_srv + eps_t / N,
         eps_t = max(eps_min, eps_max + t / T_dec * (eps_min - eps_max))
* Eq. 6  log pi~(a|s) = log pi~_srv + log pi_w + log pi_g
* Eq. 7  reward r_t = alpha p_acc - beta L_t - gamma E_t - delta Var(U/100) + b_t (for logging)

Readings (R18): trunk = two tanh layers of 64 units (unstated); the frozen
weights are a seeded initialisation passed in by the caller (no trained checkpoint
exists); utilisation enters the state as a fraction (R13), the imbalance term of Eq. 7
then uses U directly (Var(U_pct/100) = Var(U_frac)).
"""
from __future__ import annotations

import numpy as np


def state_vector(q_fifo: float, c_done: float, per_server) -> np.ndarray:
    """Eq. 1: per_server = iterable of (q_i, P_i, U_i)."""
    rows = [float(v) for srv in per_server for v in srv]
    return np.asarray([float(q_fifo), float(c_done)] + rows, np.float64)


def state_from_telemetry(records: np.ndarray, q_fifo: float, c_done: float) -> np.ndarray:
    """Eq. 1 from the all-gathered float32[N, 8] telemetry records (telemetry.FIELDS:
    queue_len, power_W, util_frac, ...)."""
    r = np.asarray(records, np.float64)
    return state_vector(q_fifo, c_done, r[:, :3])


def log_softmax(l: np.ndarray) -> np.ndarray:
    m = l.max(axis=-1, keepdims=True)
    return l - m - np.log(np.exp(l - m).sum(axis=-1, keepdims=True))


def epsilon(t: float, eps_min: float, eps_max: float, t_dec: float) -> float:
    """Eq. 5 schedule: linear decay from eps_max to eps_min over T_dec steps, clamped at eps_min."""
    return max(eps_min, eps_max + t / t_dec * (eps_min - eps_max))


class FrozenRouter:
    """params: dict W1 [H, D], b1 [H], W2 [H, H], b2 [H], and per head h in (srv, w, g, v):
    W_h [n_h, H], b_h [n_h] (n_v = 1).  widths / groups label the w and g categories."""

    def __init__(self, params: dict, widths=(0.25, 0.5, 0.75, 1.0), groups=(16, 64, 256),
                 eps_min: float = 0.05, eps_max: float = 0.5, t_dec: float = 10_000.0):
        self.p = {k: np.asarray(v, np.float64) for k, v in params.items()}
        self.widths, self.groups = tuple(widths), tuple(groups)
        self.eps_min, self.eps_max, self.t_dec = eps_min, eps_max, t_dec
        assert self.p["W_w"].shape[0] == len(self.widths) and self.p["W_g"].shape[0] == len(self.groups)

    @staticmethod
    def init(n_servers: int, hidden: int = 64, n_widths: int = 4, n_groups: int = 3, seed: int = 2510_09018):
        """Seeded initialisation (the frozen weights when no trained checkpoint exists)."""
        g = np.random.Generator(np.random.PCG64([seed, 91]))
        D = 2 + 3 * n_servers
        u = lambda o, i: g.uniform(-1.0, 1.0, (o, i)) / np.sqrt(i)
        p = dict(W1=u(hidden, D), b1=np.zeros(hidden), W2=u(hidden, hidden), b2=np.zeros(hidden))
        for h, n in (("srv", n_servers), ("w", n_widths), ("g", n_groups), ("v", 1)):
            p[f"W_{h}"], p[f"b_{h}"] = u(n, hidden), np.zeros(n)
        return p

    def forward(self, s: np.ndarray):
        """Eq. 3: returns (l_srv, l_w, l_g, V)."""
        p = self.p
        h = np.tanh(p["W1"] @ s + p["b1"])
        h = np.tanh(p["W2"] @ h + p["b2"])
        heads = [p[f"W_{k}"] @ h + p[f"b_{k}"] for k in ("srv", "w", "g", "v")]
        return heads[0], heads[1], heads[2], float(heads[3][0])

    def probs(self, s: np.ndarray, t: float):
        """Eqs. 4-5: (pi~_srv, pi_w, pi_g) for state s at step t."""
        l_srv, l_w, l_g, _ = self.forward(s)
        eps = epsilon(t, self.eps_min, self.eps_max, self.t_dec)
        p_srv = (1.0 - eps) * np.exp(log_softmax(l_srv)) + eps / l_srv.shape[0]
        return p_srv, np.exp(log_softmax(l_w)), np.exp(log_softmax(l_g))

    def log_prob(self, s: np.ndarray, t: float, a) -> float:
        """Eq. 6: log pi~(a|s) = log pi~_srv(a_srv) + log pi_w(a_w) + log pi_g(a_g)."""
        p_srv, p_w, p_g = self.probs(s, t)
        return float(np.log(p_srv[a[0]]) + np.log(p_w[a[1]]) + np.log(p_g[a[2]]))

    def act(self, s: np.ndarray, t: float, rng: np.random.Generator, greedy: bool = False):
        """Sample a_t = (srv, w, g) (Eq. 2).  Returns (srv index, width, group size, log-prob)."""
        p_srv, p_w, p_g = self.probs(s, t)
        if greedy:
            a = (int(np.argmax(p_srv)), int(np.argmax(p_w)), int(np.argmax(p_g)))
        else:
            a = (int(rng.choice(len(p_srv), p=p_srv)), int(rng.choice(len(p_w), p=p_w)),
                 int(rng.choice(len(p_g), p=p_g)))
        lp = float(np.log(p_srv[a[0]]) + np.log(p_w[a[1]]) + np.log(p_g[a[2]]))
        return a[0], self.widths[a[1]], self.groups[a[2]], lp


def reward(p_acc: float, latency_s: float, mean_power_w: float, utils, alpha: float, beta: float,
           gamma: float, delta: float, bonus: float = 0.0) -> float:
    """Eq. 7 with E_t = mean power x L_t and the variance of the normalised utilisations."""
    energy = mean_power_w * latency_s
    return alpha * p_acc - beta * latency_s - gamma * energy - delta * float(np.var(np.asarray(utils, np.float64))) + bonus
