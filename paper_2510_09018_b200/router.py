"""Request routing for the multi-device stream (CFG5) -- host-side control.

The paper's router is a factored PPO policy choosing (server, width, micro-batch
group) per scheduled block (Eq. 2).  PPO training is out of
scope (its reward weights alpha..delta are unstated); what the hot path
needs is a *replicated, deterministic* routing decision so that every rank of the
`torchrun` job executes exactly its own requests with no coordinator.  Policies:

* ``random``   -- the paper's baseline: device, width tuple and group drawn
                  uniformly at random (Table III; SPEC random policy).
* ``slim``     -- every request at the slimmest tuple (0.25)^4, round-robin devices
                  (the behaviour the "overfit" PPO converged to, Table IV).
* ``table_rr`` -- round-robin devices, width tuples cycling through Tables I-II.
* ``ppo_frozen`` -- the factored policy itself (Eqs. 1-6, `ppo_router.FrozenRouter`, frozen seeded
                  weights): each action a = (server, width, group g) takes the next g requests of the
                  FIFO; the state (Eq. 1) is built from the telemetry all-gathered one tick earlier,
                  with each server's queue length advanced by what this tick already assigned to it
                  (`route_frozen`).

All ranks call `route()` / `route_frozen()` with the same seed (and the same gathered telemetry) and
obtain identical assignments.
"""
from __future__ import annotations

import numpy as np

# Width tuples of PAPER.md Table I (uniform, l.164) and Table II (mixed, l.172-175).
TABLE_TUPLES = (
    (0.25, 0.25, 0.25, 0.25), (0.5, 0.5, 0.5, 0.5), (0.75, 0.75, 0.75, 0.75), (1.0, 1.0, 1.0, 1.0),
    (1.0, 0.75, 0.5, 0.25), (0.75, 1.0, 0.25, 0.5), (0.5, 0.25, 1.0, 0.75), (0.25, 0.5, 0.75, 1.0),
)
# micro-batch group sizes G for the factored action (knob; the paper gives no values)
GROUPS = (16, 64, 256)
POLICIES = ("random", "slim", "table_rr", "ppo_frozen")
# uniform tuple (w, w, w, w) of a width the frozen policy picks -> its index in TABLE_TUPLES
_UNIFORM = {0.25: 0, 0.5: 1, 0.75: 2, 1.0: 3}


def route(n: int, world: int, policy: str = "random", seed: int = 2510_09018):
    """Assign n requests: returns (device[n] int, tuple_index[n] int into TABLE_TUPLES, group[n] int).

    Deterministic in (n, world, policy, seed): identical on every rank.
    """
    if policy == "ppo_frozen":     # no telemetry yet: the state of an idle cluster at t = 0
        return route_frozen(n, world, np.zeros((world, 8), np.float32), 0, seed=seed)
    if policy not in POLICIES:
        raise ValueError(f"unknown policy {policy!r}; one of {POLICIES}")
    g = np.random.Generator(np.random.PCG64([seed, 77]))
    if policy == "random":
        dev = g.integers(0, world, n)
        tup = g.integers(0, len(TABLE_TUPLES), n)
        grp = np.asarray(GROUPS)[g.integers(0, len(GROUPS), n)]
    elif policy == "slim":
        dev = np.arange(n) % world
        tup = np.zeros(n, np.int64)
        grp = np.full(n, GROUPS[-1])
    else:
        dev = np.arange(n) % world
        tup = (np.arange(n) // world) % len(TABLE_TUPLES)
        grp = np.full(n, GROUPS[-1])
    return dev.astype(np.int64), tup.astype(np.int64), grp.astype(np.int64)


def shard(dev: np.ndarray, rank: int) -> np.ndarray:
    """Indices of the requests this rank executes."""
    return np.nonzero(dev == rank)[0]


_FROZEN = {}


def route_frozen(n: int, world: int, records, t: int, c_done: float = 0.0, seed: int = 2510_09018):
    """Route n FIFO requests with the frozen factored PPO router (Eqs. 1-6).

    records: the all-gathered telemetry float32[world, 8] of the previous tick (telemetry.FIELDS).
    Repeatedly: s = Eq. 1 state (q_fifo = requests still unrouted, c_done, per server (q_i + routed_i,
    P_i, U_i)); a = (srv, w, g) ~ pi~(.|s) at step t (Eqs. 4-5); the next g requests go to srv at the
    uniform tuple (w, w, w, w).  The sampling RNG is seeded by (seed, t): deterministic in
    (n, world, records, t), hence identical on every rank that holds the same gathered records.
    Returns (device[n], tuple_index[n], group[n]) like `route`."""
    from .ppo_router import FrozenRouter, state_vector
    if world not in _FROZEN:
        _FROZEN[world] = FrozenRouter(FrozenRouter.init(world, seed=seed), groups=GROUPS)
    fr = _FROZEN[world]
    rec = np.asarray(records, np.float64).reshape(world, -1)
    g = np.random.Generator(np.random.PCG64([seed, 78, int(t)]))
    dev = np.empty(n, np.int64)
    tup = np.empty(n, np.int64)
    grp = np.empty(n, np.int64)
    routed = np.zeros(world)
    i = 0
    while i < n:
        s = state_vector(n - i, c_done, [(rec[k, 0] + routed[k], rec[k, 1], rec[k, 2]) for k in range(world)])
        srv, w, gsz, _ = fr.act(s, t, g)
        j = min(n, i + gsz)
        dev[i:j], tup[i:j], grp[i:j] = srv, _UNIFORM[w], gsz
        routed[srv] += j - i
        i = j
    return dev, tup, grp
