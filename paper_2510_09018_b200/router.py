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

All ranks call `route()` with the same seed and obtain identical assignments.
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
POLICIES = ("random", "slim", "table_rr")


def route(n: int, world: int, policy: str = "random", seed: int = 2510_09018):
    """Assign n requests: returns (device[n] int, tuple_index[n] int into TABLE_TUPLES, group[n] int).

    Deterministic in (n, world, policy, seed): identical on every rank.
    """
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
