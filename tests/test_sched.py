"""Alg. 1 greedy segment-slim scheduler -- the
native decision engine (slim_sched_*) on CPU (host only, no GPU needed).

Pins: each line of Alg. 1 by a hand-built case (FIFO head-key batching l.3-4, best fit
l.5/l.11-12, CANLOAD's VRAM and utilisation gates l.13-20, requeue to the front l.9,
scale-up P:49, t_last update l.10, UNLOADERLOOP l.21-25), and a randomized equivalence
against `RefAlg1`, a plain Python transcription of Alg. 1 written here from the paper.
"""
import numpy as np
import pytest

import paper_2510_09018_b200 as slim

W4 = (0.25, 0.5, 0.75, 1.0)


@pytest.fixture(scope="module")
def cfg():
    return slim.default_config()


def seg_bytes(cfg, s, w):
    return slim.slim_segment_bytes(cfg, s, w, w)


def req(i, s, w, wp=0.0):
    return (i, s, w, wp if s else 0.0, 1000 + i)


def test_fifo_head_key_batching(cfg):
    S = slim.Scheduler(cfg, B_max=3)
    S.enqueue([req(0, 1, 0.5, 1.0), req(1, 0, 0.25), req(2, 1, 0.5, 1.0), req(3, 1, 0.5, 0.25),
               req(4, 1, 0.5, 1.0), req(5, 1, 0.5, 1.0)])
    a = S.next(0.0)
    assert a["kind"] == "run" and a["n_loaded"] == 1
    assert (a["seg"], a["w_req"], a["w_prev"]) == (1, 0.5, 1.0)
    assert list(a["ids"]) == [0, 2, 4] and list(a["slots"]) == [1000, 1002, 1004]   # B_max=3, FIFO
    b = S.next(0.0)   # the rest keeps its order: head is now request 1 (seg 0)
    assert b["kind"] == "run" and list(b["ids"]) == [1]
    c = S.next(0.0)   # the first instance (seg 1, 0.5) is busy -> another one is loaded for key (1, .5, .25)
    assert list(c["ids"]) == [3] and c["n_loaded"] == 1 and c["inst"] not in (a["inst"], b["inst"])
    S.complete(a["inst"], 1.0)
    d = S.next(1.0)   # request 5 reuses the now-free first instance (best fit, no load)
    assert list(d["ids"]) == [5] and d["inst"] == a["inst"] and d["n_loaded"] == 0
    assert S.next(1.0)["kind"] == "idle"


def test_best_fit_smallest_width_at_least_requested(cfg):
    S = slim.Scheduler(cfg, B_max=8)
    ids = {}
    for w in (1.0, 0.5):   # instances of seg 2 at widths 1.0 and 0.5 (the first busy while the second loads)
        S.enqueue([req(int(w * 100), 2, w, w)])
        a = S.next(0.0)
        assert a["n_loaded"] == 1
        ids[w] = a["inst"]
    for i in ids.values():
        S.complete(i, 0.0)
    S.enqueue([req(7, 2, 0.25, 0.5)])
    a = S.next(0.0)
    assert a["inst"] == ids[0.5] and a["inst_w"] == 0.5 and a["w_req"] == 0.25 and a["n_loaded"] == 0
    S.enqueue([req(8, 2, 0.75, 0.5)])
    b = S.next(0.0)   # 0.5 is busy and too narrow anyway: 1.0 is the best fit
    assert b["inst"] == ids[1.0] and b["inst_w"] == 1.0
    S.enqueue([req(9, 2, 0.25, 0.5)])
    c = S.next(0.0)   # both busy -> CANLOAD a new instance at the requested width
    assert c["n_loaded"] == 1 and c["inst_w"] == 0.25


def test_canload_vram_cap_and_requeue_to_front(cfg):
    b3 = seg_bytes(cfg, 3, 1.0)
    S = slim.Scheduler(cfg, B_max=2, M_max_bytes=float(b3 + 1000))
    S.enqueue([req(0, 3, 1.0, 1.0), req(1, 3, 1.0, 1.0), req(2, 0, 0.5), req(3, 3, 1.0, 1.0)])
    a = S.next(0.0)
    assert a["kind"] == "run" and list(a["ids"]) == [0, 1]
    # seg 0 at 0.5 would exceed M_max next to the live seg-3 instance: requeue (l.9)
    r = S.next(0.0, vram_external=0)
    assert r["kind"] == "requeue" and r["batch"] == 1 and S.queue_len() == 2
    # the requeued batch is at the FRONT: head is still request 2
    S.complete(a["inst"], 0.5)
    S.unload_idle(10.0)   # t_idle = 1 s default -> the seg-3 instance goes, VRAM frees
    assert S.instances() == []
    c = S.next(10.0)
    assert c["kind"] == "run" and list(c["ids"]) == [2]
    # external usage counts against the cap too
    S2 = slim.Scheduler(cfg, M_max_bytes=float(b3 + 1000))
    S2.enqueue([req(0, 3, 1.0, 1.0)])
    assert S2.next(0.0, vram_external=2000)["kind"] == "requeue"
    assert S2.next(0.0, vram_external=0)["kind"] == "run"


def test_canload_utilisation_gate(cfg):
    S = slim.Scheduler(cfg, U_blk=0.9)
    S.enqueue([req(0, 0, 1.0)])
    assert S.next(0.0, util=0.95)["kind"] == "requeue"
    assert S.next(0.0, util=0.90)["kind"] == "requeue"     # u >= U_blk blocks (l.18)
    a = S.next(0.0, util=0.5)
    assert a["kind"] == "run"
    S.complete(a["inst"], 0.1)
    S.enqueue([req(1, 0, 1.0)])
    assert S.next(0.2, util=0.99)["kind"] == "run"          # a free instance needs no CANLOAD
    S.enqueue([req(2, 0, 0.5)])
    assert S.next(0.2, util=-1.0)["kind"] == "run"          # no utilisation sample: not gated


def test_scale_up_by_n_new_when_queue_reaches_q_th(cfg):
    S = slim.Scheduler(cfg, B_max=4, Q_th=10, N_new=3)
    S.enqueue([req(i, 1, 0.75, 0.75) for i in range(9)])
    a = S.next(0.0)
    assert a["n_loaded"] == 1                    # 9 < Q_th: one instance
    S.enqueue([req(100 + i, 1, 0.25, 0.5) for i in range(12)])
    S.complete(a["inst"], 0.0)
    S.next(0.0)   # key (1,.75,.75): 5 left, free instance reused
    S.next(0.0)   # 1 left, instance busy -> 1 new (1 < Q_th)
    b = S.next(0.0)   # key (1,.25,.5): 12 queued >= Q_th -> N_new = 3 instances
    assert (b["w_req"], b["n_loaded"]) == (0.25, 3)
    assert sum(1 for i in S.instances() if i["w"] == 0.25) == 3
    c = S.next(0.0)
    assert c["n_loaded"] == 0 and c["inst"] != b["inst"]   # the scale-up instances serve the next batches
    # the VRAM cap bounds a scale-up
    one = seg_bytes(cfg, 2, 1.0)
    S2 = slim.Scheduler(cfg, B_max=1, Q_th=2, N_new=4, M_max_bytes=2.5 * one)
    S2.enqueue([req(i, 2, 1.0, 1.0) for i in range(5)])
    assert S2.next(0.0)["n_loaded"] == 2


def test_unloader_idle_time_and_t_last(cfg):
    S = slim.Scheduler(cfg, t_idle_s=2.0)
    S.enqueue([req(0, 0, 0.25), req(1, 1, 0.5, 0.25)])
    a = S.next(0.0)
    b = S.next(0.0)
    S.complete(a["inst"], 1.0)
    assert S.unload_idle(2.5) == []             # idle 1.5 s < t_idle; b is busy
    assert S.unload_idle(3.0) == [a["inst"]]    # idle 2.0 s >= t_idle (l.24)
    assert S.unload_idle(100.0) == []           # busy instances are never unloaded
    S.complete(b["inst"], 50.0)
    assert [i["t_last"] for i in S.instances()] == [50.0]
    assert S.unload_idle(52.0) == [b["inst"]]


def test_invalid_keys_rejected_and_queue_unchanged(cfg):
    S = slim.Scheduler(cfg)
    S.enqueue([req(0, 0, 0.5)])
    with pytest.raises(slim.SlimError):
        S.enqueue([req(1, 0, 0.5), req(2, 1, 0.3, 0.5)])   # 0.3 not in the width set
    with pytest.raises(slim.SlimError):
        S.enqueue([req(3, 4, 0.5)])
    assert S.queue_len() == 1
    with pytest.raises(slim.SlimError):
        S.complete(12345, 0.0)
    with pytest.raises(slim.SlimError):
        slim.Scheduler(cfg, B_max=0)


class RefAlg1:
    """Alg. 1 transcribed line by line, with the readings of DESIGN.md R17."""

    def __init__(self, cfg, B_max, M_max, U_blk, t_idle, Q_th, N_new):
        self.cfg, self.B_max, self.M_max, self.U_blk = cfg, B_max, M_max, U_blk
        self.t_idle, self.Q_th, self.N_new = t_idle, Q_th, N_new
        self.Q, self.I, self.nid = [], [], 0

    def key(self, q):
        return (q[1], q[2], q[3] if q[1] else 0.0)

    def canload(self, s, w, ext, u):
        b = slim.slim_segment_bytes(self.cfg, s, w, w)
        if ext + sum(i["bytes"] for i in self.I) + b > self.M_max:
            return None
        if u >= 0 and u >= self.U_blk:
            return None
        return b

    def next(self, now, u, ext):
        if not self.Q:
            return ("idle",)
        k = self.key(self.Q[0])
        B = [q for q in self.Q if self.key(q) == k][:self.B_max]
        n_key = sum(1 for q in self.Q if self.key(q) == k)
        rest = [q for q in self.Q if q not in B]
        free = [i for i in self.I if not i["busy"] and i["seg"] == k[0] and i["w"] >= k[1]]
        inst, loaded = (min(free, key=lambda i: i["w"]) if free else None), 0
        if inst is None:
            for _ in range(self.N_new if n_key >= self.Q_th else 1):
                b = self.canload(k[0], k[1], ext, u)
                if b is None:
                    break
                self.I.append(dict(id=self.nid, seg=k[0], w=k[1], busy=False, t_last=now, bytes=b))
                self.nid += 1
                loaded += 1
            if loaded:
                inst = self.I[len(self.I) - loaded]
        if inst is None:
            self.Q = B + rest
            return ("requeue", len(B))
        inst["busy"], inst["t_last"] = True, now
        self.Q = rest
        return ("run", inst["id"], tuple(q[0] for q in B), loaded)

    def complete(self, iid, now):
        for i in self.I:
            if i["id"] == iid:
                i["busy"], i["t_last"] = False, now

    def unload(self, now):
        gone = [i["id"] for i in self.I if not i["busy"] and now - i["t_last"] >= self.t_idle]
        self.I = [i for i in self.I if i["id"] not in gone]
        return gone


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5, 6, 7, 8])
def test_randomized_equivalence_with_alg1_transcription(cfg, seed):
    g = np.random.default_rng(seed)
    knobs = dict(B_max=int(g.integers(1, 6)), M_max_bytes=float(g.uniform(2e6, 4e7)), U_blk=0.8, t_idle_s=0.5,
                 Q_th=int(g.integers(2, 8)), N_new=int(g.integers(1, 4)))
    S = slim.Scheduler(cfg, **knobs)
    R = RefAlg1(cfg, knobs["B_max"], knobs["M_max_bytes"], 0.8, 0.5, knobs["Q_th"], knobs["N_new"])
    now, rid, busy = 0.0, 0, []
    for _ in range(400):
        op = g.random()
        now += float(g.uniform(0, 0.1))
        if op < 0.35:
            reqs = []
            for _ in range(int(g.integers(1, 5))):
                s = int(g.integers(0, 4))
                reqs.append((rid, s, float(g.choice(W4)), float(g.choice(W4)) if s else 0.0, rid))
                rid += 1
            S.enqueue(reqs, now)
            R.Q += reqs
        elif op < 0.75:
            u = float(g.choice([-1.0, 0.3, 0.85]))
            ext = int(g.integers(0, 3)) * 1_000_000
            a, b = S.next(now, u, ext), R.next(now, u, ext)
            assert a["kind"] == b[0]
            if b[0] == "run":
                assert (a["inst"], tuple(int(x) for x in a["ids"]), a["n_loaded"]) == b[1:]
                busy.append(a["inst"])
            elif b[0] == "requeue":
                assert a["batch"] == b[1]
        elif op < 0.92 and busy:
            iid = busy.pop(int(g.integers(0, len(busy))))
            S.complete(iid, now)
            R.complete(iid, now)
        else:
            assert S.unload_idle(now) == R.unload(now)
        assert S.queue_len() == len(R.Q)
        assert [(i["id"], i["busy"]) for i in S.instances()] == [(i["id"], i["busy"]) for i in R.I]
