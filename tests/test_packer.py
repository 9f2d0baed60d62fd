"""Batch packer (Alg. 1 lines 3-4): host-only, no GPU.

Examples from SPEC.md form_batch plus the FIFO/equivalence properties."""
import numpy as np
import pytest

import paper_2510_09018_b200 as slim

CFG = None


def cfg():
    global CFG
    if CFG is None:
        CFG = slim.default_config()
    return CFG


def req(i, seg, wr, wp=0.25):
    return (i, seg, wr, wp, i)


def test_scan_semantics_kkjk():
    # queue keys [k,k,j,k], B_max=8 -> batch of 3 k-requests, then [j]
    q = [req(0, 1, 0.5), req(1, 1, 0.5), req(2, 1, 0.75), req(3, 1, 0.5)]
    descs, order = slim.slim_pack(cfg(), q, 8)
    assert [d["batch"] for d in descs] == [3, 1]
    assert list(order[:3]) == [0, 1, 3] and order[3] == 2
    assert descs[0]["r"] == 0.5 and descs[1]["r"] == 0.75


def test_cap_and_singleton():
    q = [req(i, 2, 1.0) for i in range(10)]
    descs, order = slim.slim_pack(cfg(), q, 4)
    assert [d["batch"] for d in descs] == [4, 4, 2]
    assert list(order) == list(range(10))
    descs, order = slim.slim_pack(cfg(), [req(0, 0, 0.25)], 1)
    assert descs == [dict(seg=0, r_prev=0.25, r=0.25, batch=1, first=0)]


def test_w_prev_is_part_of_the_key_except_seg0():
    q = [req(0, 1, 0.5, 0.25), req(1, 1, 0.5, 1.0), req(2, 0, 0.5, 0.25), req(3, 0, 0.5, 1.0)]
    descs, _ = slim.slim_pack(cfg(), q, 8)
    assert [d["batch"] for d in descs] == [1, 1, 2]


def test_invalid_width_rejected():
    with pytest.raises(slim.SlimError):
        slim.slim_pack(cfg(), [req(0, 1, 0.3)], 8)


def test_random_streams_property():
    """Every batch is key-homogeneous, FIFO inside a key, <= B_max, a permutation overall, and
    equals a brute-force replay of Alg.1's peek-head / form-batch loop."""
    g = np.random.default_rng(0)
    W = (0.25, 0.5, 0.75, 1.0)
    for trial in range(20):
        n = int(g.integers(1, 200))
        B = int(g.integers(1, 17))
        q = [(i, int(g.integers(0, 4)), W[g.integers(0, 4)], W[g.integers(0, 4)], i) for i in range(n)]
        descs, order = slim.slim_pack(cfg(), q, B)
        assert sorted(order.tolist()) == list(range(n))
        key = lambda r: (r[1], r[2], r[3] if r[1] > 0 else None)
        # brute force replay
        queue = list(range(n))
        ref = []
        while queue:
            k = key(q[queue[0]])
            batch = [i for i in queue if key(q[i]) == k][:B]
            ref.append(batch)
            queue = [i for i in queue if i not in batch]
        got = [order[d["first"]:d["first"] + d["batch"]].tolist() for d in descs]
        assert got == ref


@pytest.mark.parametrize("seg", [0, 1, 3])
def test_pack_arrays_equals_pack(seg):
    """The vectorised marshalling (slim_pack_arrays) hands the packer the same requests."""
    g = np.random.default_rng(seg)
    W = (0.25, 0.5, 0.75, 1.0)
    n = 300
    wr = np.asarray(W)[g.integers(0, 4, n)]
    wp = np.asarray(W)[g.integers(0, 4, n)]
    reqs = [(i, seg, float(wr[i]), float(wp[i]) if seg else 0.0, i) for i in range(n)]
    d1, o1 = slim.slim_pack(cfg(), reqs, 64)
    d2, o2 = slim.slim_pack_arrays(cfg(), seg, wr, wp if seg else None, 64)
    assert d1 == d2 and np.array_equal(o1, o2)
    d3, o3 = slim.slim_pack_arrays(cfg(), seg, wr[:0], wp[:0], 64)
    assert d3 == [] and o3.shape == (0,)
