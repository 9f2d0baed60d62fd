"""Golden fixtures under tests/golden/ (each cites its source in its header):

* paper_width_tuples.txt -- Tables I-II of the paper (the width tuples the workloads draw from)
* active_channels.txt    -- c(r, C) = ceil(r*C) written by hand for the paper's width set and
                            three universal widths
* delta_seg01.txt        -- the delta network's closed form on a tiny input, written by
                            tests/golden/make_delta_fixture.py from the formula alone
The paper prints no forward-pass values (its Tables need trained weights and CIFAR-100), so
these are the paper-/mathematics-fixed values available to pin the oracle and the host code."""
import os

import numpy as np
import pytest

import oracle
import synth
import paper_2510_09018_b200 as slim
from paper_2510_09018_b200 import router
from tests.test_oracle_pins import _delta_net

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _rows(name):
    return [l.split() for l in open(os.path.join(G, name)) if l.strip() and not l.startswith("#")]


def test_width_tuples_are_the_papers():
    tup = [tuple(float(v) for v in r) for r in _rows("paper_width_tuples.txt")]
    assert len(tup) == 8
    assert [tuple(t) for t in synth.TABLE_TUPLES] == tup
    assert [tuple(t) for t in router.TABLE_TUPLES] == tup


def test_active_channels_table():
    for r, *cs in _rows("active_channels.txt"):
        for C, c in zip((64, 128, 256, 512), cs):
            assert oracle.channels(float(r), C) == int(c), (r, C)
            assert synth.active_channels(float(r), C) == int(c), (r, C)
            assert slim.slim_channels(float(r), C) == int(c), (r, C)


def test_delta_network_closed_form_fixture():
    d = {l.split()[0]: np.array([float(v) for v in l.split()[1:]]) for l in open(os.path.join(G, "delta_seg01.txt"))
         if not l.startswith("#")}
    x = d["x"].reshape(2, 4, 4, 3)
    m = oracle.Model(*_delta_net())
    for r in (0.25, 1.0):
        h0 = m.segment(0, x, None, r)
        assert h0.shape[-1] == oracle.channels(r, 64)
        np.testing.assert_allclose(h0[..., :3].ravel(), d["seg0"], rtol=1e-12, atol=1e-12)
        assert not h0[..., 3:].any()
        h1 = m.segment(1, h0, r, 0.5)
        np.testing.assert_allclose(h1[..., :3].ravel(), d["seg1"], rtol=1e-12, atol=1e-12)
        assert not h1[..., 3:].any()
