"""Host-side policies on CPU: the bench's SM-share rule, the hand-off plan at world 1, and the
Alg. 1 scheduler with a universal width set (keys validated against the configured widths)."""
import numpy as np
import pytest

import bench
import paper_2510_09018_b200 as slim
from paper_2510_09018_b200 import handoff


def test_sm_share_rule():
    w = (0.25, 0.5, 0.75, 1.0)
    auto = bench.sm_shares(w, "auto")
    assert [round(auto[r], 6) for r in w] == [0.2, 0.3, 0.4, 0.5]   # 0.1 + 0.4 r
    assert all(v == 1.0 for v in bench.sm_shares(w, "none").values())
    assert bench.sm_shares(w, "0.1,0.2,0.3,0.4") == {0.25: 0.1, 0.5: 0.2, 0.75: 0.3, 1.0: 0.4}
    with pytest.raises(AssertionError):
        bench.sm_shares(w, "0.1,0.2")
    assert 0 < min(bench.sm_shares((0.01, 1.0), "auto").values()) and max(bench.sm_shares((1.0,), "auto").values()) <= 1


def test_handoff_world_one_has_no_exchange():
    dev = handoff.plan_segments(50, 1, "random")
    assert (dev == 0).all()
    for s in range(3):
        send, recv = handoff.exchange_lists(dev, s, 0, 1)
        assert len(send) == len(recv) == 1 and len(send[0]) == len(recv[0]) == 0


def test_scheduler_with_universal_widths():
    cfg = slim.default_config(widths=(0.25, 0.3, 0.6, 0.9, 1.0))
    S = slim.Scheduler(cfg, B_max=4)
    S.enqueue([(0, 1, 0.3, 0.9, 0), (1, 1, 0.3, 0.9, 1), (2, 0, 0.6, 0.0, 2)])
    a = S.next(0.0)
    assert a["kind"] == "run" and abs(a["w_req"] - 0.3) < 1e-6 and list(a["ids"]) == [0, 1]
    with pytest.raises(slim.SlimError):
        S.enqueue([(3, 1, 0.5, 0.9, 3)])        # 0.5 is not a configured width here
    b = S.next(0.0)
    assert abs(b["w_req"] - 0.6) < 1e-6 and b["n_loaded"] == 1
    # CANLOAD's bytes follow the universal channel counts (ceil(r*C))
    assert slim.slim_segment_bytes(cfg, 1, 0.3, 0.3) < slim.slim_segment_bytes(cfg, 1, 0.6, 0.6)
    assert slim.slim_segment_bytes(cfg, 1, 0.5, 0.5) == 0   # not configured
