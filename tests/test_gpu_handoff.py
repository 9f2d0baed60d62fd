"""GPU: segment-routed execution with activation hand-off between (emulated) ranks
 gives every request exactly the logits of its own chain (bit-exact:
the kernels are batch-independent and the hand-off moves bytes).  All ranks run in one
process on the one GPU; the collective is replaced by the in-process all-to-all of
handoff.run_local (the gloo test covers the collective's split sizes)."""
import numpy as np
import pytest
import torch

import synth
import paper_2510_09018_b200 as slim
from paper_2510_09018_b200 import handoff

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def net():
    n = slim.SlimNet(synth.make_weights(), synth.make_bn(), max_batch=128)
    yield n
    n.close()


@pytest.mark.parametrize("world,policy,lanes", [(2, "random", 1), (3, "random", 4), (2, "pipeline", 1),
                                               (4, "sticky", 8)])
def test_handoff_matches_chain(net, world, policy, lanes):
    n = 150
    g = np.random.default_rng(world)
    tuples = np.asarray(synth.TABLE_TUPLES, np.float32)[g.integers(0, 8, n)]
    x = torch.from_numpy(synth.make_images(n, offset=world)).to(torch.bfloat16).cuda()
    dev = handoff.plan_segments(n, world, policy, seed=world)
    exs = [handoff.HandoffExecutor(net, n, r, world, B_max=64, lanes=lanes) for r in range(world)]
    got = handoff.run_local(exs, x, tuples, dev)
    exp = torch.empty_like(got)
    for t in {tuple(map(float, r)) for r in tuples}:
        idx = torch.from_numpy(np.nonzero((tuples == np.asarray(t, np.float32)).all(1))[0]).cuda()
        exp[idx] = net.forward_chain(x[idx].contiguous(), t)
    torch.testing.assert_close(got, exp, rtol=0, atol=0)
    moved = int((dev[:, 1:] != dev[:, :-1]).sum())
    assert sum(e.stats["sent_rows"] for e in exs) == moved == sum(e.stats["recv_rows"] for e in exs)
