"""The exact configuration bench.py times (VERDICT r01 next #1d): bench.Cfg2Step built from bench.py's
default arguments -- max_batch = 128, per-width SM shares ("auto"), CUDA-graph replay, the four width
instances on four concurrent streams -- run for a few steps; sampled logits of every width against
the fp64 oracle (north_star tolerance), and the concurrent step bit-identical to each width's chain
run alone on all SMs (the shares only move tiles between CTAs)."""
import numpy as np
import pytest
import torch

import bench
import oracle
import synth

pytestmark = pytest.mark.gpu

TAU_BF16 = 2e-2


def test_bench_cfg2_step_matches_oracle():
    args = bench.build_parser().parse_args([])
    assert args.batch == 128 and args.sm_share == "auto" and not args.no_graph and not args.sequential
    dev = torch.device("cuda", 0)
    step = bench.Cfg2Step(args, dev)
    assert step.net.cfg.max_batch == 128
    assert len(set(step.streams.values())) == 4
    for _ in range(3):
        step.step()
    torch.cuda.synchronize()
    got = {r: step.logits[r].cpu().numpy().copy() for r in step.widths}
    ref = oracle.Model(synth.make_weights(), synth.make_bn())
    g = np.random.default_rng(128)
    for r in step.widths:
        idx = np.sort(g.choice(step.B, 6, replace=False))
        idx[-1] = step.B - 1                                   # the last image of the batch
        x = synth.make_images(step.B, offset=step.image_offsets[r])[idx]
        exp = ref.chain(x, (r,) * 4)
        err = oracle.per_image_rel_err(got[r][idx], exp)
        assert np.isfinite(got[r]).all()
        assert err.max() <= TAU_BF16, (r, err.max())
    # the same chains alone, all SMs, eager: bitwise equal to the concurrent graph-replayed step
    step.set_shares({r: 1.0 for r in step.widths})
    for r in step.widths:
        step.chain(r, step.stream)
        torch.cuda.synchronize()
        assert np.array_equal(step.logits[r].cpu().numpy(), got[r]), r
    step.net.close()
