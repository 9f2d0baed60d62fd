"""Run a few chains of the bench workload for ncu captures (no timing is reported from here).

    python tools/profile_chain.py --widths 1.0 --batch 128 --reps 2
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_2510_09018_b200 as slim  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--widths", type=float, nargs="+", default=[1.0])
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--norm", default="bn")
    a = ap.parse_args()
    net = slim.SlimNet(synth.make_weights(), synth.make_bn(), max_batch=a.batch, norm=a.norm)
    x = torch.from_numpy(synth.make_images(a.batch)).to(torch.bfloat16).cuda()
    for _ in range(a.reps):
        for r in a.widths:
            net.forward_chain(x, (r,) * 4)
    torch.cuda.synchronize()
    print("done", slim.slim_launch_count(net.ctx), "launches")


if __name__ == "__main__":
    main()
