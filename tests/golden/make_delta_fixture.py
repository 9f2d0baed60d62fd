"""Writes delta_seg01.txt: the closed form of the delta network (SURVEY §8(c) "Closed form";
tests/test_oracle_pins.py::_delta_net) on a tiny input, computed from the formula alone -- no
oracle/ and no CUDA call: with centre-tap identity kernels and BN folding to the identity, the
stem is relu(x) on the 3 image channels, each stride-1 BasicBlock maps h >= 0 to 2h, and the
down-sampling block of segment s >= 1 maps h to 2 * h[::2, ::2] (conv path h + projection h).

    seg0 output = 4 * relu(x)            (stem, then two blocks)
    seg1 output = 4 * seg0[::2, ::2]     (down-sampling block, then one block)

    python tests/golden/make_delta_fixture.py
"""
import os

import numpy as np

x = (np.arange(2 * 4 * 4 * 3, dtype=np.float64).reshape(2, 4, 4, 3) % 7 - 3) / 2.0   # exact halves
seg0 = 4.0 * np.maximum(x, 0.0)
seg1 = 4.0 * seg0[:, ::2, ::2, :]
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "delta_seg01.txt"), "w") as f:
    f.write("# delta network closed form, tests/golden/make_delta_fixture.py; shapes x/seg0 [2,4,4,3], seg1 [2,2,2,3]\n")
    for name, a in (("x", x), ("seg0", seg0), ("seg1", seg1)):
        f.write(name + " " + " ".join(f"{v:g}" for v in a.ravel()) + "\n")
