"""D2 evaluation models (reading #13) assembled from tests/golden/d2_model.npz
(written by tests/golden/make_d2_fixture.py, which calls only oracle/) plus the synth draw.
No arithmetic here: dict assembly and bf16 bit-pattern decoding only."""
from __future__ import annotations

import functools
import os

import numpy as np

import synth

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "d2_model.npz")


@functools.lru_cache(maxsize=1)
def _npz():
    return dict(np.load(PATH))


def model(ti: int):
    """(weights, bn) of the D2 model of width tuple synth.TABLE_TUPLES[ti]: synth weights with the
    NCM head as fc_w/fc_b, synth BN with the calibrated mean/var at the tuple's widths."""
    d = _npz()
    tup = synth.TABLE_TUPLES[ti]
    weights = dict(synth.make_weights())
    weights["fc_w"] = (d[f"t{ti}/fc_w"].astype(np.uint32) << 16).view(np.float32)
    weights["fc_b"] = d[f"t{ti}/fc_b"]
    bn = {k: [dict(e) for e in v] for k, v in synth.make_bn().items()}
    for sp in synth.layer_specs():
        wi = synth.WIDTHS.index(tup[sp["seg"]])
        e = bn[sp["name"]][wi]
        e["mean"] = d[f"t{ti}/{sp['name']}/mean"]
        e["var"] = d[f"t{ti}/{sp['name']}/var"]
    return weights, bn


def eval_images(n: int):
    """D2 evaluation draw (offset 1; the calibration set is offset 0): images, labels."""
    x, y, _ = synth.make_prototype_images(n, sigma=float(_npz()["sigma"]), offset=1)
    return x, y
