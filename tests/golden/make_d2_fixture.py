"""Writes tests/golden/d2_model.npz: the D2 evaluation models (SURVEY.md §8(d) "D2 prototypes",
§8(c) O10 and reading #13; VERDICT r01 next #1a).  Calls only oracle/ (and synth/ for the seeded
numbers); nothing here comes from the CUDA path.

For every width tuple of PAPER.md Tables I-II:

1. BN calibration (O10, `oracle.Model.calibrate_bn`): the synth weights and the synth gamma/beta
   draw, with running mean / biased variance of every BN the tuple uses set from
   `N_CAL` = 512 D2 calibration images (prototypes + 0.1 N(0,1), calibration draw offset 0),
   layer by layer.
2. NCM head (`oracle.ncm_head`): from the pooled features of the 100 clean prototypes under the
   calibrated model: W[k] = 4 (f_k - m)/||f_k - m||, b = -m W^T, rounded to bf16.

Stored per tuple t (index into synth.TABLE_TUPLES): "t{t}/{layer}/mean", "t{t}/{layer}/var"
(float32, the layers of the segments at their tuple width), "t{t}/fc_w" (bf16 bit patterns,
uint16 [100, 512]), "t{t}/fc_b" (float32, bf16-representable).  tests/d2_fixture.py assembles a
(weights, bn) pair from these plus synth.  Regenerate with

    python tests/golden/make_d2_fixture.py          (about a minute on 8 cores)
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "d2_model.npz")
N_CAL = 512          # "BN is calibrated on 512 D2 samples"
SIGMA = 0.1          # sigma = 0.1 (0.25 fails the bf16 tolerance)


def layers_of_segment(s: int):
    return [sp["name"] for sp in synth.layer_specs() if sp["seg"] == s]


def build_tuple(ti: int, weights, bn, x_cal, protos):
    tup = synth.TABLE_TUPLES[ti]
    m = oracle.Model(weights, bn)
    bn_t = m.calibrate_bn(x_cal, tup)
    m_t = oracle.Model(weights, bn_t)
    feats = m_t.features(protos, tup)
    fc_w, fc_b = oracle.ncm_head(feats, synth.NUM_CLASSES, synth.BASE_CHANNELS[3])
    out = {}
    for s in range(4):
        wi = synth.WIDTHS.index(tup[s])
        for name in layers_of_segment(s):
            out[f"t{ti}/{name}/mean"] = np.asarray(bn_t[name][wi]["mean"], np.float32)
            out[f"t{ti}/{name}/var"] = np.asarray(bn_t[name][wi]["var"], np.float32)
    out[f"t{ti}/fc_w"] = synth.bf16_bits(fc_w)
    out[f"t{ti}/fc_b"] = fc_b.astype(np.float32)
    return out


def main():
    weights, bn = synth.make_weights(), synth.make_bn()
    x_cal, _, protos = synth.make_prototype_images(N_CAL, sigma=SIGMA, offset=0)
    data = {"n_cal": np.int64(N_CAL), "sigma": np.float64(SIGMA)}
    for ti in range(len(synth.TABLE_TUPLES)):
        t0 = time.time()
        data.update(build_tuple(ti, weights, bn, x_cal, protos))
        print(f"tuple {synth.TABLE_TUPLES[ti]}: {time.time() - t0:.1f} s", flush=True)
    np.savez_compressed(OUT, **data)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
