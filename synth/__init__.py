"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module is the ONE place both sides draw from (task rule: "only the seeded
input generators serve both, from a module of their own that holds none of the
method's arithmetic").  It produces numbers -- weights, BatchNorm statistics,
images, request streams -- and nothing here evaluates a convolution, a BN, a
pool or a classifier.  The oracle (`oracle/`) and the CUDA binding
(`paper_2510_09018_b200/`) both consume these arrays; neither imports the other.

Recipe:

* master seed 2510_09018; named substreams weights=+1, bn=+2, D1 inputs=+3,
  D2 prototypes=+4, request stream=+5.
* Architecture reading D1: CIFAR ResNet-18, BasicBlock
  x[2,2,2,2], base channels C=[64,128,256,512], 3x3 stem without max-pool,
  segment s = residual stage s (stem in segment 0, pool+FC in segment 3).
  PAPER.md:148 only says "SlimResNet partitioned into four sequential segments".
* Conv weights: Kaiming-normal, std sqrt(2/fan_in_full), rounded to bf16 (RNE)
  so every value is exactly representable on both sides.  FC: U(+-1/sqrt(512)).
* BN statistics per (layer, width) -- "switchable BN" (north_star): gamma~U(.5,1.5),
  beta~U(-.1,.1); running var = 2 * (c_in(r)/C_in_full) * m2_in * U(.8,1.25)
  (the expected output variance of a Kaiming conv over the active fan-in, so
  that every width stays O(1) instead of shrinking by ~r per layer);
  running mean = sqrt(var) * U(-.2,.2).  Distinct for every width.
* D1 images: i.i.d. N(0,1) [B,32,32,3] NHWC, rounded to bf16.
* D2 images: 100 class prototypes N(0,1); x = proto[y] + sigma*N(0,1).

All float arrays are float32 holding bf16-representable values unless said.
"""
from __future__ import annotations

import numpy as np

MASTER_SEED = 2510_09018

# Architecture.  Width set W ("w in {1.00,0.75,0.50,0.25}").
BASE_CHANNELS = (64, 128, 256, 512)
BLOCKS_PER_SEG = (2, 2, 2, 2)
IN_CHANNELS = 3
NUM_CLASSES = 100
IMAGE_HW = 32
WIDTHS = (0.25, 0.5, 0.75, 1.0)
BN_EPS = 1e-5

# The eight width tuples of PAPER.md Tables I (l.164) and II (l.172-175).
TABLE_TUPLES = (
    (0.25, 0.25, 0.25, 0.25), (0.5, 0.5, 0.5, 0.5), (0.75, 0.75, 0.75, 0.75), (1.0, 1.0, 1.0, 1.0),
    (1.0, 0.75, 0.5, 0.25), (0.75, 1.0, 0.25, 0.5), (0.5, 0.25, 1.0, 0.75), (0.25, 0.5, 0.75, 1.0),
)


def active_channels(r: float, C: int) -> int:
    """ceil(r*C) for sizing generated arrays (integer form, exact for r=k/4)."""
    return int(np.ceil(r * C - 1e-9))


def round_bf16(a) -> np.ndarray:
    """Round float32 values to the nearest bf16 (round-to-nearest-even); returns float32."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    bits = a.view(np.uint32).astype(np.uint64)
    bias = 0x7FFF + ((bits >> 16) & 1)
    out = ((bits + bias) >> 16) << 16
    return out.astype(np.uint32).view(np.float32).reshape(a.shape)


def bf16_bits(a) -> np.ndarray:
    """uint16 bit patterns of bf16-representable float32 values (no rounding done here)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    return (a.view(np.uint32) >> 16).astype(np.uint16)


def _rng(sub: int, seed: int = MASTER_SEED) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64([seed, sub]))


def layer_specs(base=BASE_CHANNELS, blocks=BLOCKS_PER_SEG, in_ch=IN_CHANNELS):
    """Conv layers in the fixed manifest order used by every consumer.

    seg 0: stem, then per block: c1, c2.   seg s>0, block 0: c1 (stride 2), c2, sc (1x1 s2
    projection); later blocks: c1, c2.  Each entry: name, seg, block, kind, cout, cin, k, stride.
    `cin` is the FULL input channel count of the shared weight tensor.
    """
    specs = []
    for s in range(4):
        C = base[s]
        if s == 0:
            specs.append(dict(name="stem", seg=0, block=-1, kind="stem", cout=C, cin=in_ch, k=3, stride=1))
        for b in range(blocks[s]):
            down = (s > 0 and b == 0)
            cin = base[s - 1] if down else C
            specs.append(dict(name=f"s{s}b{b}c1", seg=s, block=b, kind="c1", cout=C, cin=cin, k=3,
                              stride=2 if down else 1))
            specs.append(dict(name=f"s{s}b{b}c2", seg=s, block=b, kind="c2", cout=C, cin=C, k=3, stride=1))
            if down:
                specs.append(dict(name=f"s{s}b{b}sc", seg=s, block=b, kind="sc", cout=C, cin=cin, k=1, stride=2))
    return specs


def make_weights(seed: int = MASTER_SEED, base=BASE_CHANNELS, blocks=BLOCKS_PER_SEG):
    """Full-width shared weights, KRSC [Cout][k][k][Cin] float32 (bf16-representable).

    Returns dict name -> array, plus "fc_w" [100][C3] and "fc_b" [100].
    """
    g = _rng(1, seed)
    out = {}
    for sp in layer_specs(base, blocks):
        fan_in = sp["k"] * sp["k"] * sp["cin"]
        w = g.standard_normal((sp["cout"], sp["k"], sp["k"], sp["cin"]), dtype=np.float32)
        out[sp["name"]] = round_bf16(w * np.float32(np.sqrt(2.0 / fan_in)))
    bound = 1.0 / np.sqrt(base[3])
    out["fc_w"] = round_bf16(g.uniform(-bound, bound, (NUM_CLASSES, base[3])).astype(np.float32))
    out["fc_b"] = round_bf16(g.uniform(-bound, bound, (NUM_CLASSES,)).astype(np.float32))
    return out


def make_bn(seed: int = MASTER_SEED, base=BASE_CHANNELS, blocks=BLOCKS_PER_SEG, widths=WIDTHS):
    """Switchable BN statistics: dict name -> list over widths of dict(gamma,beta,mean,var).

    Each array has length c_out(width) = ceil(width*Cout).  For input-width
    dependence the recipe assumes the previous segment ran at the same width.
    """
    g = _rng(2, seed)
    out = {}
    for sp in layer_specs(base, blocks):
        per_w = []
        for r in widths:
            c = active_channels(r, sp["cout"])
            cin_act = sp["cin"] if sp["kind"] == "stem" else active_channels(r, sp["cin"])
            m2_in = 1.0 if sp["kind"] == "stem" else 0.55
            var_est = 2.0 * cin_act / sp["cin"] * m2_in
            gamma = g.uniform(0.5, 1.5, c).astype(np.float32)
            beta = g.uniform(-0.1, 0.1, c).astype(np.float32)
            var = (var_est * g.uniform(0.8, 1.25, c)).astype(np.float32)
            mean = (np.sqrt(var) * g.uniform(-0.2, 0.2, c)).astype(np.float32)
            per_w.append(dict(gamma=gamma, beta=beta, mean=mean, var=var))
        out[sp["name"]] = per_w
    return out


def make_images(B: int, seed: int = MASTER_SEED, offset: int = 0) -> np.ndarray:
    """D1: i.i.d. N(0,1) NHWC [B,32,32,3] rounded to bf16.  `offset` selects a disjoint draw."""
    g = _rng(3 + 1000 * offset, seed)
    x = g.standard_normal((B, IMAGE_HW, IMAGE_HW, IN_CHANNELS), dtype=np.float32)
    return round_bf16(x)


def make_prototype_images(B: int, sigma: float = 0.1, seed: int = MASTER_SEED, offset: int = 0):
    """D2: (images [B,32,32,3], labels [B], prototypes [100,32,32,3]); all bf16-representable."""
    g = _rng(4, seed)
    protos = round_bf16(g.standard_normal((NUM_CLASSES, IMAGE_HW, IMAGE_HW, IN_CHANNELS), dtype=np.float32))
    g2 = _rng(4 + 1000 * (offset + 1), seed)
    y = g2.integers(0, NUM_CLASSES, B)
    x = round_bf16(protos[y] + np.float32(sigma) * g2.standard_normal(
        (B, IMAGE_HW, IMAGE_HW, IN_CHANNELS), dtype=np.float32))
    return x, y, protos


def make_request_stream(n: int, seed: int = MASTER_SEED, tuples=TABLE_TUPLES):
    """CFG4 request stream: each request draws a width tuple uniformly from Tables I-II.

    Returns an int array [n] of tuple indices (into `tuples`).
    """
    g = _rng(5, seed)
    return g.integers(0, len(tuples), n)


def nan_poison_weights(weights: dict, r_prev: float, r: float, base=BASE_CHANNELS, blocks=BLOCKS_PER_SEG):
    """Copy of `weights` with every entry OUTSIDE the active prefix set to NaN.

    Used by the prefix-isolation invariant (SURVEY §8(c) pins): a correct slicer
    never reads those entries.  For seg-0 layers r_prev is ignored; for the first
    conv/projection of seg s>0 the input prefix is c(r_prev).  Other widths use r.
    """
    out = {}
    for sp in layer_specs(base, blocks):
        w = weights[sp["name"]].copy()
        co = active_channels(r, sp["cout"])
        if sp["kind"] == "stem":
            ci = sp["cin"]
        elif sp["seg"] > 0 and sp["block"] == 0 and sp["kind"] in ("c1", "sc"):
            ci = active_channels(r_prev, sp["cin"])
        else:
            ci = active_channels(r, sp["cin"])
        w[co:] = np.nan
        w[..., ci:] = np.nan
        out[sp["name"]] = w
    fc = weights["fc_w"].copy()
    fc[:, active_channels(r, base[3]):] = np.nan
    out["fc_w"] = fc
    out["fc_b"] = weights["fc_b"].copy()
    return out
