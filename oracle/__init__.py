"""CPU oracle for the Slim Scheduler hot path -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import this package.  The product path
(`paper_2510_09018_b200`) never imports it and shares no code with it.

It is the plain definition of the batched forward pass of the segmented
SlimResNet at a runtime-chosen width, in float64:

* convolution: `oracle.c` (direct sum, fixed kh,kw,ci order; O2),
* everything else: numpy float64, one line per formula,
* the GroupNorm variant: `groupnorm`, `Model(norm="gn")`.

Citations: P:n = /root/reference/PAPER.md line n.  The paper fixes none of the
architecture; the readings used here (ResNet-18-CIFAR, per-width BN selected by
the segment's own width, eps=1e-5, ...) are listed in DESIGN.md "Readings".

Parity status: every function below is pinned by tests/test_oracle_pins.py
(brute force, torch float64 library routines, closed forms, invariants).  The
paper's own numbers (Tables I-V) need trained weights and CIFAR-100 and cannot
pin anything here: "parity unpinned" against the paper's printed values.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

# Width set W and BN epsilon (reading #6, PyTorch default).  Kept here,
# not imported from the CUDA side.
BN_EPS = 1e-5
# GroupNorm variant ("Group Normalization instead of Batch Normalization"; SURVEY
# §8(f) NEXT-1).  Group size is unstated in the paper: reading R16 fixes
# 16 consecutive channels per group, so every width c(r, C) (a multiple of 16) holds
# whole groups and a group means the same channels at every width.
GN_GROUP_CHANNELS = 16


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (-O3, strict IEEE: no -ffast-math, no FMA contraction) -> liboracle.so."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-fopenmp", "-fPIC", "-shared", "-fno-fast-math",
                               "-ffp-contract=off", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            dp = ctypes.POINTER(ctypes.c_double)
            L = ctypes.c_long
            lib.oracle_conv2d.argtypes = [dp, L, L, L, L, dp, L, L, L, L, L, L, dp]
            lib.oracle_conv2d.restype = ctypes.c_int
            lib.oracle_conv2d_plain.argtypes = [dp, L, L, L, L, dp, L, L, L, L, L, L, dp]
            lib.oracle_conv2d_plain.restype = ctypes.c_int
            lib.oracle_set_num_threads.argtypes = [ctypes.c_int]
            lib.oracle_set_num_threads.restype = None
            lib.oracle_max_threads.restype = ctypes.c_int
            lib.oracle_out_size.argtypes = [L, L, L, L]
            lib.oracle_out_size.restype = L
            _lib = lib
    return _lib


def set_num_threads(n: int) -> None:
    """OpenMP threads of the conv loops (results do not depend on it: one sequential sum per output)."""
    _load().oracle_set_num_threads(int(n))


def max_threads() -> int:
    return _load().oracle_max_threads()


def _ptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


# ---------------------------------------------------------------- O1 channels
def channels(r: float, C: int) -> int:
    """O1: c(r, C) = ceil(r*C) (north_star "first ceil(r*C) ... channels").

    Computed in integers for the width set {k/4}: r*4 is an exact integer there.
    """
    q = r * 4.0
    if abs(q - round(q)) < 1e-9:
        return (int(round(q)) * C + 3) // 4
    return int(np.ceil(r * C - 1e-9))


# ---------------------------------------------------------------- O2 conv
def conv2d(x: np.ndarray, w: np.ndarray, c_out: int, stride: int, pad: int, plain: bool = False) -> np.ndarray:
    """O2: width-sliced convolution of dense NHWC x with the full KRSC tensor w.

    x: [B,H,W,c_in] (c_in = x.shape[-1] active channels); w: [Cout_full,k,k,Cin_full].
    Reads w[:c_out, :, :, :c_in] only.  Returns float64 [B,Ho,Wo,c_out].
    plain=True runs the one-output-at-a-time loop nest (oracle_conv2d_plain); the default
    runs the same sums vectorised across outputs -- bitwise equal (pinned).
    """
    lib = _load()
    x = np.ascontiguousarray(x, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    B, H, W, c_in = x.shape
    cout_full, k, k2, cin_full = w.shape
    assert k == k2
    Ho = lib.oracle_out_size(H, k, stride, pad)
    Wo = lib.oracle_out_size(W, k, stride, pad)
    y = np.empty((B, Ho, Wo, c_out), dtype=np.float64)
    if B == 0:
        return y
    fn = lib.oracle_conv2d_plain if plain else lib.oracle_conv2d
    rc = fn(_ptr(x), B, H, W, c_in, _ptr(w), cout_full, k, cin_full, c_out, stride, pad, _ptr(y))
    if rc != 0:
        raise ValueError("oracle_conv2d: bad arguments")
    return y


# ---------------------------------------------------------------- O3 BN, O4 ReLU
def batchnorm(y: np.ndarray, stats: dict, eps: float = BN_EPS) -> np.ndarray:
    """O3 (inference BN, unfolded): z = (y - mu) / sqrt(var + eps) * gamma + beta."""
    c = y.shape[-1]
    mu = np.asarray(stats["mean"], np.float64)[:c]
    var = np.asarray(stats["var"], np.float64)[:c]
    gamma = np.asarray(stats["gamma"], np.float64)[:c]
    beta = np.asarray(stats["beta"], np.float64)[:c]
    assert mu.shape[0] == c, "BN statistics shorter than the active channel count"
    z = y - mu                       # the formula above, evaluated left to right in place
    z /= np.sqrt(var + eps)
    z *= gamma
    z += beta
    return z


def groupnorm(y: np.ndarray, params: dict, group_channels: int = GN_GROUP_CHANNELS,
              eps: float = BN_EPS) -> np.ndarray:
    """GN (Wu & He's definition, inference = training: no running statistics).

    Per image n and group g of `group_channels` consecutive channels:
    mu = mean of y[n, :, :, g], var = mean of (y - mu)^2 over the same H*W*group_channels
    values (biased), z = (y - mu) / sqrt(var + eps) * gamma[c] + beta[c].
    params: dict with gamma, beta (per channel of this width; mean/var are not used).
    """
    B, H, W, c = y.shape
    assert c % group_channels == 0, "active channels must hold whole groups (reading R16)"
    G = c // group_channels
    yg = y.reshape(B, H, W, G, group_channels)
    mu = yg.mean(axis=(1, 2, 4), keepdims=True)
    var = ((yg - mu) ** 2).mean(axis=(1, 2, 4), keepdims=True)
    z = ((yg - mu) / np.sqrt(var + eps)).reshape(B, H, W, c)
    gamma = np.asarray(params["gamma"], np.float64)[:c]
    beta = np.asarray(params["beta"], np.float64)[:c]
    assert gamma.shape[0] == c, "GN affine shorter than the active channel count"
    return z * gamma + beta


def relu(z: np.ndarray) -> np.ndarray:
    """O4: max(z, 0)."""
    return np.maximum(z, 0.0)


# ---------------------------------------------------------------- model
class Model:
    """Full-width shared weights + per-width BN sets (the paper's slimmable backbone).

    weights: dict layer name -> KRSC array, plus "fc_w" [classes][C3], "fc_b" [classes].
    bn:      dict layer name -> list over `widths` of dict(gamma, beta, mean, var).
    Layer names follow the manifest order of synth.layer_specs (stem, s{s}b{b}c1/c2/sc).
    """

    def __init__(self, weights: dict, bn: dict, widths=(0.25, 0.5, 0.75, 1.0),
                 base=(64, 128, 256, 512), blocks=(2, 2, 2, 2), eps: float = BN_EPS,
                 norm: str = "bn", group_channels: int = GN_GROUP_CHANNELS):
        self.w = {k: np.ascontiguousarray(v, dtype=np.float64) for k, v in weights.items()}
        self.bn = bn
        self.widths = tuple(float(r) for r in widths)
        self.base = tuple(base)
        self.blocks = tuple(blocks)
        self.eps = eps
        assert norm in ("bn", "gn")
        self.norm = norm                  # "bn": O3 switchable BN (NS); "gn": GroupNorm
        self.group_channels = group_channels

    def width_index(self, r: float) -> int:
        for i, q in enumerate(self.widths):
            if abs(q - r) < 1e-6:
                return i
        raise ValueError(f"width {r} not in the slimming set {self.widths}")

    def conv_bn(self, x, name, r, stride, pad, bn_width=None):
        """conv (O2) at output width c(r, Cout) followed by BN_{name, width r} (O3),
        or by GN with that width's affine (gamma, beta) when norm == "gn".
        During O10 calibration (`calibrate_bn`) the BN statistics of this (layer, width)
        are first set from this batch."""
        w = self.w[name]
        c_out = channels(r, w.shape[0])
        y = conv2d(x, w, c_out, stride, pad)
        wi = self.width_index(r if bn_width is None else bn_width)
        if getattr(self, "_calibrating", False):
            self.bn[name][wi] = batch_statistics(y, self.bn[name][wi])
        params = self.bn[name][wi]
        if self.norm == "gn":
            return groupnorm(y, params, self.group_channels, self.eps)
        return batchnorm(y, params, self.eps)

    # O10 fixture utility: BN calibration
    def calibrate_bn(self, x, r_per_seg) -> dict:
        """O10: run the chain O1-O8 on the calibration set x at the width
        tuple r_per_seg with *batch-statistics* BN, layer by layer in forward order: each
        BN's running mean / biased variance are set from its own input batch (`batch_statistics`)
        before it is applied, so every later layer sees the already-calibrated earlier ones.
        Returns the new BN dict (a copy; entries of the widths the tuple uses are replaced,
        rounded to float32 as the C-ABI stores them; gamma and beta are kept).  self.bn is
        left unchanged.  Fixture utility, not part of the forward pass."""
        assert self.norm == "bn", "O10 calibrates BatchNorm statistics"
        saved = self.bn
        self.bn = {k: [dict(e) for e in v] for k, v in saved.items()}
        self._calibrating = True
        try:
            self.chain(x, r_per_seg, head=False)
            out = self.bn
        finally:
            self._calibrating = False
            self.bn = saved
        return out

    def features(self, x, r_per_seg):
        """Pooled features p[n, c] = (1/16) sum_{h,w<4} h[n,h,w,c] after segment 3 (O7's first line)."""
        return self.chain(x, r_per_seg, head=False).mean(axis=(1, 2))

    # O5 BasicBlock
    def basic_block(self, x, s, b, r, bn_width=None):
        """O5: t = ReLU(BN1(conv3x3_s(x))); u = BN2(conv3x3_1(t));
        sc = BN_sc(conv1x1_s(x)) for the down-sampling block, else x; out = ReLU(u + sc)."""
        down = (s > 0 and b == 0)
        stride = 2 if down else 1
        t = relu(self.conv_bn(x, f"s{s}b{b}c1", r, stride, 1, bn_width))
        u = self.conv_bn(t, f"s{s}b{b}c2", r, 1, 1, bn_width)
        sc = self.conv_bn(x, f"s{s}b{b}sc", r, stride, 0, bn_width) if down else x
        return relu(u + sc)

    # O7 head
    def head(self, h, r3):
        """O7: p = mean over the 4x4 map; logits = b + p @ W_fc[:, :c3]^T."""
        p = h.mean(axis=(1, 2))                       # [B, c3]
        c3 = h.shape[-1]
        # elementwise product + per-row sum (not BLAS gemm: the result must not
        # depend on the batch size, SURVEY §8(c) "batch independence")
        return (p[:, None, :] * self.w["fc_w"][None, :, :c3]).sum(axis=-1) + self.w["fc_b"]

    # O6 segment
    def segment(self, s, x, r_prev, r, head=True, bn_width=None):
        """O6: segment s at (r_prev, r).  Seg 0: stem conv-BN-ReLU then blocks.
        Seg s>0: block 0 reads c_{s-1}(r_prev) channels (P:49 key (s, w_req, w_prev)).
        Seg 3 ends with the head (O7) when head=True.  bn_width overrides the BN
        set (negative control only)."""
        x = np.asarray(x, dtype=np.float64)
        if s == 0:
            x = relu(self.conv_bn(x, "stem", r, 1, 1, bn_width))
        else:
            assert x.shape[-1] == channels(r_prev, self.base[s - 1]), "input width != c(r_prev)"
        for b in range(self.blocks[s]):
            x = self.basic_block(x, s, b, r, bn_width)
        if s == 3 and head:
            return self.head(x, r)
        return x

    # O8 chain
    def chain(self, x, r_per_seg, head=True):
        """O8: seg0(r0) -> seg1(r0->r1) -> seg2(r1->r2) -> seg3(r2->r3) -> head."""
        h = self.segment(0, x, None, r_per_seg[0])
        for s in range(1, 4):
            h = self.segment(s, h, r_per_seg[s - 1], r_per_seg[s], head=head)
        return h


def batch_statistics(y: np.ndarray, stats: dict) -> dict:
    """O10 step for one BN: per-channel mean and BIASED variance of y over (N, H, W), rounded to
    float32 (the stored running statistics); gamma and beta are copied unchanged."""
    mean = y.mean(axis=(0, 1, 2))
    var = ((y - mean) ** 2).mean(axis=(0, 1, 2))
    return dict(gamma=stats["gamma"], beta=stats["beta"], mean=mean.astype(np.float32), var=var.astype(np.float32))


def ncm_head(features: np.ndarray, num_classes: int, c_full: int, scale: float = 4.0):
    """Nearest-class-mean head of the D2 fixture: from the pooled features
    f_k [num_classes, c3] of the 100 clean class prototypes,

        m = mean_k f_k,  W[k, :c3] = scale * (f_k - m) / ||f_k - m||_2,  W[k, c3:] = 0,
        b[k] = -sum_c m[c] * W[k, c],

    so logits(p) = W (p - m): a cosine classifier around the mean prototype.  W and b are
    rounded to bf16 (W first; b from the rounded W) so both sides read identical values.
    Returns (W [num_classes, c_full] float32, b [num_classes] float32)."""
    f = np.asarray(features, np.float64)
    assert f.shape[0] == num_classes
    c3 = f.shape[1]
    m = f.mean(axis=0)
    d = f - m
    u = d / np.sqrt((d * d).sum(axis=1, keepdims=True))
    W = np.zeros((num_classes, c_full), np.float64)
    W[:, :c3] = scale * u
    W = _round_bf16(W)
    b = _round_bf16(-(W[:, :c3] * m[None, :]).sum(axis=1))
    return W.astype(np.float32), b.astype(np.float32)


def _round_bf16(a: np.ndarray) -> np.ndarray:
    """float64 -> nearest float32 -> nearest bf16 (round-to-nearest-even), returned as float64."""
    f = np.ascontiguousarray(a, dtype=np.float32)
    bits = f.view(np.uint32).astype(np.uint64)
    out = ((bits + 0x7FFF + ((bits >> 16) & 1)) >> 16) << 16
    return out.astype(np.uint32).view(np.float32).astype(np.float64)


def per_image_rel_err(got: np.ndarray, ref: np.ndarray) -> np.ndarray:
    """Tolerance reading D4: per image, max_k |g-o| / max_k |o| (over all elements of the image)."""
    g = np.asarray(got, np.float64).reshape(got.shape[0], -1)
    o = np.asarray(ref, np.float64).reshape(ref.shape[0], -1)
    den = np.abs(o).max(axis=1)
    num = np.abs(g - o).max(axis=1)
    return num / np.maximum(den, 1e-30)
