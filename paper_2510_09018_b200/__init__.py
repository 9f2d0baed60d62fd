"""Python binding of libslim.so (include/slim.h) -- argument marshalling only.

Every step of the forward pass runs in the CUDA kernels behind the C-ABI; this
module only converts Python objects (torch tensors, numpy arrays, floats) to the
plain pointers and sizes the ABI takes.  There is no CPU fallback: if the shared
library is missing or the GPU is absent, the calls raise.

Function names mirror the C entry points (slim_create, slim_load_segment,
slim_forward, slim_forward_chain, slim_pack, slim_launch, ...).  `SlimNet` is a
convenience wrapper that loads the four segments from a dict of named weights.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = [
    "SlimError", "load_library", "slim_config", "default_config", "slim_create", "slim_destroy",
    "slim_load_segment", "slim_unload_segment", "slim_segment_bytes", "slim_forward", "slim_forward_ws",
    "slim_forward_workspace_bytes", "slim_chain_workspace_bytes", "slim_forward_chain", "slim_pack",
    "slim_pack_arrays", "slim_launch", "slim_gather", "slim_scatter", "slim_last_error", "slim_launch_count", "slim_channels",
    "slim_act_channels", "SlimNet",
    "manifest", "LIB_PATH", "Scheduler", "NativeExecutor",
]

LIB_PATH = os.environ.get("SLIM_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libslim.so")

SLIM_OK, SLIM_EINVAL, SLIM_ENOTLOADED, SLIM_ENOMEM, SLIM_ECUDA, SLIM_EUNSUPPORTED = 0, -1, -2, -3, -4, -5
SLIM_BF16, SLIM_FP32 = 0, 1
SLIM_NORM_BN, SLIM_NORM_GN = 0, 1


class SlimError(RuntimeError):
    def __init__(self, status, msg=""):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


_STATUS = {0: "SLIM_OK", -1: "SLIM_EINVAL", -2: "SLIM_ENOTLOADED", -3: "SLIM_ENOMEM", -4: "SLIM_ECUDA",
           -5: "SLIM_EUNSUPPORTED"}


class slim_config(ctypes.Structure):
    _fields_ = [("n_widths", ctypes.c_int), ("widths", ctypes.c_float * 8), ("blocks_per_seg", ctypes.c_int * 4),
                ("base_channels", ctypes.c_int * 4), ("in_channels", ctypes.c_int), ("num_classes", ctypes.c_int),
                ("image_hw", ctypes.c_int), ("max_batch", ctypes.c_int), ("bn_eps", ctypes.c_float),
                ("dtype", ctypes.c_int), ("norm", ctypes.c_int), ("gn_group_channels", ctypes.c_int)]


class slim_seg_weights(ctypes.Structure):
    _fields_ = [("conv_w", ctypes.c_void_p * 16), ("n_conv", ctypes.c_int), ("fc_w", ctypes.c_void_p),
                ("fc_b", ctypes.c_void_p)]


class slim_bn(ctypes.Structure):
    _fields_ = [("gamma", ctypes.c_void_p), ("beta", ctypes.c_void_p), ("mean", ctypes.c_void_p),
                ("var", ctypes.c_void_p)]


class slim_bn_set(ctypes.Structure):
    _fields_ = [("per_layer", ctypes.POINTER(slim_bn)), ("n_layers", ctypes.c_int)]


class slim_request(ctypes.Structure):
    _fields_ = [("id", ctypes.c_uint64), ("seg", ctypes.c_int), ("w_req", ctypes.c_float),
                ("w_prev", ctypes.c_float), ("slot", ctypes.c_uint32)]


class slim_profile_record(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("seg", ctypes.c_int), ("layer", ctypes.c_int), ("batch", ctypes.c_int),
                ("r_prev", ctypes.c_float), ("r", ctypes.c_float), ("flops", ctypes.c_double),
                ("bytes", ctypes.c_double), ("ms", ctypes.c_float)]


KERNEL_KINDS = {0: "stem", 1: "conv_umma", 2: "head", 3: "gather", 4: "conv_f32", 5: "gn", 6: "seg_fused"}


class slim_launch_desc(ctypes.Structure):
    _fields_ = [("seg", ctypes.c_int), ("r_prev", ctypes.c_float), ("r", ctypes.c_float), ("batch", ctypes.c_int),
                ("first", ctypes.c_int)]


class slim_sched_knobs(ctypes.Structure):
    _fields_ = [("B_max", ctypes.c_int), ("M_max_bytes", ctypes.c_double), ("U_blk", ctypes.c_float),
                ("t_idle_s", ctypes.c_double), ("Q_th", ctypes.c_int), ("N_new", ctypes.c_int)]


class slim_sched_action(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("inst", ctypes.c_int), ("seg", ctypes.c_int), ("w_req", ctypes.c_float),
                ("w_prev", ctypes.c_float), ("inst_w", ctypes.c_float), ("batch", ctypes.c_int),
                ("n_loaded", ctypes.c_int)]


class slim_instance(ctypes.Structure):
    _fields_ = [("id", ctypes.c_int), ("seg", ctypes.c_int), ("w", ctypes.c_float), ("busy", ctypes.c_int),
                ("t_last", ctypes.c_double), ("bytes", ctypes.c_size_t)]


class slim_stream_stats(ctypes.Structure):
    _fields_ = [("batches", ctypes.c_int), ("launches", ctypes.c_int), ("pack_seconds", ctypes.c_double),
                ("host_seconds", ctypes.c_double)]


class slim_exec_stats(ctypes.Structure):
    _fields_ = [("batches", ctypes.c_int), ("loads", ctypes.c_int), ("requeues", ctypes.c_int),
                ("unloaded", ctypes.c_int), ("seconds", ctypes.c_double)]


SLIM_ACT_IDLE, SLIM_ACT_RUN, SLIM_ACT_REQUEUE = 0, 1, 2

_lib = None
_VP, _SZ, _I, _F = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_float


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libslim.so; raises (never falls back) if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"libslim.so not found at {path}: run `python -m paper_2510_09018_b200.build` "
                           "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    sig = {
        "slim_create": (_I, [_I, ctypes.POINTER(slim_config), ctypes.POINTER(_VP)]),
        "slim_destroy": (None, [_VP]),
        "slim_default_config": (None, [ctypes.POINTER(slim_config)]),
        "slim_load_segment": (_I, [_VP, _I, ctypes.POINTER(slim_seg_weights), ctypes.POINTER(slim_bn_set)]),
        "slim_unload_segment": (_I, [_VP, _I]),
        "slim_segment_loaded": (_I, [_VP, _I]),
        "slim_segment_bytes": (_SZ, [ctypes.POINTER(slim_config), _I, _F, _F]),
        "slim_forward": (_I, [_VP, _I, _F, _F, _I, _VP, _VP, _VP]),
        "slim_forward_workspace_bytes": (_SZ, [_VP, _I, _F, _F, _I]),
        "slim_forward_ws": (_I, [_VP, _I, _F, _F, _I, _VP, _VP, _VP, _SZ, _VP]),
        "slim_chain_workspace_bytes": (_SZ, [_VP, ctypes.POINTER(_F), _I]),
        "slim_forward_chain": (_I, [_VP, ctypes.POINTER(_F), _I, _VP, _VP, _VP, _SZ, _VP]),
        "slim_pack": (_I, [ctypes.POINTER(slim_config), ctypes.POINTER(slim_request), _I, _I,
                           ctypes.POINTER(slim_launch_desc), _I,
                           ctypes.POINTER(_I), ctypes.POINTER(ctypes.c_uint32)]),
        "slim_launch": (_I, [_VP, ctypes.POINTER(slim_launch_desc), _VP, _VP, _SZ, _VP, _VP, _VP, _SZ, _VP]),
        "slim_gather": (_I, [_VP, _VP, _VP, _I, _SZ, _VP, _VP]),
        "slim_scatter": (_I, [_VP, _VP, _VP, _I, _SZ, _VP, _SZ, _VP]),
        "slim_last_error": (_I, [_VP]),
        "slim_last_error_msg": (ctypes.c_char_p, [_VP]),
        "slim_status_str": (ctypes.c_char_p, [_I]),
        "slim_version": (_I, []),
        "slim_launch_count": (ctypes.c_uint64, [_VP]),
        "slim_num_sms": (_I, [_VP]),
        "slim_channels": (_I, [_F, _I]),
        "slim_act_channels": (_I, [_F, _I]),
        "slim_set_graph_mode": (_I, [_VP, _I]),
        "slim_set_sm_share": (_I, [_VP, _F, _F]),
        "slim_profile_begin": (_I, [_VP, _I]),
        "slim_profile_end": (_I, [_VP, ctypes.POINTER(slim_profile_record), _I, ctypes.POINTER(_I)]),
        "slim_sched_default_knobs": (None, [ctypes.POINTER(slim_sched_knobs)]),
        "slim_sched_create": (_I, [ctypes.POINTER(slim_config), ctypes.POINTER(slim_sched_knobs),
                                   ctypes.POINTER(_VP)]),
        "slim_sched_destroy": (None, [_VP]),
        "slim_sched_enqueue": (_I, [_VP, ctypes.POINTER(slim_request), _I, ctypes.c_double]),
        "slim_sched_next": (_I, [_VP, ctypes.c_double, _F, _SZ, ctypes.POINTER(slim_sched_action),
                                 ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint64)]),
        "slim_sched_complete": (_I, [_VP, _I, ctypes.c_double]),
        "slim_sched_unload_idle": (_I, [_VP, ctypes.c_double, ctypes.POINTER(_I), _I]),
        "slim_sched_queue_len": (_I, [_VP]),
        "slim_sched_b_max": (_I, [_VP]),
        "slim_sched_instances": (_I, [_VP, ctypes.POINTER(slim_instance), _I]),
        "slim_exec_create": (_I, [_VP, _VP, _I, _I, ctypes.POINTER(_VP)]),
        "slim_exec_destroy": (None, [_VP]),
        "slim_exec_run": (_I, [_VP, _VP, ctypes.POINTER(_F), _I, _VP, _SZ, ctypes.POINTER(slim_exec_stats), _VP,
                               ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
        "slim_stream_create": (_I, [_VP, _I, _I, _I, ctypes.POINTER(_VP)]),
        "slim_stream_destroy": (None, [_VP]),
        "slim_stream_run": (_I, [_VP, _VP, ctypes.POINTER(_F), _I, _VP, _VP, ctypes.POINTER(slim_stream_stats)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


EXPORTED = ("slim_create", "slim_destroy", "slim_default_config", "slim_load_segment", "slim_unload_segment",
            "slim_segment_loaded", "slim_segment_bytes", "slim_forward", "slim_forward_workspace_bytes",
            "slim_forward_ws", "slim_chain_workspace_bytes", "slim_forward_chain", "slim_pack", "slim_launch",
            "slim_gather", "slim_scatter", "slim_last_error", "slim_last_error_msg", "slim_status_str", "slim_version",
            "slim_launch_count", "slim_num_sms", "slim_channels", "slim_act_channels", "slim_set_graph_mode", "slim_set_sm_share", "slim_profile_begin",
            "slim_profile_end", "slim_sched_default_knobs", "slim_sched_create", "slim_sched_destroy",
            "slim_sched_enqueue", "slim_sched_next", "slim_sched_complete", "slim_sched_unload_idle",
            "slim_sched_queue_len", "slim_sched_b_max", "slim_sched_instances", "slim_exec_create", "slim_exec_destroy", "slim_exec_run",
            "slim_stream_create", "slim_stream_destroy", "slim_stream_run")


# ------------------------------------------------------------------ marshalling helpers
def _ptr(x):
    """Device/host pointer of a torch tensor, numpy array, int or None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()


def _stream(s):
    if s is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(s, int):
        return s
    return s.cuda_stream


def _check(ctx, status):
    if status != SLIM_OK:
        lib = load_library()
        msg = lib.slim_last_error_msg(ctx).decode() if ctx else ""
        raise SlimError(status, msg)


def default_config(**kw) -> slim_config:
    cfg = slim_config()
    load_library().slim_default_config(ctypes.byref(cfg))
    for k, v in kw.items():
        if k == "widths":
            cfg.n_widths = len(v)
            for i, r in enumerate(v):
                cfg.widths[i] = r
        elif k in ("blocks_per_seg", "base_channels"):
            for i, c in enumerate(v):
                getattr(cfg, k)[i] = c
        elif k == "dtype":
            cfg.dtype = {"bf16": SLIM_BF16, "fp32": SLIM_FP32}.get(v, v)
        elif k == "norm":
            cfg.norm = {"bn": SLIM_NORM_BN, "gn": SLIM_NORM_GN}.get(v, v)
        else:
            setattr(cfg, k, v)
    return cfg


def manifest(seg: int, blocks_per_seg=(2, 2, 2, 2)):
    """Layer names of segment `seg` in the ABI manifest order (include/slim.h slim_seg_weights)."""
    names = ["stem"] if seg == 0 else []
    for b in range(blocks_per_seg[seg]):
        names += [f"s{seg}b{b}c1", f"s{seg}b{b}c2"]
        if seg > 0 and b == 0:
            names.append(f"s{seg}b{b}sc")
    return names


# ------------------------------------------------------------------ C entry points
def slim_create(device: int = 0, cfg: slim_config | None = None):
    lib = load_library()
    cfg = cfg or default_config()
    h = ctypes.c_void_p()
    _check(None, lib.slim_create(device, ctypes.byref(cfg), ctypes.byref(h)))
    return h.value


def slim_destroy(ctx):
    load_library().slim_destroy(ctx)


def slim_load_segment(ctx, seg: int, conv_w: list, bn_per_width: list, fc_w=None, fc_b=None):
    """conv_w: fp32 host arrays in manifest order; bn_per_width: [width][layer] dicts(gamma,beta,mean,var)
    (GroupNorm mode reads gamma/beta only; mean/var may be absent)."""
    lib = load_library()
    keep = []
    w = slim_seg_weights()
    w.n_conv = len(conv_w)
    for i, a in enumerate(conv_w):
        a = np.ascontiguousarray(a, dtype=np.float32)
        keep.append(a)
        w.conv_w[i] = a.ctypes.data
    if fc_w is not None:
        fw = np.ascontiguousarray(fc_w, dtype=np.float32)
        fb = np.ascontiguousarray(fc_b, dtype=np.float32)
        keep += [fw, fb]
        w.fc_w, w.fc_b = fw.ctypes.data, fb.ctypes.data
    sets = (slim_bn_set * len(bn_per_width))()
    for wi, layers in enumerate(bn_per_width):
        arr = (slim_bn * len(layers))()
        for li, st in enumerate(layers):
            vals = [np.ascontiguousarray(st[k], dtype=np.float32) if st.get(k) is not None else None
                    for k in ("gamma", "beta", "mean", "var")]
            keep += [v for v in vals if v is not None]
            arr[li] = slim_bn(*[v.ctypes.data if v is not None else None for v in vals])
        keep.append(arr)
        sets[wi] = slim_bn_set(ctypes.cast(arr, ctypes.POINTER(slim_bn)), len(layers))
    _check(ctx, lib.slim_load_segment(ctx, seg, ctypes.byref(w), sets))


def slim_unload_segment(ctx, seg: int):
    _check(ctx, load_library().slim_unload_segment(ctx, seg))


def slim_segment_bytes(cfg: slim_config, seg: int, r_prev: float, r: float) -> int:
    return load_library().slim_segment_bytes(ctypes.byref(cfg), seg, r_prev, r)


def slim_forward(ctx, seg, r_prev, r, batch, x, out, stream=None):
    _check(ctx, load_library().slim_forward(ctx, seg, r_prev, r, batch, _ptr(x), _ptr(out), _stream(stream)))


def slim_forward_workspace_bytes(ctx, seg, r_prev, r, batch) -> int:
    return load_library().slim_forward_workspace_bytes(ctx, seg, r_prev, r, batch)


def slim_forward_ws(ctx, seg, r_prev, r, batch, x, out, ws, ws_bytes, stream=None):
    _check(ctx, load_library().slim_forward_ws(ctx, seg, r_prev, r, batch, _ptr(x), _ptr(out), _ptr(ws), ws_bytes,
                                               _stream(stream)))


def slim_chain_workspace_bytes(ctx, r_per_seg, batch) -> int:
    r4 = (ctypes.c_float * 4)(*r_per_seg)
    return load_library().slim_chain_workspace_bytes(ctx, r4, batch)


def slim_forward_chain(ctx, r_per_seg, batch, x, logits, ws, ws_bytes, stream=None):
    r4 = (ctypes.c_float * 4)(*r_per_seg)
    _check(ctx, load_library().slim_forward_chain(ctx, r4, batch, _ptr(x), _ptr(logits), _ptr(ws), ws_bytes,
                                                  _stream(stream)))


def slim_pack(cfg: slim_config, requests, B_max: int):
    """Greedy key batching (host only, no GPU).  requests: iterable of (id, seg, w_req, w_prev, slot).
    Returns (descs list of dicts, order ndarray)."""
    reqs = list(requests)
    n = len(reqs)
    q = (slim_request * max(n, 1))()
    for i, (rid, seg, wr, wp, slot) in enumerate(reqs):
        q[i] = slim_request(rid, seg, wr, wp, slot)
    descs = (slim_launch_desc * max(n, 1))()
    order = (ctypes.c_uint32 * max(n, 1))()
    nd = ctypes.c_int()
    _check(None, load_library().slim_pack(ctypes.byref(cfg), q, n, B_max, descs, max(n, 1), ctypes.byref(nd), order))
    out = [dict(seg=d.seg, r_prev=d.r_prev, r=d.r, batch=d.batch, first=d.first) for d in descs[:nd.value]]
    return out, np.frombuffer(order, dtype=np.uint32, count=n).copy()


# numpy mirror of slim_request (include/slim.h): marshal a whole request array without a Python loop
_REQ_DTYPE = np.dtype({"names": ["id", "seg", "w_req", "w_prev", "slot"],
                       "formats": [np.uint64, np.int32, np.float32, np.float32, np.uint32],
                       "offsets": [0, 8, 12, 16, 20], "itemsize": ctypes.sizeof(slim_request)})


def slim_pack_arrays(cfg: slim_config, seg: int, w_req, w_prev, B_max: int, ids=None, slots=None):
    """slim_pack on arrays (one segment): request i = (id ids[i] (default i), seg, w_req[i], w_prev[i],
    slot slots[i] (default i)).  Marshalling only, vectorised.  Returns (descs list, order ndarray)."""
    w_req = np.asarray(w_req, np.float32)
    n = w_req.shape[0]
    q = np.zeros(max(n, 1), _REQ_DTYPE)
    q["id"][:n] = np.arange(n) if ids is None else ids
    q["seg"][:n] = seg
    q["w_req"][:n] = w_req
    q["w_prev"][:n] = np.asarray(w_prev, np.float32) if seg else 0.0
    q["slot"][:n] = np.arange(n) if slots is None else slots
    descs = (slim_launch_desc * max(n, 1))()
    order = np.zeros(max(n, 1), np.uint32)
    nd = ctypes.c_int()
    _check(None, load_library().slim_pack(ctypes.byref(cfg), q.ctypes.data_as(ctypes.POINTER(slim_request)), n,
                                          B_max, descs, max(n, 1), ctypes.byref(nd),
                                          order.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))))
    out = [dict(seg=d.seg, r_prev=d.r_prev, r=d.r, batch=d.batch, first=d.first) for d in descs[:nd.value]]
    return out, order[:n]


def slim_launch(ctx, desc: dict, slots, pool, pool_row_bytes, slab, out, ws, ws_bytes, stream=None):
    d = slim_launch_desc(desc["seg"], desc["r_prev"], desc["r"], desc["batch"], desc.get("first", 0))
    _check(ctx, load_library().slim_launch(ctx, ctypes.byref(d), _ptr(slots), _ptr(pool), pool_row_bytes,
                                           _ptr(slab), _ptr(out), _ptr(ws), ws_bytes, _stream(stream)))


def slim_gather(ctx, src, idx, n, row_bytes, dst, stream=None):
    _check(ctx, load_library().slim_gather(ctx, _ptr(src), _ptr(idx), n, row_bytes, _ptr(dst), _stream(stream)))


def slim_scatter(ctx, src, idx, n, row_bytes, dst, dst_stride, stream=None):
    _check(ctx, load_library().slim_scatter(ctx, _ptr(src), _ptr(idx), n, row_bytes, _ptr(dst), dst_stride,
                                            _stream(stream)))


def slim_last_error(ctx) -> int:
    return load_library().slim_last_error(ctx)


def slim_launch_count(ctx) -> int:
    return load_library().slim_launch_count(ctx)


def slim_channels(r: float, C: int) -> int:
    return load_library().slim_channels(r, C)


def slim_act_channels(r: float, C: int) -> int:
    """Channels an activation of width r carries (c(r, C) padded to the kernel granule; extra ones are 0)."""
    return load_library().slim_act_channels(r, C)


def slim_set_graph_mode(ctx, enable: bool):
    _check(ctx, load_library().slim_set_graph_mode(ctx, int(bool(enable))))


def slim_set_sm_share(ctx, r: float, share: float):
    _check(ctx, load_library().slim_set_sm_share(ctx, r, share))


def slim_profile_begin(ctx, max_launches: int):
    _check(ctx, load_library().slim_profile_begin(ctx, max_launches))


def slim_profile_end(ctx, max_out: int = 1 << 20):
    """Synchronises; returns a list of dicts (kind, seg, layer, batch, r_prev, r, flops, bytes, ms)."""
    lib = load_library()
    n = ctypes.c_int()
    _check(ctx, lib.slim_profile_end(ctx, None, 0, ctypes.byref(n)))
    recs = (slim_profile_record * max(n.value, 1))()
    _check(ctx, lib.slim_profile_end(ctx, recs, n.value, ctypes.byref(n)))
    return [dict(kind=KERNEL_KINDS.get(r.kind, r.kind), seg=r.seg, layer=r.layer, batch=r.batch, r_prev=r.r_prev,
                 r=r.r, flops=r.flops, bytes=r.bytes, ms=r.ms) for r in recs[:n.value]]


# ------------------------------------------------------------------ Alg. 1 scheduler (host)
class Scheduler:
    """Marshalling wrapper of the native Alg. 1 decision engine (slim_sched_*, include/slim.h).

    requests: iterables of (id, seg, w_req, w_prev, slot).  next() returns a dict
    (kind, inst, seg, w_req, w_prev, inst_w, batch, n_loaded, slots, ids)."""

    KIND = {SLIM_ACT_IDLE: "idle", SLIM_ACT_RUN: "run", SLIM_ACT_REQUEUE: "requeue"}

    def __init__(self, cfg: slim_config, **knobs):
        lib = load_library()
        self.k = slim_sched_knobs()
        lib.slim_sched_default_knobs(ctypes.byref(self.k))
        for name, v in knobs.items():
            setattr(self.k, name, v)
        h = ctypes.c_void_p()
        _check(None, lib.slim_sched_create(ctypes.byref(cfg), ctypes.byref(self.k), ctypes.byref(h)))
        self.h = h.value
        self._slots = (ctypes.c_uint32 * self.k.B_max)()
        self._ids = (ctypes.c_uint64 * self.k.B_max)()

    def enqueue(self, requests, t_enq: float = 0.0):
        reqs = list(requests)
        q = (slim_request * max(len(reqs), 1))()
        for i, (rid, seg, wr, wp, slot) in enumerate(reqs):
            q[i] = slim_request(rid, seg, wr, wp, slot)
        _check(None, load_library().slim_sched_enqueue(self.h, q, len(reqs), t_enq))

    def next(self, now: float, util: float = -1.0, vram_external: int = 0) -> dict:
        act = slim_sched_action()
        _check(None, load_library().slim_sched_next(self.h, now, util, vram_external, ctypes.byref(act),
                                                    self._slots, self._ids))
        n = act.batch if act.kind == SLIM_ACT_RUN else 0
        return dict(kind=self.KIND[act.kind], inst=act.inst, seg=act.seg, w_req=act.w_req, w_prev=act.w_prev,
                    inst_w=act.inst_w, batch=act.batch, n_loaded=act.n_loaded,
                    slots=np.frombuffer(self._slots, np.uint32, n).copy(),
                    ids=np.frombuffer(self._ids, np.uint64, n).copy())

    def complete(self, inst: int, now: float):
        _check(None, load_library().slim_sched_complete(self.h, inst, now))

    def unload_idle(self, now: float):
        buf = (ctypes.c_int * 256)()
        n = load_library().slim_sched_unload_idle(self.h, now, buf, 256)
        return list(buf[:min(n, 256)])

    def queue_len(self) -> int:
        return load_library().slim_sched_queue_len(self.h)

    def instances(self):
        lib = load_library()
        n = lib.slim_sched_instances(self.h, None, 0)
        buf = (slim_instance * max(n, 1))()
        lib.slim_sched_instances(self.h, buf, n)
        return [dict(id=i.id, seg=i.seg, w=i.w, busy=bool(i.busy), t_last=i.t_last, bytes=i.bytes) for i in buf[:n]]

    def close(self):
        if self.h:
            load_library().slim_sched_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class NativeExecutor:
    """Marshalling wrapper of the native Alg. 1 executor (slim_exec_*): the LOOP runs in C++."""

    def __init__(self, net, n_max: int, B_max: int = 256, **knobs):
        self.net = net
        self.sched = Scheduler(net.cfg, B_max=B_max, **knobs)
        h = ctypes.c_void_p()
        _check(net.ctx, load_library().slim_exec_create(net.ctx, self.sched.h, n_max, B_max, ctypes.byref(h)))
        self.h = h.value
        self.n_max = n_max
        self.stats = {}

    def run(self, images, tuples, logits=None, vram_external: int = 0, stream=None, arrivals=None):
        """images: device [n,H,W,C]; tuples: [n,4] widths.  Returns fp32 logits [n, classes].
        arrivals: optional ascending arrival times (s) -- open loop; then self.done holds each
        request's completion time (s, same clock) and self.latency = done - arrivals."""
        import torch
        t = np.ascontiguousarray(np.asarray(tuples, np.float32))
        n = t.shape[0]
        if logits is None:
            logits = torch.empty(n, self.net.cfg.num_classes, dtype=torch.float32, device=images.device)
        st = slim_exec_stats()
        dp = ctypes.POINTER(ctypes.c_double)
        arr = None if arrivals is None else np.ascontiguousarray(np.asarray(arrivals, np.float64))
        done = np.zeros(n, np.float64)
        _check(self.net.ctx, load_library().slim_exec_run(
            self.h, _ptr(images), t.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), n, _ptr(logits), vram_external,
            ctypes.byref(st), _stream(stream), None if arr is None else arr.ctypes.data_as(dp), done.ctypes.data_as(dp)))
        self.done = done
        self.latency = done - (arr if arr is not None else 0.0)
        self.stats = dict(batches=st.batches, loads=st.loads, requeues=st.requeues, unloaded=st.unloaded,
                          seconds=st.seconds)
        return logits

    def close(self):
        if self.h:
            load_library().slim_exec_destroy(self.h)
            self.h = None
        self.sched.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ convenience
class SlimNet:
    """A context with all four segments loaded from named weights.

    weights: dict layer name -> KRSC fp32 array (+ "fc_w", "fc_b");
    bn: dict layer name -> list over widths of dict(gamma, beta, mean, var).
    """

    def __init__(self, weights: dict, bn: dict, device: int = 0, segments=(0, 1, 2, 3), **cfg_kw):
        self.cfg = default_config(**cfg_kw)
        self.ctx = slim_create(device, self.cfg)
        self.widths = tuple(self.cfg.widths[i] for i in range(self.cfg.n_widths))
        self._host = (weights, bn)   # host copy: Alg. 1's offloaded segments reload from here
        for s in segments:
            self.load_segment(s)
        self._ws = {}

    def load_segment(self, s: int):
        """(Re)load segment s from the host copy (slim_load_segment copies to the device)."""
        weights, bn = self._host
        names = manifest(s, tuple(self.cfg.blocks_per_seg))
        conv = [weights[n] for n in names]
        bn_sets = [[bn[n][wi] for n in names] for wi in range(self.cfg.n_widths)]
        if s == 3:
            slim_load_segment(self.ctx, s, conv, bn_sets, weights["fc_w"], weights["fc_b"])
        else:
            slim_load_segment(self.ctx, s, conv, bn_sets)

    def unload_segment(self, s: int):
        slim_unload_segment(self.ctx, s)

    def set_sm_shares(self, shares: dict):
        """{width: share of the SMs} for concurrent width instances (slim_set_sm_share)."""
        for r, sh in shares.items():
            slim_set_sm_share(self.ctx, r, sh)

    def segment_loaded(self, s: int) -> bool:
        return bool(load_library().slim_segment_loaded(self.ctx, s))

    @property
    def act_dtype(self):
        import torch
        return torch.bfloat16 if self.cfg.dtype == SLIM_BF16 else torch.float32

    def chain_workspace(self, r_per_seg, batch):
        import torch
        nbytes = slim_chain_workspace_bytes(self.ctx, r_per_seg, batch)
        key = ("chain", nbytes)
        if key not in self._ws:
            self._ws = {key: torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{self.device_index}")}
        return self._ws[key], nbytes

    @property
    def device_index(self):
        import torch
        return torch.cuda.current_device()

    def forward_chain(self, x, r_per_seg, logits=None, stream=None):
        """x: [B,32,32,3] device tensor of act_dtype.  Returns fp32 logits [B, classes]."""
        import torch
        B = x.shape[0]
        if logits is None:
            logits = torch.empty(B, self.cfg.num_classes, dtype=torch.float32, device=x.device)
        ws, nbytes = self.chain_workspace(r_per_seg, B)
        slim_forward_chain(self.ctx, r_per_seg, B, x, logits, ws, nbytes, stream)
        return logits

    def segment_out_shape(self, seg, r, B):
        if seg == 3:
            return (B, self.cfg.num_classes)
        H = self.cfg.image_hw >> seg
        return (B, H, H, slim_act_channels(r, self.cfg.base_channels[seg]))

    def forward(self, seg, x, r_prev, r, out=None, stream=None):
        import torch
        B = x.shape[0]
        if out is None:
            dt = torch.float32 if seg == 3 else self.act_dtype
            out = torch.empty(self.segment_out_shape(seg, r, B), dtype=dt, device=x.device)
        slim_forward(self.ctx, seg, r_prev, r, B, x, out, stream)
        return out

    def close(self):
        if self.ctx:
            slim_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
