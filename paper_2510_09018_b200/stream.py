"""Request-stream executor (CFG4): greedy key batching + gather + segment forwards.

A request carries a width tuple (w_0..w_3) and re-enters the queue after each
segment with key k = (s, w_req = w_s, w_prev = w_{s-1}).  Per
segment this executor

  1. groups the live requests by key with the ABI packer (`slim_pack`, Alg. 1
     lines 3-4: FIFO head key, up to B_max requests of that key),
  2. runs each group with `slim_launch`: the device gather kernel copies the
     requests' activations from the segment's input pool into a contiguous slab,
     then the segment forward runs on it (RUNBATCH, Alg. 1 l.10),
  3. scatters the group's outputs back to the next segment's pool (`slim_scatter`),
     or the logits for segment 3.

Every data movement and all arithmetic run in libslim's kernels; this module only
sequences calls (host control, SURVEY §3 stack 2).  Buffers are allocated once
for n_max requests; graph mode caches one CUDA graph per (group shape, buffers).
"""
from __future__ import annotations

import time

import numpy as np
import torch

from . import SlimNet, slim_act_channels, slim_forward_workspace_bytes, slim_launch, slim_pack_arrays, slim_scatter


class StreamExecutor:
    def __init__(self, net: SlimNet, n_max: int, B_max: int = 256, device=None, lanes: int = 1):
        self.net = net
        self.cfg = net.cfg
        self.n_max = n_max
        self.B_max = B_max
        self.dev = torch.device(device if device is not None else f"cuda:{torch.cuda.current_device()}")
        cfg = self.cfg
        self.eb = 2 if cfg.dtype == 0 else 4
        self.adt = torch.bfloat16 if cfg.dtype == 0 else torch.float32
        hw = cfg.image_hw
        wmax = cfg.widths[cfg.n_widths - 1]
        # per-segment input pools, rows sized for the widest previous width (dense prefix per row)
        self.row_elems = [hw * hw * cfg.in_channels]
        for s in range(1, 4):
            h = hw >> (s - 1)
            self.row_elems.append(h * h * slim_act_channels(wmax, cfg.base_channels[s - 1]))
        self.pools = [None] + [torch.empty(n_max * self.row_elems[s], dtype=self.adt, device=self.dev)
                               for s in range(1, 4)]
        self.logits = torch.empty(n_max, cfg.num_classes, dtype=torch.float32, device=self.dev)
        # lanes: batches of one segment with different keys are independent -- with lanes > 1 they
        # run concurrently on their own streams (one lane per width; the context's per-width SM
        # shares keep them side by side), joined before the next segment reads the pools
        self.lanes = max(1, int(lanes))
        out_elems = max(max(self.row_elems[1:]), cfg.num_classes * 4 // self.eb)
        self.wsb = max(slim_forward_workspace_bytes(net.ctx, s, wmax, wmax, B_max) for s in range(4))
        self.lane_buf = [(torch.empty(B_max * max(self.row_elems), dtype=self.adt, device=self.dev),
                          torch.empty(B_max * out_elems, dtype=self.adt, device=self.dev),
                          torch.empty(self.wsb, dtype=torch.uint8, device=self.dev)) for _ in range(self.lanes)]
        self.slab, self.out, self.ws = self.lane_buf[0]
        self.lane_streams = [torch.cuda.Stream(device=self.dev) for _ in range(self.lanes)] if self.lanes > 1 else []
        self.widths = [cfg.widths[i] for i in range(cfg.n_widths)]
        # two pinned staging buffers for the per-segment request orders, used alternately: a buffer is
        # rewritten only after the H2D copy that last read it (enqueued on the run's stream) is done
        self.order_h = [torch.empty(4 * n_max, dtype=torch.int32).pin_memory() for _ in range(2)]
        self._order_ev = [None, None]
        self._buf = 0
        self.order_d = torch.empty(4 * n_max, dtype=torch.int32, device=self.dev)
        self._plan_key = None
        self.last_batches = []
        self.cache_plans = True     # False: pack every call (a fresh request stream each step)
        self.pack_s = []            # host seconds of each packing (slim_pack on all four segments)

    def _plan(self, tuples: np.ndarray, st):
        """Pack all four segments (host only) and stage the request orders to the device on `st`.
        Cached for a repeated stream unless cache_plans is False."""
        key = (tuples.shape[0], hash(tuples.tobytes()))
        if self.cache_plans and key == self._plan_key:
            return self._plan_cache
        n = tuples.shape[0]
        t0 = time.perf_counter()
        plan = []
        for s in range(4):
            descs, order = slim_pack_arrays(self.cfg, s, tuples[:, s], tuples[:, s - 1] if s else None, self.B_max)
            plan.append((descs, order.astype(np.int32)))
        self.pack_s.append(time.perf_counter() - t0)
        self._plan_key, self._plan_cache = key, plan
        b = self._buf
        self._buf ^= 1
        if self._order_ev[b] is not None:
            self._order_ev[b].synchronize()        # the copy that last read order_h[b] has run
        oh = self.order_h[b]
        oh[:4 * n].view(4, n).copy_(torch.from_numpy(np.stack([p[1] for p in plan])))
        with torch.cuda.stream(st):               # ordered before the lanes forked from st read order_d
            self.order_d[:4 * n].copy_(oh[:4 * n], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(st)
        self._order_ev[b] = ev
        self.last_batches = [[d["batch"] for d in p[0]] for p in plan]
        return plan

    def run(self, images: torch.Tensor, tuples: np.ndarray, stream=None) -> torch.Tensor:
        """images: device [n, H, W, C] (activation dtype); tuples: [n, 4] width per segment.
        Returns the logits [n, classes] (a view into the executor's buffer)."""
        n = images.shape[0]
        assert n <= self.n_max and tuples.shape == (n, 4)
        st = stream if stream is not None else torch.cuda.current_stream(self.dev)
        plan = self._plan(np.asarray(tuples, np.float32), st)
        hw, cfg = self.cfg.image_hw, self.cfg
        for s in range(4):
            descs, _ = plan[s]
            pool = images if s == 0 else self.pools[s]
            pool_row = self.row_elems[s] * self.eb
            base = s * n
            if self.lanes > 1:   # fork: every lane starts after the previous segment's scatters
                fork = torch.cuda.Event()
                fork.record(st)
                for ls in self.lane_streams:
                    ls.wait_event(fork)
            per_width = {}
            for d in descs:
                b, first = d["batch"], d["first"]
                idx = self.order_d[base + first: base + first + b]
                # lane = width index, plus (lanes > widths) a rotation over the width's batches of this segment
                wi = self.widths.index(min(self.widths, key=lambda w: abs(w - d["r"])))
                j = per_width.get(wi, 0)
                per_width[wi] = j + 1
                nw = len(self.widths)
                lane = (wi + nw * (j % max(1, self.lanes // nw))) % self.lanes
                slab, out, ws = self.lane_buf[lane]
                ls = self.lane_streams[lane] if self.lanes > 1 else st
                slim_launch(self.net.ctx, d, idx, pool, pool_row, slab, out, ws, self.wsb, ls)
                if s < 3:
                    h = hw >> s
                    row = h * h * slim_act_channels(d["r"], cfg.base_channels[s]) * self.eb
                    slim_scatter(self.net.ctx, out, idx, b, row, self.pools[s + 1],
                                 self.row_elems[s + 1] * self.eb, ls)
                else:
                    slim_scatter(self.net.ctx, out, idx, b, cfg.num_classes * 4, self.logits,
                                 cfg.num_classes * 4, ls)
            if self.lanes > 1:   # join before the next segment gathers from the pools
                for ls in self.lane_streams:
                    st.wait_stream(ls)
        return self.logits[:n]


class NativeStreamExecutor:
    """The same request-stream sequencing as StreamExecutor, run by libslim (slim_stream_*): one
    C-ABI call per stream packs the four segments, stages the request orders and enqueues every
    gather / segment / scatter launch.  Marshalling only; same buffers and lane rule."""

    def __init__(self, net: SlimNet, n_max: int, B_max: int = 256, device=None, lanes: int = 1):
        import ctypes
        from . import _check, load_library
        self.net, self.cfg, self.n_max, self.B_max = net, net.cfg, n_max, B_max
        self.dev = torch.device(device if device is not None else f"cuda:{torch.cuda.current_device()}")
        self.lanes = max(1, int(lanes))
        h = ctypes.c_void_p()
        _check(net.ctx, load_library().slim_stream_create(net.ctx, n_max, B_max, self.lanes, ctypes.byref(h)))
        self.h = h.value
        self.logits = torch.empty(n_max, self.cfg.num_classes, dtype=torch.float32, device=self.dev)
        self.pack_s, self.host_s, self.last_launches, self.last_n_batches = [], [], 0, 0

    def run(self, images: torch.Tensor, tuples: np.ndarray, stream=None) -> torch.Tensor:
        import ctypes
        from . import _check, _stream, load_library, slim_stream_stats
        t = np.ascontiguousarray(np.asarray(tuples, np.float32))
        n = t.shape[0]
        assert n <= self.n_max and t.shape == (n, 4)
        st = slim_stream_stats()
        _check(self.net.ctx, load_library().slim_stream_run(
            self.h, images.data_ptr(), t.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), n, self.logits.data_ptr(),
            _stream(stream if stream is not None else torch.cuda.current_stream(self.dev)), ctypes.byref(st)))
        self.pack_s.append(st.pack_seconds)
        self.host_s.append(st.host_seconds)
        self.last_launches, self.last_n_batches = st.launches, st.batches
        return self.logits[:n]

    def close(self):
        if self.h:
            from . import load_library
            load_library().slim_stream_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
