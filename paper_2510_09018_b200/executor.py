"""Alg. 1 greedy segment-slim executor on one GPU.

The native scheduler (`Scheduler`, slim_sched_* in libslim) makes every decision of
Alg. 1 -- FIFO head-key batching, best-fit instance, CANLOAD with the VRAM cap and the
utilisation gate, scale-up, requeue, idle unload.  This loop only carries them out:

* RUN (l.10, RUNBATCH): the batch's rows are gathered from the segment's input pool into
  the instance's slab and the segment runs there (`slim_launch`: gather kernel + forward
  kernels), then its outputs are scattered to the next segment's pool (`slim_scatter`),
  all on the instance's own CUDA stream -- instances run concurrently on the GPU.
* completion: an event per batch; when it has fired the instance is released
  (`complete`) and each request re-enters the queue with the next key
  (s+1, w_{s+1}, w_s), or is finished after segment 3.
* UNLOADERLOOP (l.21-25): removed instances free their buffers; with `offload=True` a
  segment left without instances is unloaded from the device ("offload to CPU, free
  VRAM") and reloaded from the host copy when CANLOAD admits a new instance of it.

Every data movement and all arithmetic run in libslim's kernels; this is host control.
"""
from __future__ import annotations

import time

import numpy as np
import torch

from . import Scheduler, SlimNet, slim_act_channels, slim_forward_workspace_bytes, slim_launch, slim_scatter


class _Instance:
    def __init__(self, ex: "GreedyExecutor"):
        dev, B = ex.dev, ex.B_max
        self.stream = torch.cuda.Stream(device=dev)
        self.slab = torch.empty(B * max(ex.row_elems), dtype=ex.adt, device=dev)
        self.out = torch.empty(B * ex.out_elems, dtype=ex.adt, device=dev)
        self.ws = torch.empty(ex.wsb, dtype=torch.uint8, device=dev)
        self.slots_h = torch.empty(B, dtype=torch.int32).pin_memory()
        self.slots_d = torch.empty(B, dtype=torch.int32, device=dev)
        self.event = torch.cuda.Event()


class GreedyExecutor:
    def __init__(self, net: SlimNet, n_max: int, B_max: int = 256, offload: bool = False, util_fn=None,
                 vram_fn=None, **knobs):
        self.net, self.cfg, self.n_max, self.B_max = net, net.cfg, n_max, B_max
        self.offload = offload
        self.util_fn = util_fn or (lambda: -1.0)      # latest GPU utilisation in [0,1]; -1 = no sample
        # VRAM used besides the instances' weight slices: torch's allocations (pools, instance buffers)
        self.vram_fn = vram_fn or (lambda: torch.cuda.memory_allocated(self.dev))
        self.sched = Scheduler(net.cfg, B_max=B_max, **knobs)
        self.dev = torch.device(f"cuda:{torch.cuda.current_device()}")
        cfg = self.cfg
        self.eb = 2 if cfg.dtype == 0 else 4
        self.adt = torch.bfloat16 if cfg.dtype == 0 else torch.float32
        hw, wmax = cfg.image_hw, cfg.widths[cfg.n_widths - 1]
        self.row_elems = [hw * hw * cfg.in_channels]
        for s in range(1, 4):
            h = hw >> (s - 1)
            self.row_elems.append(h * h * slim_act_channels(wmax, cfg.base_channels[s - 1]))
        self.out_elems = max(max(self.row_elems[1:]), cfg.num_classes * 4 // self.eb)
        self.wsb = max(slim_forward_workspace_bytes(net.ctx, s, wmax, wmax, B_max) for s in range(4))
        self.pools = [None] + [torch.empty(n_max * self.row_elems[s], dtype=self.adt, device=self.dev)
                               for s in range(1, 4)]
        self.logits = torch.empty(n_max, cfg.num_classes, dtype=torch.float32, device=self.dev)
        self.inst = {}            # instance id -> _Instance (buffers + stream)
        self.stats = dict(batches=0, loads=0, requeues=0, unloaded=0, seg_reloads=0, batch_sizes=[], t_next=0.0,
                          t_launch=0.0, t_wait=0.0)

    # --------------------------------------------------------------- RUNBATCH
    def _run(self, act, images, tuples):
        iid, s, b = act["inst"], act["seg"], act["batch"]
        if iid not in self.inst:
            self.inst[iid] = _Instance(self)
        if self.offload and not self.net.segment_loaded(s):
            self.net.load_segment(s)               # reload an offloaded segment (CANLOAD admitted it)
            self.stats["seg_reloads"] += 1
        I = self.inst[iid]
        slots = act["slots"].astype(np.int32)
        I.slots_h[:b].copy_(torch.from_numpy(slots))
        with torch.cuda.stream(I.stream):
            I.slots_d[:b].copy_(I.slots_h[:b], non_blocking=True)
            pool = images if s == 0 else self.pools[s]
            d = dict(seg=s, r_prev=act["w_prev"], r=act["w_req"], batch=b, first=0)
            ctx, hw, cfg = self.net.ctx, self.cfg.image_hw, self.cfg
            st = I.stream.cuda_stream
            slim_launch(ctx, d, I.slots_d, pool, self.row_elems[s] * self.eb, I.slab, I.out, I.ws, self.wsb, st)
            if s < 3:
                h = hw >> s
                row = h * h * slim_act_channels(act["w_req"], cfg.base_channels[s]) * self.eb
                slim_scatter(ctx, I.out, I.slots_d, b, row, self.pools[s + 1], self.row_elems[s + 1] * self.eb, st)
            else:
                slim_scatter(ctx, I.out, I.slots_d, b, cfg.num_classes * 4, self.logits, cfg.num_classes * 4, st)
            I.event.record(I.stream)
        self.pending[iid] = (s, act["ids"].astype(np.int64))
        self.stats["batches"] += 1
        self.stats["batch_sizes"].append(b)

    def _reap(self, now, tuples, block: bool) -> int:
        """Release instances whose batch finished; re-enqueue their requests for the next segment."""
        t0 = time.perf_counter()
        done = [iid for iid in self.pending if self.inst[iid].event.query()]
        while not done and block and self.pending:   # wait for whichever batch finishes first
            done = [iid for iid in self.pending if self.inst[iid].event.query()]
        self.stats["t_wait"] += time.perf_counter() - t0
        finished = 0
        for iid in done:
            s, ids = self.pending.pop(iid)
            self.sched.complete(iid, now)
            if s < 3:
                self.sched.enqueue([(int(i), s + 1, float(tuples[i, s + 1]), float(tuples[i, s]), int(i))
                                    for i in ids], now)
            else:
                finished += len(ids)
        return finished

    def _unload(self, now) -> int:
        removed = self.sched.unload_idle(now)
        for iid in removed:
            self.inst.pop(iid, None)
            self.stats["unloaded"] += 1
        if self.offload:
            live = {i["seg"] for i in self.sched.instances()}
            for s in range(4):
                if s not in live and self.net.segment_loaded(s):
                    torch.cuda.synchronize(self.dev)   # no batch of segment s may be in flight
                    self.net.unload_segment(s)
        return len(removed)

    def _wait_idle(self, now) -> bool:
        """Requeued with every instance idle: sleep until the oldest idle instance reaches t_idle."""
        idle = [i for i in self.sched.instances() if not i["busy"]]
        if not idle:
            return False
        t = min(i["t_last"] for i in idle) + self.sched.k.t_idle_s - now
        time.sleep(max(t, 0.0) + 1e-4)
        return True

    # --------------------------------------------------------------- LOOP
    def run(self, images: torch.Tensor, tuples) -> torch.Tensor:
        """images: device [n, H, W, C] (activation dtype); tuples: [n, 4] widths per segment.
        Returns fp32 logits [n, classes] in request order."""
        tuples = np.asarray(tuples, np.float32)
        n = images.shape[0]
        assert n <= self.n_max and tuples.shape == (n, 4)
        images = images.contiguous()
        torch.cuda.current_stream(self.dev).synchronize()   # inputs written before the instance streams read
        t0 = time.perf_counter()
        clock = lambda: time.perf_counter() - t0
        self.sched.enqueue([(i, 0, float(tuples[i, 0]), 0.0, i) for i in range(n)], 0.0)
        self.pending = {}
        finished = 0
        while finished < n:
            now = clock()
            act = self.sched.next(now, self.util_fn(), self.vram_fn())
            self.stats["t_next"] += clock() - now
            self.stats["loads"] += act["n_loaded"]
            if act["kind"] == "run":
                t1 = clock()
                self._run(act, images, tuples)
                self.stats["t_launch"] += clock() - t1
                finished += self._reap(clock(), tuples, block=False)
                continue
            if act["kind"] == "requeue":
                self.stats["requeues"] += 1
                if not self.pending:   # nothing will free up by itself: only the unloader can help
                    if self._unload(clock()) == 0 and not self._wait_idle(clock()):
                        raise RuntimeError("Alg. 1 deadlock: no instance can be loaded (M_max / U_blk) and none is busy")
                    continue
            finished += self._reap(clock(), tuples, block=True)
            self._unload(clock())
        for I in self.inst.values():
            I.stream.synchronize()
        return self.logits[:n]
