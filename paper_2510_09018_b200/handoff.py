"""Per-segment cross-device routing with activation hand-off.

The paper's router acts per scheduled block and the request key carries w_prev, so a
request may run segment s on one server and segment s+1 on another (
SPEC routes every segment stage through the router).  Between segments the request's
activation [H_s, H_s, c_act(w_s)] moves to the next device.

Per rank and segment s (all ranks step through the segments together):

  1. compute: the requests routed here for segment s are batched by key with the ABI
     packer (slim_pack) and run with slim_launch (gather kernel + segment kernels); each
     batch's outputs are scattered (slim_scatter) into this rank's pool of segment s+1;
  2. pack: rows of requests whose segment s+1 runs elsewhere are gathered (slim_gather)
     into one send buffer ordered by destination rank, ascending request index;
  3. exchange: one all_to_all_single of those bytes (NCCL over NVLink on the GPUs; gloo on
     CPU in the tests) -- every rank derives every split size from the replicated plan;
  4. unpack: received rows are scattered (slim_scatter) into the pool rows of the requests.

Rows are exchanged at the pool's fixed row size (the widest c_act of the segment), so the
buffers are uniform; the active prefix is what the next segment reads.  The data path
is libslim's kernels and the collective; this module sequences them (host control).
"""
from __future__ import annotations

import numpy as np

from . import slim_act_channels, slim_forward_workspace_bytes, slim_gather, slim_launch, slim_pack, slim_scatter

POLICIES = ("pipeline", "random", "sticky")


def plan_segments(n: int, world: int, policy: str = "random", seed: int = 2510_09018) -> np.ndarray:
    """dev[n, 4]: the rank that runs segment s of request i.  Deterministic in the arguments
    (replicated on every rank).  pipeline: segment s on rank floor(s*world/4); random: uniform
    per (request, segment) (SPEC: every stage routed); sticky: one uniform rank per request."""
    if policy not in POLICIES:
        raise ValueError(f"unknown policy {policy!r}; one of {POLICIES}")
    g = np.random.Generator(np.random.PCG64([seed, 313]))
    if policy == "pipeline":
        return np.tile((np.arange(4) * world) // 4, (n, 1)).astype(np.int64)
    if policy == "random":
        return g.integers(0, world, (n, 4)).astype(np.int64)
    return np.repeat(g.integers(0, world, (n, 1)), 4, axis=1).astype(np.int64)


def exchange_lists(dev: np.ndarray, s: int, rank: int, world: int):
    """Boundary s -> s+1: send[d] = requests leaving this rank for d, recv[src] = requests
    arriving from src (both ascending request index; empty for d == rank)."""
    send = [np.nonzero((dev[:, s] == rank) & (dev[:, s + 1] == d))[0] if d != rank else np.zeros(0, np.int64)
            for d in range(world)]
    recv = [np.nonzero((dev[:, s] == src) & (dev[:, s + 1] == rank))[0] if src != rank else np.zeros(0, np.int64)
            for src in range(world)]
    return send, recv


class CollectiveTransport:
    """all_to_all_single over the default process group (NCCL on GPUs, gloo on CPU)."""

    def exchange(self, send_buf, send_bytes, recv_buf, recv_bytes):
        import torch.distributed as dist
        dist.all_to_all_single(recv_buf, send_buf, output_split_sizes=list(recv_bytes),
                               input_split_sizes=list(send_bytes))
        return recv_buf


class HandoffExecutor:
    """One rank's share of a segment-routed request stream on its GPU."""

    def __init__(self, net, n_max: int, rank: int, world: int, B_max: int = 256, lanes: int = 1):
        import torch
        self.net, self.cfg, self.n_max, self.rank, self.world, self.B_max = net, net.cfg, n_max, rank, world, B_max
        cfg = self.cfg
        self.dev = torch.device(f"cuda:{torch.cuda.current_device()}")
        self.eb = 2 if cfg.dtype == 0 else 4
        self.adt = torch.bfloat16 if cfg.dtype == 0 else torch.float32
        hw, wmax = cfg.image_hw, cfg.widths[cfg.n_widths - 1]
        self.row_elems = [hw * hw * cfg.in_channels] + [
            (hw >> (s - 1)) ** 2 * slim_act_channels(wmax, cfg.base_channels[s - 1]) for s in range(1, 4)]
        self.pools = [None] + [torch.zeros(n_max * self.row_elems[s], dtype=self.adt, device=self.dev)
                               for s in range(1, 4)]
        self.logits = torch.zeros(n_max, cfg.num_classes, dtype=torch.float32, device=self.dev)
        self.wsb = max(slim_forward_workspace_bytes(net.ctx, s, wmax, wmax, B_max) for s in range(4))
        # lanes (as in stream.StreamExecutor): a segment's key batches on one stream per width
        self.lanes = max(1, int(lanes))
        self.lane_buf = [(torch.empty(B_max * max(self.row_elems), dtype=self.adt, device=self.dev),
                          torch.empty(B_max * max(max(self.row_elems[1:]), cfg.num_classes * 4 // self.eb),
                                      dtype=self.adt, device=self.dev),
                          torch.empty(self.wsb, dtype=torch.uint8, device=self.dev)) for _ in range(self.lanes)]
        self.lane_streams = [torch.cuda.Stream(device=self.dev) for _ in range(self.lanes)] if self.lanes > 1 else []
        self.widths = [cfg.widths[i] for i in range(cfg.n_widths)]
        self.stats = dict(sent_rows=0, recv_rows=0, batches=0)

    def _plan(self, tuples: np.ndarray, dev: np.ndarray):
        """Key batching of all four segments and every exchange list (host), with ONE host-to-device
        copy of all slot arrays; cached while (tuples, plan) repeat."""
        key = (hash(tuples.tobytes()), hash(dev.tobytes()))
        if getattr(self, "_pkey", None) == key:
            return self._pc
        parts, segs, off = [], [], 0

        def add(a):
            nonlocal off
            parts.append(np.asarray(a, np.int32))
            off += len(a)
            return off - len(a), len(a)
        for s in range(4):
            mine = np.nonzero(dev[:, s] == self.rank)[0]
            batches = []
            if len(mine):
                reqs = [(int(i), s, float(tuples[i, s]), float(tuples[i, s - 1]) if s else 0.0, int(i)) for i in mine]
                descs, order = slim_pack(self.cfg, reqs, self.B_max)
                batches = [(d, add(mine[order[d["first"]:d["first"] + d["batch"]]])) for d in descs]
            ex = None
            if s < 3 and self.world > 1:
                send, recv = exchange_lists(dev, s, self.rank, self.world)
                ex = (add(np.concatenate(send)), [len(x) for x in send], add(np.concatenate(recv)), [len(x) for x in recv])
            segs.append((batches, ex))
        import torch
        host = torch.from_numpy(np.concatenate(parts) if parts else np.zeros(1, np.int32))
        self._slots_d = host.to(self.dev)
        self._pkey, self._pc = key, segs
        return segs

    def _sl(self, span):
        return self._slots_d[span[0]:span[0] + span[1]]

    def compute(self, s: int, images, tuples: np.ndarray, dev: np.ndarray, stream=None):
        """Run segment s for the requests routed to this rank (key batching + RUNBATCH)."""
        import torch
        cfg, hw = self.cfg, self.cfg.image_hw
        pool = images if s == 0 else self.pools[s]
        main = stream if stream is not None else torch.cuda.current_stream(self.dev)
        if self.lanes > 1:
            fork = torch.cuda.Event()
            fork.record(main)
            for ls in self.lane_streams:
                ls.wait_event(fork)
        per_width = {}
        for d, span in self._plan(np.asarray(tuples, np.float32), dev)[s][0]:
            b = d["batch"]
            slots = self._sl(span)
            # lane = width index, plus (lanes > widths) a rotation over the width's batches (as in stream.py)
            wi = self.widths.index(min(self.widths, key=lambda w: abs(w - d["r"])))
            j = per_width.get(wi, 0)
            per_width[wi] = j + 1
            nw = len(self.widths)
            lane = (wi + nw * (j % max(1, self.lanes // nw))) % self.lanes
            slab, out, ws = self.lane_buf[lane]
            ls = self.lane_streams[lane] if self.lanes > 1 else main
            slim_launch(self.net.ctx, d, slots, pool, self.row_elems[s] * self.eb, slab, out, ws, self.wsb, ls)
            if s < 3:
                row = (hw >> s) ** 2 * slim_act_channels(d["r"], cfg.base_channels[s]) * self.eb
                slim_scatter(self.net.ctx, out, slots, b, row, self.pools[s + 1], self.row_elems[s + 1] * self.eb, ls)
            else:
                slim_scatter(self.net.ctx, out, slots, b, cfg.num_classes * 4, self.logits, cfg.num_classes * 4, ls)
            self.stats["batches"] += 1
        if self.lanes > 1:
            for ls in self.lane_streams:
                main.wait_stream(ls)

    def pack(self, s: int, dev: np.ndarray, stream=None):
        """Send buffer (uint8) of the rows leaving after segment s, and its per-destination byte counts."""
        import torch
        send_span, send_n, _, recv_n = self._pc[s][1]
        row = self.row_elems[s + 1] * self.eb
        n = send_span[1]
        buf = torch.empty(max(n, 1) * row, dtype=torch.uint8, device=self.dev)
        if n:
            slim_gather(self.net.ctx, self.pools[s + 1], self._sl(send_span), n, row, buf, stream)
        self.stats["sent_rows"] += n
        return buf[:n * row], [c * row for c in send_n], [c * row for c in recv_n]

    def unpack(self, s: int, dev: np.ndarray, recv_buf, stream=None):
        _, _, recv_span, _ = self._pc[s][1]
        n = recv_span[1]
        if n:
            row = self.row_elems[s + 1] * self.eb
            slim_scatter(self.net.ctx, recv_buf, self._sl(recv_span), n, row, self.pools[s + 1], row, stream)
        self.stats["recv_rows"] += n

    def run(self, images, tuples, dev: np.ndarray, transport=None, stream=None):
        """All four segments with the hand-offs between them (collective transport).  Returns the
        logits buffer; rows i with dev[i, 3] == rank are this rank's results."""
        import torch
        transport = transport or CollectiveTransport()
        tuples = np.asarray(tuples, np.float32)
        for s in range(4):
            self.compute(s, images, tuples, dev, stream)
            if s < 3 and self.world > 1:
                send_buf, sb, rb = self.pack(s, dev, stream)
                recv_buf = torch.empty(max(sum(rb), 1), dtype=torch.uint8, device=self.dev)
                # rows packed (on the stream compute/pack used) before the collective reads them
                (stream if stream is not None else torch.cuda.current_stream(self.dev)).synchronize()
                transport.exchange(send_buf, sb, recv_buf[:sum(rb)], rb)
                self.unpack(s, dev, recv_buf, stream)
        return self.logits


def run_local(executors, images, tuples, dev: np.ndarray):
    """Every rank in ONE process on one device (tests): compute, pack, an in-process
    all-to-all (rank r receives, in source order, the slices the sources addressed to r), unpack."""
    import torch
    tuples = np.asarray(tuples, np.float32)
    world = len(executors)
    for s in range(4):
        for ex in executors:
            ex.compute(s, images, tuples, dev)
        if s == 3:
            break
        packed = [ex.pack(s, dev) for ex in executors]
        for r, ex in enumerate(executors):
            parts = []
            for src in range(world):
                buf, sb, _ = packed[src]
                off = sum(sb[:r])
                parts.append(buf[off:off + sb[r]])
            recv = torch.cat(parts) if parts else torch.empty(0, dtype=torch.uint8, device=ex.dev)
            ex.unpack(s, dev, recv)
    out = torch.empty_like(executors[0].logits)
    for i, r in enumerate(dev[:, 3]):
        out[i] = executors[int(r)].logits[i]
    return out
