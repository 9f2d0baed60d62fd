#!/usr/bin/env python
"""bench.py -- images/s of the width-sliced SlimResNet forward on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1], "CFG2"): the full segmented SlimResNet
(4 segments + pool/FC, 100 classes) at each width ratio r in {0.25, 0.5, 0.75, 1.0},
batch 128, synthetic CIFAR-100-shaped 32x32x3 inputs, random-init weights
(synth/, seeded).  One STEP = one full-chain forward of a 128-image batch at
every width (512 images), through the C-ABI (slim_forward_chain, CUDA-graph
replay).  Multi-GPU (torchrun, one rank per GPU): every rank runs its own
batches (weak scaling, no data-path collective) and all-gathers a float32[8]
telemetry record per step over NCCL on a side stream (north_star).

Timing: W warm-up steps, then K steps, each bracketed by CUDA events on the
launching stream; L2 is flushed (256 MiB write) before every timed step, outside
the events; barrier + synchronize around the region; max over ranks.

`--impl reference` times the fp64 CPU oracle (oracle/) on a bounded sample of the
same workload (one image per width per step) -- the base contract's reference arm
for a tier with no reference implementation.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "SlimResNet images/s per width at 1/2/4/8 B200; tensor-pipe % of peak"
WIDTHS = (0.25, 0.5, 0.75, 1.0)


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(hbm=d["hbm_gbs"], bf16=d["bf16_tflops"], bf16_sus=d.get("bf16_tflops_sustained"),
                    src="measured (MEASURED_PEAKS.json)")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="fallback (B200_PROFILING.md)")


def sm_shares(widths, spec: str):
    """Per-width SM shares for the concurrent width instances (slim_set_sm_share).  auto: share(r) =
    0.1 + 0.4 r, clamped to (0, 1] (fitted to the B=128 sweeps in profiles/r01_sm_share_sweep.txt:
    0.2 / 0.3 / 0.4 / 0.5 of the SMs for r = .25 / .5 / .75 / 1 -- the shares overlap, their sum is
    1.4; ~1.24 M images/s vs 0.88 M with every kernel on all SMs); none: every width may use all
    SMs; else a comma list, one share per width."""
    if spec == "none":
        return {r: 1.0 for r in widths}
    if spec == "auto":
        return {r: min(1.0, max(0.05, 0.1 + 0.4 * r)) for r in widths}
    vals = [float(v) for v in spec.split(",")]
    assert len(vals) == len(widths), "--sm-share needs one value per width"
    return dict(zip(widths, vals))


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


# ------------------------------------------------------------------ CPU oracle legs
def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform
    return platform.processor() or "unknown"


def oracle_protocol(norm: str = "bn", widths=WIDTHS, budget_s: float = 30.0):
    """SURVEY §8(d) "Oracle beside it": the fp64 oracle (oracle/, as it stands) on this host, on the
    same workload definitions, all threads and 1 thread; CPU model and thread counts recorded.

    * CFG2 = CFG3 at B = 128: the full chain per width, all threads (the line's cpu_baseline value
      blends the four widths like the GPU step: 4 x 128 images / total seconds);
    * CFG3 at B in {1, 8} per width, all threads;
    * CFG2 per width single-threaded (a 4-image sample per width -- CPU cost is linear in B);
    * CFG1 exactly (segment 0, r = 0.25, B = 8), all threads and 1 thread.
    The oracle computes in fp64 (reading R15; the north_star names an FP32 oracle)."""
    import oracle
    import synth
    m = oracle.Model(synth.make_weights(), synth.make_bn(widths=widths), norm=norm, widths=widths)
    x = synth.make_images(128, offset=1)
    nthr = oracle.max_threads()
    m.chain(x[:1], (widths[0],) * 4)                    # warm-up: library load, thread pool
    t_start = time.perf_counter()

    def timed(fn):
        t0 = time.perf_counter()
        fn()
        return time.perf_counter() - t0

    out = {"cpu_model": _cpu_model(), "threads_all": nthr, "precision": "fp64 (reading R15; NS names FP32)"}
    cfg3 = {}
    for B in (1, 8, 128):
        for r in widths:
            if time.perf_counter() - t_start > budget_s and B == 128:
                break
            dt = timed(lambda: m.chain(x[:B], (r,) * 4))
            cfg3[f"B{B}_r{r:g}"] = B / dt
    out["cfg3_images_per_s_all_threads"] = cfg3
    full = [r for r in widths if f"B128_r{r:g}" in cfg3]
    out["cfg2_images_per_s_all_threads"] = {str(r): cfg3[f"B128_r{r:g}"] for r in full}
    seconds = sum(128 / cfg3[f"B128_r{r:g}"] for r in full)
    out["cfg2_blended_images_per_s"] = 128 * len(full) / seconds if full else None
    out["cfg1_us_all_threads"] = 1e6 * min(timed(lambda: m.segment(0, x[:8], None, 0.25)) for _ in range(3))
    oracle.set_num_threads(1)
    try:
        out["cfg1_us_1_thread"] = 1e6 * timed(lambda: m.segment(0, x[:8], None, 0.25))
        out["cfg2_images_per_s_1_thread"] = {str(r): 4 / timed(lambda: m.chain(x[:4], (r,) * 4)) for r in widths}
    finally:
        oracle.set_num_threads(nthr)
    out["seconds"] = time.perf_counter() - t_start
    return out


def oracle_throughput(norm: str = "bn", widths=WIDTHS, budget_s: float = 30.0):
    """cpu_baseline of the bench line: the protocol above; value = CFG2 blended over the widths."""
    p = oracle_protocol(norm, widths, budget_s)
    return dict(value=p["cfg2_blended_images_per_s"], unit="images/s", cores=p["threads_all"], kind="oracle",
                sample=f"CFG2: the full chain at B=128 for each width (all {p['threads_all']} threads of "
                       f"{p['cpu_model']}), fp64 C oracle; {p['seconds']:.1f} s incl. the rest of the protocol",
                protocol=p)


def run_reference(args):
    """--impl reference: the oracle as it stands, on this arm's config/metric/unit; each step = a bounded
    sample of CFG2 (args.ref_batch images per width through the full chain), all host threads."""
    world, rank, _ = _dist()
    if rank != 0:
        return 0
    import oracle
    import synth
    m = oracle.Model(synth.make_weights(), synth.make_bn(), norm=args.norm)
    nb = args.ref_batch
    x = synth.make_images(128, offset=1)
    step = lambda k: [m.chain(x[(k * nb) % 128:(k * nb) % 128 + nb], (r,) * 4) for r in WIDTHS]
    for k in range(args.warmup):
        step(k)
    t0 = time.perf_counter()
    for k in range(args.steps):
        step(k)
    dt = time.perf_counter() - t0
    imgs = nb * len(WIDTHS) * args.steps
    value = imgs / dt
    cores = oracle.max_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": 0,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "CFG2: full SlimResNet chain (4 segments + pool/FC, 100 classes) at each width "
                               f"r in {{0.25,0.5,0.75,1.0}}; reference step = {nb} images per width", "batch": nb,
                   "image": [32, 32, 3], "widths": list(WIDTHS), "norm": args.norm},
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": cores, "kind": "oracle",
                         "cpu_model": _cpu_model(),
                         "sample": f"{args.steps} steps x {nb} images per width of the CFG2 chain (fp64)"},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


class Cfg2Step:
    """The CFG2 step bench.py times (BASELINE configs[1]): one full-chain forward of a B-image batch at
    every width, the width instances on their own CUDA streams (concurrently, on per-width SM shares),
    CUDA-graph replay.  tests/test_gpu_bench_step.py builds the same object from bench.py's default
    arguments and checks its logits against the oracle."""

    def __init__(self, args, dev, rank: int = 0):
        import torch

        import synth
        import paper_2510_09018_b200 as slim
        self.slim = slim
        self.B = B = args.batch
        self.widths = WIDTHS = tuple(args.widths)   # default: the paper's set; others = universal widths (NEXT-4)
        weights, bn = synth.make_weights(), synth.make_bn(widths=WIDTHS)
        self.net = net = slim.SlimNet(weights, bn, device=dev.index, max_batch=max(B, 16), norm=args.norm,
                                      widths=WIDTHS, dtype=args.dtype)
        adt = torch.bfloat16 if args.dtype == "bf16" else torch.float32
        if not args.no_graph:
            slim.slim_set_graph_mode(net.ctx, True)
        self.stream = stream = torch.cuda.current_stream(dev)
        self.image_offsets = {r: 100 + rank * 8 + i for i, r in enumerate(WIDTHS)}
        self.xs = {r: torch.from_numpy(synth.make_images(B, offset=self.image_offsets[r])).to(adt).to(dev)
                   for r in WIDTHS}
        self.logits = {r: torch.empty(B, 100, dtype=torch.float32, device=dev) for r in WIDTHS}
        self.wsb = max(slim.slim_chain_workspace_bytes(net.ctx, (r,) * 4, B) for r in WIDTHS)
        # one workspace and one stream per width instance: the four (segment-chain, width)
        # instances of a step serve their batches concurrently (Alg. 1 runs every loaded
        # instance independently); --sequential runs them one after another
        self.wss = {r: torch.empty(self.wsb, dtype=torch.uint8, device=dev) for r in WIDTHS}
        # --stream-priority wide: the wider (longer) chains' streams get higher CUDA priority
        prio = {r: 0 for r in WIDTHS}
        if args.stream_priority in ("wide", "narrow"):
            for i, r in enumerate(sorted(WIDTHS, reverse=args.stream_priority == "wide")):
                prio[r] = -max(0, 2 - i)
        self.streams = {r: (stream if args.sequential else torch.cuda.Stream(device=dev, priority=prio[r]))
                        for r in WIDTHS}
        self.order = sorted(WIDTHS, reverse=args.launch_order == "desc")
        # FP32 mode: the SIMT GEMMs are compute-bound on every SM -- shares measured 5 % slower
        self.shares = sm_shares(WIDTHS, "none" if (args.sequential or len(WIDTHS) == 1 or args.dtype == "fp32")
                                else args.sm_share)
        self.set_shares(self.shares)

    def chain(self, r, st=None):
        self.slim.slim_forward_chain(self.net.ctx, (r,) * 4, self.B, self.xs[r], self.logits[r], self.wss[r],
                                     self.wsb, st if st is not None else self.streams[r])

    def step(self, events=None):
        """One step; events: optional {r: (start, end)} CUDA events recorded around each width's chain
        on that width's stream."""
        import torch
        fork = torch.cuda.Event()
        fork.record(self.stream)
        for r in self.order:
            self.streams[r].wait_event(fork)
            if events is not None:
                events[r][0].record(self.streams[r])
            self.chain(r)
            if events is not None:
                events[r][1].record(self.streams[r])
        for r in self.widths:
            self.stream.wait_stream(self.streams[r])

    def set_shares(self, sh):
        for r in self.widths:
            self.slim.slim_set_sm_share(self.net.ctx, r, sh[r])


_BACKEND = {"name": "nccl"}


def _coll_dev(dev):
    """Device of tensors handed to collectives: the GPU for NCCL, the host for gloo."""
    return dev if _BACKEND["name"] == "nccl" else "cpu"


def _init_nccl(dev):
    """Process group (NCCL over NVLink, one rank per GPU; `--dist-backend gloo` is the functional check
    for several ranks sharing a GPU -- NCCL refuses that); returns a record proving the communicator
    spans every rank (an all-reduce of ones == world size)."""
    import torch
    import torch.distributed as dist
    if _BACKEND["name"] == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group("gloo")
    one = torch.ones(1, device=_coll_dev(dev))
    dist.all_reduce(one)
    torch.cuda.synchronize(dev)
    rec = {"backend": dist.get_backend(), "world": dist.get_world_size(), "rank": dist.get_rank(),
           "allreduce_ones": int(one.item()), "nccl_version": ".".join(map(str, torch.cuda.nccl.version()))}
    rec["comm_nranks_ok"] = rec["allreduce_ones"] == rec["world"]
    print(f"[rank {rec['rank']}] process group up: {rec}", file=sys.stderr, flush=True)
    return rec


# ------------------------------------------------------------------ GPU arm
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2510_09018_b200 as slim
    from paper_2510_09018_b200 import build as slim_build
    from paper_2510_09018_b200.telemetry import NvmlSampler, TelemetryExchange, TelemetrySource

    world, rank, local = _dist()
    assert torch.cuda.is_available(), "bench.py (ours) needs a GPU; the oracle arm is --impl reference"
    local = local % torch.cuda.device_count()   # (gloo functional check: several ranks on one GPU)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    nccl = _init_nccl(dev) if world > 1 else None
    slim_build.build()

    cfg2 = Cfg2Step(args, dev, rank)
    B, WIDTHS, net, xs, logits = cfg2.B, cfg2.widths, cfg2.net, cfg2.xs, cfg2.logits
    stream, streams, wss, wsb = cfg2.stream, cfg2.streams, cfg2.wss, cfg2.wsb
    chain, step, shares, set_shares = cfg2.chain, cfg2.step, cfg2.shares, cfg2.set_shares
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2
    sampler = NvmlSampler(local)
    telem = TelemetryExchange(device=_coll_dev(dev)) if world > 1 else None
    tsrc = TelemetrySource(sampler, rank)
    imgs_per_step = B * len(WIDTHS)
    last_ms = [0.0]

    def tick(k, ev):
        """Router tick after step k: this rank's record (NVML power / util / energy from the sampler
        thread, latency of the newest completed step) all-gathered over NCCL on a side stream."""
        if telem is None:
            return
        for j in range(k, max(-1, k - 4), -1):           # newest step whose end event has completed
            if ev[j][1].query():
                last_ms[0] = ev[j][0].elapsed_time(ev[j][1])
                break
        telem.tick(tsrc.record(queue_len=0.0, mean_latency_s=last_ms[0] / 1e3, completed=(k + 1) * imgs_per_step))

    set_shares(shares)
    sampler.start()
    wev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(max(4, args.warmup))]
    for k in range(args.warmup):
        flush.zero_()
        wev[k % 4][0].record(stream)
        step()
        wev[k % 4][1].record(stream)
        tick(k % 4, wev) if telem else None
    torch.cuda.synchronize()

    # ---------------- timed region: K steps, events on the launching stream; per-width events on the
    # width instances' own streams (the per-width numbers of the timed mode)
    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    evw = [{r: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for r in WIDTHS}
           for _ in range(K)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = slim.slim_launch_count(net.ctx)
    ns0 = len(sampler.samples)
    for k in range(K):
        flush.zero_()
        ev[k][0].record(stream)
        step()
        ev[k][1].record(stream)
        tick(k, ev)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    timed_samples = len(sampler.samples) - ns0
    launches = slim.slim_launch_count(net.ctx) - launches0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device=_coll_dev(dev))
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_max_ms = float(t.item())
    value = world * imgs_per_step * K / (total_max_ms / 1e3)
    # per-width time inside the concurrent step: the same step again (outside the timed region, events on
    # each width's stream around its chain; recording them costs ~6 % of the step, so not in the timed loop)
    in_step_ms = None
    if args.width_events:
        for k in range(K):
            flush.zero_()
            step(evw[k])
        torch.cuda.synchronize()
        in_step_ms = {r: float(np.mean([e[r][0].elapsed_time(e[r][1]) for e in evw])) for r in WIDTHS}

    # ---------------- energy (Eq. 7's E_t = P * L): the same step, L2 flush included, in a loop
    # of >= args.energy_seconds; NVML total-energy counter delta / images.  Clocks sampled throughout.
    torch.cuda.synchronize()
    e0 = sampler.energy_mj()
    t0 = time.perf_counter()
    n_energy = 0
    while args.energy_seconds > 0:
        for _ in range(50):
            flush.zero_()
            step()
        n_energy += 50
        if n_energy % 500 == 0:
            torch.cuda.synchronize()
            if time.perf_counter() - t0 >= args.energy_seconds:
                break
    torch.cuda.synchronize()
    energy_s = time.perf_counter() - t0
    e1 = sampler.energy_mj()
    sampler.stop()
    clocks = sampler.summary()
    clocks["samples_timed_region"] = timed_samples
    clocks["note"] = (f"sampled every {sampler.period * 1e3:.0f} ms over warm-up, the timed region and the "
                      f"{energy_s:.1f} s energy loop of the same step")
    energy = ({"j_per_image": (e1 - e0) / 1e3 / (imgs_per_step * n_energy), "seconds": energy_s,
               "images": imgs_per_step * n_energy, "mean_power_w": (e1 - e0) / 1e3 / energy_s,
               "images_per_s_in_loop": imgs_per_step * n_energy / energy_s,
               "method": "nvmlDeviceGetTotalEnergyConsumption delta over the loop (host wall clock)"}
              if (e0 is not None and e1 is not None and e1 > e0 and n_energy > 0) else None)

    # ---------------- per-launch records (eager, an event pair around every launch, PDL off) of the SAME
    # step configuration (the widths' SM shares select the same kernels as in the timed step): the
    # algorithmic FLOPs/bytes of every kernel and its standalone duration -> the kernels' shares
    KP = max(1, min(K, args.profile_steps))
    slim.slim_profile_begin(net.ctx, KP * 80 * len(WIDTHS) + 16)
    for _ in range(KP):
        flush.zero_()
        for r in WIDTHS:
            chain(r, stream)
    recs = slim.slim_profile_end(net.ctx)
    # ---------------- per-width: each width's chain alone (L2 flushed before it), on all SMs, graph replay
    # with PDL -- the same kernels as the step without the other instances
    set_shares({r: 1.0 for r in WIDTHS})
    KW = max(3, min(K, args.profile_steps * 4))
    width_ms = {}
    for r in WIDTHS:
        chain(r, stream)   # (re)capture the graph outside the timed events
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(KW)]
        for k in range(KW):
            flush.zero_()
            evs[k][0].record(stream)
            chain(r, stream)
            evs[k][1].record(stream)
        torch.cuda.synchronize()
        width_ms[r] = sum(x.elapsed_time(y) for x, y in evs) / KW

    peaks = _peaks()
    if args.dtype == "fp32":
        # FP32 mode runs on the CUDA cores (FFMA): peak = 148 SMs x 128 FP32 lanes x 2 FLOP x 1.965 GHz
        # (B200 unit counts and the max SM clock of this pool) -- an ALU roofline
        peaks = dict(peaks, bf16=148 * 128 * 2 * 1.965e9 / 1e12, bf16_sus=None, src="derived (FFMA lanes x clock)")
    P_tc, P_hbm = peaks["bf16"] * 1e12, peaks["hbm"] * 1e9
    by_kind, by_width = {}, {}
    for rc in recs:
        roof = max(rc["flops"] / P_tc, rc["bytes"] / P_hbm) * 1e3
        for key, tab in ((rc["kind"], by_kind), (rc["r"], by_width)):
            d = tab.setdefault(key, dict(ms=0.0, flops=0.0, bytes=0.0, n=0, roof_ms=0.0))
            d["ms"] += rc["ms"]
            d["flops"] += rc["flops"]
            d["bytes"] += rc["bytes"]
            d["n"] += 1
            d["roof_ms"] += roof
    kern_ms = sum(d["ms"] for d in by_kind.values())
    dom = max(by_kind, key=lambda k: by_kind[k]["ms"])
    D = by_kind[dom]
    step_ms_mean = total_max_ms / K
    share = D["ms"] / kern_ms
    conv_flops_step = D["flops"] / KP
    # dominant kernel in the TIMED step: its algorithmic FLOPs per step / (step time x its share of the
    # kernel time); launches per step from the same records
    achieved = conv_flops_step / (step_ms_mean * share / 1e3) / 1e12
    bound = "tensor" if args.dtype == "bf16" else "alu"
    roof = {"bound": bound, "achieved": achieved, "peak": peaks["bf16"], "unit": "TFLOP/s",
            "frac": achieved / peaks["bf16"],
            "traffic": _ncu_traffic() if args.dtype == "bf16" else None,
            "kernel": f"{dom} (every tcgen05 conv launch of the step)" if args.dtype == "bf16" else dom,
            "how": "achieved = the dominant kernel's algorithmic FLOPs per step / (ms_per_step x its share of "
                   "the summed kernel time); share from the per-launch records (events around each launch), "
                   "to agree with the ncu launch list's share (profiles/)",
            "share_of_kernel_time": share, "launches_per_step": D["n"] / KP,
            "algorithmic_flops_per_launch": D["flops"] / D["n"], "algorithmic_bytes_per_launch": D["bytes"] / D["n"],
            "peak_source": peaks["src"] + (", bf16 burst" if args.dtype == "bf16" else "")}
    if peaks.get("bf16_sus"):
        roof["frac_vs_sustained_peak"] = achieved / peaks["bf16_sus"]
    roof["step_aggregate"] = {"tflops": sum(r_["flops"] for r_ in recs) / KP / (step_ms_mean / 1e3) / 1e12,
                              "note": "all algorithmic FLOPs of a step (every kernel) / the device-timed step"}
    roof["step_aggregate"]["frac"] = roof["step_aggregate"]["tflops"] / peaks["bf16"]
    roof["standalone_per_launch"] = {
        "tflops": D["flops"] / (D["ms"] / 1e3) / 1e12, "frac": D["flops"] / (D["ms"] / 1e3) / 1e12 / peaks["bf16"],
        "per_layer_roofline_frac": D["roof_ms"] / D["ms"],
        "note": "each launch timed alone (eager, PDL off, events around it): latency-chain view of B=128 kernels"}
    roof["tensor_pipe_pct_ncu"] = _ncu_tensor_pipe() if args.dtype == "bf16" else None
    roof["by_kind_standalone"] = {k: {"launches_per_step": d["n"] / KP, "ms_per_step": d["ms"] / KP,
                                      "tflops": d["flops"] / (d["ms"] / 1e3) / 1e12,
                                      "gbs": d["bytes"] / (d["ms"] / 1e3) / 1e9,
                                      "per_layer_roofline_frac": d["roof_ms"] / d["ms"]} for k, d in by_kind.items()}
    # per width: images/s in the timed (concurrent) step and alone, and the fraction of the per-layer
    # roofline (sum over launches of max(F/P_tc, bytes/P_hbm) / measured time)
    per_width = {}
    for r in WIDTHS:
        d = by_width.get(r, by_width.get(float(np.float32(r))))
        roof_ms = d["roof_ms"] / KP if d else None
        per_width[str(r)] = {} if in_step_ms is None else {
            "images_per_s_in_step": B / (in_step_ms[r] / 1e3), "ms_in_step": in_step_ms[r],
            "per_layer_roofline_frac_in_step": roof_ms / in_step_ms[r] if roof_ms else None}
        per_width[str(r)].update({
            "images_per_s_alone": B / (width_ms[r] / 1e3), "ms_alone": width_ms[r],
            "per_layer_roofline_frac_alone": roof_ms / width_ms[r] if roof_ms else None,
            "per_layer_roofline_ms": roof_ms, "gflop_per_batch": d["flops"] / KP / 1e9 if d else None,
            "tflops_alone": d["flops"] / KP / (width_ms[r] / 1e3) / 1e12 if d else None})

    # ---------------- e2e through the public API with host buffers
    # Every step copies its images from pinned host memory and reads its logits back.  As a
    # serving loop would, the H2D copy of step k+1 runs on a copy stream into the other of two
    # device input buffers while step k computes (events order buffer reuse).
    xh = {r: xs[r].cpu().pin_memory() for r in WIDTHS}
    lh = {r: [torch.empty(B, 100, dtype=torch.float32).pin_memory() for _ in range(2)] for r in WIDTHS}
    xin = {r: [xs[r], torch.empty_like(xs[r])] for r in WIDTHS}
    cstreams = {r: torch.cuda.Stream(device=dev) for r in WIDTHS}
    ev_ready = {r: [torch.cuda.Event(), torch.cuda.Event()] for r in WIDTHS}
    ev_free = {r: [torch.cuda.Event(), torch.cuda.Event()] for r in WIDTHS}
    KE = max(1, min(K, args.e2e_steps))
    set_shares(shares)
    for _ in range(2):   # warm both input buffers' graphs
        for r in WIDTHS:
            for b in range(2):
                slim.slim_forward_chain(net.ctx, (r,) * 4, B, xin[r][b], logits[r], wss[r], wsb, streams[r])
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(KE):
        b = k & 1
        flush.zero_()                                  # L2 flushed between steps, as in the device-timed loop
        fork = torch.cuda.Event()
        fork.record(stream)
        for r in WIDTHS:
            cs, st = cstreams[r], streams[r]
            st.wait_event(fork)
            cs.wait_event(ev_free[r][b])              # the chain that last read buffer b is done
            with torch.cuda.stream(cs):
                xin[r][b].copy_(xh[r], non_blocking=True)
                ev_ready[r][b].record(cs)
            st.wait_event(ev_ready[r][b])
            slim.slim_forward_chain(net.ctx, (r,) * 4, B, xin[r][b], logits[r], wss[r], wsb, st)
            ev_free[r][b].record(st)
            with torch.cuda.stream(st):
                lh[r][b].copy_(logits[r], non_blocking=True)
    for r in WIDTHS:
        streams[r].synchronize()
        cstreams[r].synchronize()
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], dtype=torch.float64, device=_coll_dev(dev))
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_val = world * imgs_per_step * KE / float(te.item())
    gathered = telem.gathered().tolist() if telem else None

    if rank == 0:
        cpu = oracle_throughput(norm=args.norm, widths=WIDTHS, budget_s=args.cpu_seconds) \
            if (world == 1 and not args.no_cpu) else None
        line = {
            "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": total_max_ms / K, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": args.dtype if args.dtype == "bf16" else "f32",
            "data": "synthetic (seeded N(0,1) images, random-init weights)",
            "config": {"workload": "CFG2: full SlimResNet chain (4 segments + pool/FC, 100 classes) at each width "
                                   f"r in {{{','.join(f'{r:g}' for r in WIDTHS)}}}, batch {B} per width, "
                                   f"1 step = {len(WIDTHS)} x {B} images",
                       "batch": B, "image": [32, 32, 3], "widths": list(WIDTHS), "norm": args.norm,
                       "parallelism": f"dp{world} (independent per-GPU batches)",
                       "l2": "flushed (256 MiB write) before every timed step", "graphs": not args.no_graph,
                       "instances": "sequential" if args.sequential else
                                    f"{len(WIDTHS)} width instances, one CUDA stream each, run concurrently",
                       "sm_share": {str(r): v for r, v in shares.items()}},
            "per_width": per_width,
            "per_width_images_per_s": {k: v.get("images_per_s_in_step", v["images_per_s_alone"])
                                       for k, v in per_width.items()},
            "roofline": roof,
            "kernel_time_by_kind_ms_per_step_standalone": {k: v["ms"] / KP for k, v in by_kind.items()},
            "gpu_launches": launches,
            **({"nccl": nccl, "telemetry_allgather_us_mean": 1e3 * float(np.mean(telem.gather_ms))
                if telem.gather_ms else None, "telemetry_ticks_timed": len(telem.gather_ms),
                "telemetry_last_gathered": gathered} if telem else {}),
            "energy_j_per_image": energy["j_per_image"] if energy else None,
            "energy": energy,
            "clocks": clocks,
            "e2e": {"value": e2e_val, "unit": "images/s", "h2d_bytes_per_step": sum(x.numel() * 2 for x in xh.values()),
                    "d2h_bytes_per_step": sum(l[0].numel() * 4 for l in lh.values()),
                    "api": "slim_forward_chain with a pinned-host input copy (double-buffered on a copy stream) + logits read-back every step; L2 flushed every step (inside the wall-clock)"},
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))
        if args.json_out:
            with open(args.json_out, "w") as f:
                json.dump(dict(line, profile=recs[:200]), f, indent=1)
    net.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _clock_energy_json(sampler, e0, e1, n_images):
    return sampler.summary(), (((e1 - e0) / 1e3 / n_images) if (e0 is not None and e1 is not None) else None)


def run_stream(args):
    """CFG4 (N=1) / CFG5 (torchrun N>1): the mixed-width request stream through the key packer,
    gather, segment forwards and scatter; requests routed to ranks by a replicated policy.

    Every step routes a FRESH stream of --requests x N requests (the policy's draw for that step;
    --repeat-stream replays step 0's), so the router and the packer (slim_pack on all four segments)
    run inside the timed region.  --policy ppo_frozen routes with the frozen factored PPO policy on the
    telemetry all-gathered two ticks earlier (fixed lag: identical on every rank, no GPU wait)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    import paper_2510_09018_b200 as slim
    from paper_2510_09018_b200 import build as slim_build
    from paper_2510_09018_b200 import router
    from paper_2510_09018_b200.stream import NativeStreamExecutor, StreamExecutor
    from paper_2510_09018_b200.telemetry import NvmlSampler, TelemetryExchange, TelemetrySource

    world, rank, local = _dist()
    local = local % torch.cuda.device_count()   # (gloo functional check: several ranks on one GPU)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    nccl = _init_nccl(dev) if world > 1 else None
    slim_build.build()
    net = slim.SlimNet(synth.make_weights(), synth.make_bn(), device=local, max_batch=args.bmax, norm=args.norm)
    greedy = args.executor == "greedy"
    native = args.executor == "native"
    if (greedy or native) and args.alg1_shares:   # opt-in: partition the SMs by width as in cfg2
        for r, sh in sm_shares(tuple(net.cfg.widths[i] for i in range(net.cfg.n_widths)), args.sm_share).items():
            slim.slim_set_sm_share(net.ctx, r, sh)
    # Alg. 1 executors: eager launches by default -- their batches land on whichever instance is free, so
    # (key, batch size, instance buffers) combinations keep changing and graph capture would dominate
    # stream executor: CUDA graphs pay off only when batch shapes repeat (--repeat-stream); a fresh
    # stream changes every key's batch size each step, so eager launches (no per-step capture)
    graphs = args.alg1_graphs if (greedy or native) else (
        args.repeat_stream if args.stream_graphs == "auto" else args.stream_graphs == "on")
    slim.slim_set_graph_mode(net.ctx, graphs)
    n_total = args.requests * world
    n_max = n_total                                   # a rank may receive up to the whole stream
    x = torch.from_numpy(synth.make_images(n_max, offset=200 + rank)).to(torch.bfloat16).to(dev)
    if native:   # Alg. 1 with the LOOP itself in C++ (slim_exec_*)
        nx = slim.NativeExecutor(net, n_max=n_max, B_max=args.bmax, Q_th=args.q_th, N_new=args.n_new)

        class _NAdapter:
            last_batches = [[]]
            pack_s = []

            def run(self, x, tuples, stream=None):
                out = nx.run(x, tuples)
                self.last_batches = [[0] * nx.stats["batches"]]
                return out
        ex = _NAdapter()
    elif greedy:   # Alg. 1: native scheduler decisions, instances on their own CUDA streams
        from paper_2510_09018_b200.executor import GreedyExecutor
        gx = GreedyExecutor(net, n_max=n_max, B_max=args.bmax, Q_th=args.q_th, N_new=args.n_new)

        class _Adapter:
            last_batches = [[]]
            pack_s = []

            def run(self, x, tuples, stream=None):
                gx.stats["batch_sizes"] = []
                out = gx.run(x, tuples)
                self.last_batches = [gx.stats["batch_sizes"]]
                return out
        ex = _Adapter()
    else:
        if args.lanes is None:   # the Python sequencer is host-bound on a fresh stream: extra lanes cost host time
            args.lanes = 1 if (args.stream_impl == "python" and not args.repeat_stream) else 8
        if args.stream_impl == "native":   # pack + enqueue in libslim (slim_stream_run)
            ex = NativeStreamExecutor(net, n_max=n_max, B_max=args.bmax, device=dev, lanes=args.lanes)
        else:
            ex = StreamExecutor(net, n_max=n_max, B_max=args.bmax, device=dev, lanes=args.lanes)
            ex.cache_plans = args.repeat_stream
        # one lane per width: partition the SMs by width as in cfg2 -- unless the policy routes a
        # single width (the "slim" policy keeps every SM for its one lane)
        if args.lanes > 1 and args.policy != "slim":
            cw = tuple(net.cfg.widths[i] for i in range(net.cfg.n_widths))
            for r, sh in sm_shares(cw, args.sm_share).items():
                slim.slim_set_sm_share(net.ctx, r, sh)
    sampler = NvmlSampler(local)
    telem = TelemetryExchange(device=_coll_dev(dev)) if world > 1 else None
    tsrc = TelemetrySource(sampler, rank)
    stream = torch.cuda.current_stream(dev)
    LAG = 2

    def routed(k):
        """This rank's requests of step k: (tuples [m, 4], m) -- identical decisions on every rank."""
        kk = 0 if args.repeat_stream else k
        if args.policy == "ppo_frozen":
            if telem is not None and telem.ticks() > LAG - 1:
                rec = telem.records(telem.ticks() - LAG)
            else:
                rec = np.zeros((world, 8), np.float32)
            devs, tups, _ = router.route_frozen(n_total, world, rec, t=kk, c_done=float(k * n_total))
        else:
            devs, tups, _ = router.route(n_total, world, args.policy, seed=2510_09018 + kk)
        mine = router.shard(devs, rank)
        return np.asarray(router.TABLE_TUPLES, np.float32)[tups[mine]], len(mine)

    done = [0]

    def one_step(k):
        tuples, m = routed(k)
        ex.run(x[:m], tuples, stream)
        done[0] += m
        if telem:
            telem.tick(tsrc.record(queue_len=float(n_total - m), completed=float(done[0])))
        return m

    sampler.start()
    for k in range(args.warmup):
        one_step(k)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = slim.slim_launch_count(net.ctx)
    e0 = sampler.energy_mj()
    n_pack0 = len(getattr(ex, "pack_s", []))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    mine_total = 0
    batches = []
    n_batches = 0
    host_s = []
    for k in range(args.steps):
        mine_total += one_step(args.warmup + k)
        if isinstance(ex, NativeStreamExecutor):
            n_batches += ex.last_n_batches
            host_s.append(ex.host_s[-1])
        else:
            batches += [bb for seg in ex.last_batches for bb in seg]
            n_batches += sum(len(seg) for seg in ex.last_batches)
    b.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = a.elapsed_time(b)
    t = torch.tensor([ms], dtype=torch.float64, device=_coll_dev(dev))
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    value = n_total * args.steps / (float(t.item()) / 1e3)
    # energy: the same steps continued for >= --energy-seconds (NVML counter delta / this rank's images)
    e0 = sampler.energy_mj()
    t0 = time.perf_counter()
    n_e = 0
    k = args.warmup + args.steps
    while args.energy_seconds > 0:
        n_e += one_step(k)
        k += 1
        if k % 8 == 0:
            torch.cuda.synchronize()
            stop = time.perf_counter() - t0 >= args.energy_seconds
            if world > 1:   # every step ticks a collective: all ranks must leave the loop at the same step
                f = torch.tensor([1.0 if stop else 0.0], device=_coll_dev(dev))
                dist.all_reduce(f, op=dist.ReduceOp.MAX)
                stop = float(f.item()) > 0
            if stop:
                break
    torch.cuda.synchronize()
    sampler.stop()
    e1 = sampler.energy_mj()
    clocks, energy = _clock_energy_json(sampler, e0, e1, max(n_e, 1)) if n_e else (sampler.summary(), None)
    pack = getattr(ex, "pack_s", [])[n_pack0:]
    n_desc = n_batches
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": float(t.item()) / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"{'CFG5' if world > 1 else 'CFG4'}: mixed-width request stream "
                                   f"(width tuples of Tables I-II), greedy (segment, w_req, w_prev) batching, "
                                   f"B_max={args.bmax}, routing={args.policy}, executor={args.executor}"
                                   + (f", lanes={args.lanes}, sequencer={args.stream_impl}"
                                      if not (greedy or native) else "")
                                   + (f" (Alg. 1: Q_th={args.q_th}, N_new={args.n_new})" if greedy or native else ""),
                       "requests_per_rank": args.requests, "parallelism": f"dp{world} routed",
                       "stream": "replayed (step 0's routing every step)" if args.repeat_stream else
                                 "fresh routing + packing every step (inside the timed region)",
                       "graphs": graphs},
            "batches_per_step_rank0": n_desc / args.steps,
            "mean_batch_rank0": (float(mine_total * 4 / max(1, n_desc)) if n_desc else None),
            "packer_host_us": ({"per_step": 1e6 * float(np.mean(pack)), "per_batch": 1e6 * float(np.sum(pack)) /
                                max(1, n_desc), "note": "slim_pack on all four segments + marshalling, host"}
                               if pack else None),
            **({"sequencer_host_us_per_step": 1e6 * float(np.mean(host_s))} if host_s else {}),
            **({"alg1_host_s_per_step": {k: gx.stats[k] / (args.steps + args.warmup)
                                         for k in ("t_next", "t_launch", "t_wait")},
                "alg1_instances": len(gx.sched.instances())} if greedy else {}),
            **({"nccl": nccl, "telemetry_allgather_us_mean": 1e3 * float(np.mean(telem.gather_ms))
                if telem.gather_ms else None} if telem else {}),
            "gpu_launches": slim.slim_launch_count(net.ctx) - l0, "energy_j_per_image": energy, "clocks": clocks,
        }))
    net.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_poisson(args):
    """CFG4 latency variant (SPEC Poisson arrivals): an open-loop Poisson request
    stream at --rate requests/s through the native Alg. 1 executor.  Reports completed
    images/s and per-request latency percentiles (arrival -> segment-3 batch complete)."""
    import numpy as np
    import torch

    import synth
    import paper_2510_09018_b200 as slim
    from paper_2510_09018_b200 import build as slim_build
    from paper_2510_09018_b200 import router
    from paper_2510_09018_b200.telemetry import NvmlSampler

    world, rank, local = _dist()
    if rank != 0:
        return 0
    torch.cuda.set_device(local)
    slim_build.build()
    net = slim.SlimNet(synth.make_weights(), synth.make_bn(), device=local, max_batch=args.bmax, norm=args.norm)
    n = args.requests
    g = np.random.Generator(np.random.PCG64([2510_09018, 5]))      # request-stream substream (+5)
    tuples = np.asarray(router.TABLE_TUPLES, np.float32)[g.integers(0, len(router.TABLE_TUPLES), n)]
    arrivals = np.cumsum(g.exponential(1.0 / args.rate, n))
    x = torch.from_numpy(synth.make_images(n, offset=400)).to(torch.bfloat16).cuda()
    slim.slim_set_graph_mode(net.ctx, args.alg1_graphs)
    ex = slim.NativeExecutor(net, n_max=n, B_max=args.bmax, Q_th=args.q_th, N_new=args.n_new,
                             M_max_bytes=args.m_max_gb * 1e9)
    for _ in range(args.warmup):
        ex.run(x, tuples, arrivals=arrivals)
    sampler = NvmlSampler(local)
    e0 = sampler.energy_mj()
    sampler.start()
    lat, spans, batches = [], [], 0
    for _ in range(args.steps):
        ex.run(x, tuples, arrivals=arrivals)
        lat.append(ex.latency.copy())
        spans.append(float(ex.done.max()))
        batches += ex.stats["batches"]
    sampler.stop()
    e1 = sampler.energy_mj()
    lat = np.concatenate(lat) * 1e3
    clocks, energy = _clock_energy_json(sampler, e0, e1, n * args.steps)
    print(json.dumps({
        "metric": METRIC, "value": n * args.steps / sum(spans), "unit": "images/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sum(spans) / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": f"CFG4 latency variant: open-loop Poisson arrivals at {args.rate:g} requests/s, width "
                               f"tuples uniform over Tables I-II, native Alg. 1 executor, B_max={args.bmax}",
                   "requests_per_step": n, "graphs": args.alg1_graphs, "M_max_GB": args.m_max_gb},
        "offered_rate": args.rate,
        "latency_ms": {"p50": float(np.percentile(lat, 50)), "p95": float(np.percentile(lat, 95)),
                       "p99": float(np.percentile(lat, 99)), "mean": float(lat.mean())},
        "mean_batch": 4.0 * n * args.steps / max(batches, 1),
        "gpu_launches": None, "energy_j_per_image": energy, "clocks": clocks,
    }))
    ex.close()
    net.close()
    return 0


def run_handoff(args):
    """NEXT-2: the mixed-width stream with per-SEGMENT routing (handoff.plan_segments): every
    rank runs the segments routed to it and hands activations to the next segment's rank with
    one all_to_all_single per segment boundary (NCCL over NVLink).  N=1: no exchange."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    import paper_2510_09018_b200 as slim
    from paper_2510_09018_b200 import build as slim_build
    from paper_2510_09018_b200 import handoff, router
    from paper_2510_09018_b200.telemetry import NvmlSampler

    world, rank, local = _dist()
    local = local % torch.cuda.device_count()   # (gloo functional check: several ranks on one GPU)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    slim_build.build()
    net = slim.SlimNet(synth.make_weights(), synth.make_bn(), device=local, max_batch=args.bmax, norm=args.norm)
    slim.slim_set_graph_mode(net.ctx, True)
    n = args.requests * world                      # weak scaling: requests per rank fixed
    g = np.random.Generator(np.random.PCG64([2510_09018, 5]))
    tuples = np.asarray(router.TABLE_TUPLES, np.float32)[g.integers(0, len(router.TABLE_TUPLES), n)]
    plan = handoff.plan_segments(n, world, args.seg_policy)
    x = torch.from_numpy(synth.make_images(n, offset=300)).to(torch.bfloat16).to(dev)
    if args.lanes is None:
        args.lanes = 8
    ex = handoff.HandoffExecutor(net, n, rank, world, B_max=args.bmax, lanes=args.lanes)
    if args.lanes > 1 and len(np.unique(tuples)) > 1:
        for r, sh in sm_shares(tuple(net.cfg.widths[i] for i in range(net.cfg.n_widths)), args.sm_share).items():
            slim.slim_set_sm_share(net.ctx, r, sh)
    for _ in range(args.warmup):
        ex.run(x, tuples, plan)
    torch.cuda.synchronize()
    sampler = NvmlSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = slim.slim_launch_count(net.ctx)
    e0 = sampler.energy_mj()
    sampler.start()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.steps):
        ex.run(x, tuples, plan)
    b.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler.stop()
    e1 = sampler.energy_mj()
    t = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device=_coll_dev(dev))
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    value = n * args.steps / (float(t.item()) / 1e3)
    clocks, energy = _clock_energy_json(sampler, e0, e1, args.requests * args.steps)
    moved = int((plan[:, 1:] != plan[:, :-1]).sum())
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": float(t.item()) / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"NEXT-2: mixed-width request stream routed per segment ({args.seg_policy}), "
                                   f"activation hand-off by all_to_all_single between segments, B_max={args.bmax}",
                       "requests_per_rank": args.requests, "parallelism": f"dp{world} segment-routed"},
            "handoffs_per_step": moved, "handoff_bytes_per_step": int(sum(
                ex.row_elems[s + 1] * ex.eb * int((plan[:, s] != plan[:, s + 1]).sum()) for s in range(3))),
            "gpu_launches": slim.slim_launch_count(net.ctx) - l0, "energy_j_per_image": energy, "clocks": clocks,
        }))
    net.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_points(args):
    """cfg1: seg 0 at r=0.25, B=8 (BASELINE configs[0]); sweep: CFG3, B in 1..4096 x widths.
    One JSON line per point (graph replay, L2 flushed before each timed replay batch)."""
    import torch

    import synth
    import paper_2510_09018_b200 as slim
    from paper_2510_09018_b200 import build as slim_build

    world, rank, local = _dist()
    if rank != 0:
        return 0
    torch.cuda.set_device(local)
    slim_build.build()
    peaks = _peaks()
    points = [(8, 0.25, "seg0")] if args.workload == "cfg1" else \
        [(B, r, "chain") for B in (1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096) for r in WIDTHS]
    bmax = max(p[0] for p in points)
    net = slim.SlimNet(synth.make_weights(), synth.make_bn(), device=local, max_batch=bmax, norm=args.norm)
    slim.slim_set_graph_mode(net.ctx, True)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    xall = torch.from_numpy(synth.make_images(bmax, offset=300)).to(torch.bfloat16).cuda()
    st = torch.cuda.current_stream()
    for B, r, kind in points:
        x = xall[:B]
        if kind == "seg0":
            out = torch.empty(B, 32, 32, slim.slim_channels(r, 64), dtype=torch.bfloat16, device="cuda")
            wsb = slim.slim_forward_workspace_bytes(net.ctx, 0, r, r, B)
            ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
            fn = lambda: slim.slim_forward_ws(net.ctx, 0, r, r, B, x, out, ws, wsb, st)
        else:
            out = torch.empty(B, 100, dtype=torch.float32, device="cuda")
            wsb = slim.slim_chain_workspace_bytes(net.ctx, (r,) * 4, B)
            ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
            fn = lambda: slim.slim_forward_chain(net.ctx, (r,) * 4, B, x, out, ws, wsb, st)
        for _ in range(max(3, args.warmup)):
            fn()
        reps = max(1, min(args.steps, 20000 // max(1, B)))
        # per-launch records for the roofline of this point (profiled pass, no graph)
        slim.slim_profile_begin(net.ctx, 64)
        fn()
        recs = slim.slim_profile_end(net.ctx)
        flops = sum(x_["flops"] for x_ in recs)
        roof_s = sum(max(x_["flops"] / (peaks["bf16"] * 1e12), x_["bytes"] / (peaks["hbm"] * 1e9)) for x_ in recs)
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            fn()
        b.record(st)
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / reps * 1e3
        floor = {}
        if kind == "seg0":   # CFG1: the launch floor -- a CUDA graph of as many empty-ish kernels
            t1 = torch.zeros(1, device="cuda")
            g = torch.cuda.CUDAGraph()
            cs = torch.cuda.Stream()
            with torch.cuda.stream(cs):
                t1.add_(1)
                torch.cuda.synchronize()
                with torch.cuda.graph(g, stream=cs):
                    for _ in range(len(recs)):
                        t1.add_(1)
            for _ in range(3):
                g.replay()
            torch.cuda.synchronize()
            a.record()
            for _ in range(reps):
                g.replay()
            b.record()
            torch.cuda.synchronize()
            fl = a.elapsed_time(b) / reps * 1e3
            floor = {"launch_floor_us": fl, "ratio_to_launch_floor": us / fl,
                     "launch_floor": f"CUDA graph of {len(recs)} one-element torch kernels, same replay count"}
        print(json.dumps({
            "metric": METRIC, "value": B / us * 1e6, "unit": "images/s", "n_gpus": 1, "steps": reps,
            "warmup": max(3, args.warmup), "ms_per_step": us / 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": ("CFG1: segment 0 (first residual stage) r=0.25 B=8" if kind == "seg0"
                                    else "CFG3: full chain batch sweep"), "batch": B, "width": r,
                       "l2": "flushed once before the timed replays (steady-state L2 reuse across replays)"},
            "us_per_call": us, "tflops": flops / (us * 1e-6) / 1e12,
            "per_layer_roofline_frac": roof_s / (us * 1e-6), "gpu_launches_per_call": len(recs), **floor,
        }), flush=True)
    net.close()
    return 0


def _ncu_traffic():
    """dram bytes per conv launch from the committed ncu --set full summary, if present."""
    p = os.path.join(ROOT, "profiles", "ncu_conv_summary.json")
    if not os.path.exists(p):
        return None
    try:
        return json.load(open(p)).get("dram_bytes_per_launch")
    except Exception:
        return None


def _ncu_tensor_pipe():
    """Tensor-pipe activity of the conv kernels from the committed ncu --set full summaries (the
    metric's "tensor-pipe % of peak"): mean over the captured conv launches, % of elapsed and of
    active cycles (sm__pipe_tensor_cycles_active / sm__pipe_tc_cycles_active)."""
    out = {}
    for key, f in (("b128_all_widths", "r02_ncu_chain_b128.json"), ("b1024_r1", "r02_ncu_b1024_r1.json")):
        p = os.path.join(ROOT, "profiles", f)
        try:
            L = [r for r in json.load(open(p))["launches"] if "conv" in r["kernel"]]
            out[key] = {"pct_of_peak_elapsed": sum(r.get("tensor_pct", 0.0) for r in L) / len(L),
                        "pct_of_peak_active": sum(r.get("tc_pipe_pct_active", 0.0) for r in L) / len(L),
                        "launches": len(L), "source": f"profiles/{f}"}
        except Exception:
            pass
    return out or None


def build_parser():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--dist-backend", choices=("nccl", "gloo"), default="nccl",
                    help="N > 1: nccl (one rank per GPU); gloo = functional check of the multi-rank path with "
                         "several ranks sharing a GPU (not a scaling measurement)")
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--sequential", action="store_true", help="run the 4 width instances one after another")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--cpu-seconds", type=float, default=30.0, help="cpu_baseline: time budget of the oracle protocol")
    ap.add_argument("--ref-batch", type=int, default=8, help="--impl reference: images per width per step")
    ap.add_argument("--profile-steps", type=int, default=50)
    ap.add_argument("--e2e-steps", type=int, default=200)
    ap.add_argument("--width-events", type=int, default=1,
                    help="cfg2: record CUDA events around each width's chain inside the timed step (per-width "
                         "time in the concurrent step); 0 = off")
    ap.add_argument("--energy-seconds", type=float, default=2.0, help="cfg2: length of the NVML energy loop (>= 1 s)")
    ap.add_argument("--json-out", default=None)
    ap.add_argument("--workload", choices=("cfg2", "cfg1", "sweep", "stream", "handoff", "poisson", "env"),
                    default="cfg2",
                    help="cfg2 (default, BASELINE configs[1]); cfg1 = seg0 r=0.25 B=8; sweep = CFG3 batch sweep "
                         "(one JSON line per point); stream = CFG4/CFG5 mixed-width routed request stream")
    ap.add_argument("--requests", type=int, default=1024, help="stream: requests per rank per step")
    ap.add_argument("--bmax", type=int, default=256, help="stream: B_max of the key batching")
    ap.add_argument("--policy", default="random",
                    help="stream: routing policy (random | slim | table_rr | ppo_frozen)")
    ap.add_argument("--stream-graphs", choices=("auto", "on", "off"), default="auto",
                    help="stream: CUDA-graph replay per batch shape (auto: only with --repeat-stream)")
    ap.add_argument("--repeat-stream", action="store_true",
                    help="stream: replay step 0's routing every step (packer plan cached) instead of a fresh stream")
    ap.add_argument("--launch-order", choices=("asc", "desc"), default="asc",
                    help="cfg2: order in which the width instances are enqueued each step")
    ap.add_argument("--stream-priority", choices=("none", "wide", "narrow"), default="none",
                    help="cfg2: CUDA stream priorities of the width instances")
    ap.add_argument("--sm-share", default="auto",
                    help="cfg2: SM shares of the concurrent width instances (auto | none | comma list per width)")
    ap.add_argument("--dtype", choices=("bf16", "fp32"), default="bf16",
                    help="cfg2: bf16 storage + fp32 accumulate (tcgen05, default) or the FP32/TF32-off mode (SIMT FFMA)")
    ap.add_argument("--widths", type=float, nargs="+", default=list(WIDTHS),
                    help="cfg2: width set (default the paper's {.25,.5,.75,1}; others = universal widths, NEXT-4)")
    ap.add_argument("--seg-policy", default="random", help="handoff: per-segment routing (random | pipeline | sticky)")
    ap.add_argument("--executor", choices=("stream", "greedy", "native"), default="stream",
                    help="stream: whole-stream packing per segment (graph replay); greedy: Alg. 1 executor "
                         "(native scheduler, per-instance streams)")
    ap.add_argument("--rate", type=float, default=300_000.0, help="poisson: offered load, requests/s")
    ap.add_argument("--m-max-gb", type=float, default=8.0,
                    help="poisson: Alg. 1 VRAM cap M_max (GB) -- bounds the instances the executor scales up to")
    ap.add_argument("--lanes", type=int, default=None,
                    help="stream/handoff: concurrent lanes (streams) per segment: one per width, times lanes/widths "
                         "rotating over a width's batches (default 8; 1 for the Python sequencer on a fresh stream)")
    ap.add_argument("--stream-impl", choices=("native", "python"), default="native",
                    help="stream executor: native = slim_stream_run (pack + enqueue in libslim); python = stream.py")
    ap.add_argument("--alg1-graphs", action="store_true", help="greedy/native: CUDA-graph replay per batch shape")
    ap.add_argument("--alg1-shares", action="store_true", help="greedy/native: per-width SM shares (--sm-share)")
    ap.add_argument("--q-th", type=int, default=512, help="greedy: Alg. 1 scale trigger Q_th")
    ap.add_argument("--n-new", type=int, default=2, help="greedy: Alg. 1 scale cap N_new")
    ap.add_argument("--norm", choices=("bn", "gn"), default="bn",
                    help="bn = switchable BatchNorm (north_star, default); gn = GroupNorm variant (P:148, NEXT-1)")
    return ap


def launcher_cmd(argv, n: int, port: int):
    """The torchrun command bench.py re-executes itself under for --gpus N > 1 (one process per GPU,
    rendezvous on 127.0.0.1), as the driver's own launch does."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_env(args):
    """Diagnostic workload: each rank reports the launcher environment (and, with world > 1, a gloo
    all-gather of the ranks proves the group spans them).  No GPU needed."""
    world, rank, local = _dist()
    rec = {"rank": rank, "local_rank": local, "world_size": world, "gpus_arg": args.gpus,
           "master_addr": os.environ.get("MASTER_ADDR"), "pid": os.getpid()}
    if world > 1:
        import torch
        import torch.distributed as dist
        dist.init_process_group("gloo")
        t = torch.tensor([rank], dtype=torch.int64)
        got = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(got, t)
        rec["gathered_ranks"] = [int(x) for x in got]
        dist.destroy_process_group()
    os.write(1, ("ENV " + json.dumps(rec) + "\n").encode())   # one write: ranks share the pipe
    return 0


def main(argv=None):
    ap = build_parser()
    raw = list(sys.argv[1:] if argv is None else argv)
    args = ap.parse_args(raw)
    _BACKEND["name"] = args.dist_backend
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `bench.py --gpus N` run directly: re-execute under torchrun with N ranks (the driver launches
        # N>1 through torchrun itself, which sets WORLD_SIZE and lands in the branch below)
        import subprocess
        return subprocess.call(launcher_cmd(raw, args.gpus, _free_port()))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl != "reference" and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (one rank per GPU)")
    if args.workload == "env":
        return run_env(args)
    assert args.warmup >= 0 and args.steps >= 1
    if args.impl == "reference":
        return run_reference(args)
    if args.workload == "stream":
        return run_stream(args)
    if args.workload == "handoff":
        return run_handoff(args)
    if args.workload == "poisson":
        return run_poisson(args)
    if args.workload in ("cfg1", "sweep"):
        return run_points(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
