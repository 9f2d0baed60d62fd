"""Per-device telemetry: NVML sampling and the NCCL all-gather of the router's state.

PAPER.md:49 -- the executor "samples utilization and emits telemetry data
(utilization, VRAM, per-segment queue sizes, latency percentiles)"; Eq. 1
 -- the router state holds, per server i, (q_i, P_i, U_i).  Each rank
packs one float32[8] record (SI units, SURVEY §8(c) reading #15):

    [queue_len, power_W, util_frac, mean_latency_s, energy_J_since_tick,
     completed, vram_used_GB, rank]

and `TelemetryExchange.tick()` all-gathers the records of all ranks with one
`all_gather_into_tensor` (NCCL over NVLink on GPUs, gloo on CPU) on a side stream.
This is host-side control plumbing, not the compute path.
"""
from __future__ import annotations

import threading
import time

import numpy as np

RECORD_LEN = 8
FIELDS = ("queue_len", "power_W", "util_frac", "mean_latency_s", "energy_J", "completed", "vram_used_GB", "rank")

# NVML clock-event reason bits (nvml.h) -> names used in the bench JSON line
_REASONS = {0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x10: "sync_boost",
            0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
            0x100: "display_clock_setting"}


def reason_names(mask: int):
    return [n for b, n in _REASONS.items() if mask & b]


def pack_record(queue_len=0.0, power_w=0.0, util=0.0, mean_latency_s=0.0, energy_j=0.0, completed=0.0,
                vram_gb=0.0, rank=0.0) -> np.ndarray:
    return np.array([queue_len, power_w, util, mean_latency_s, energy_j, completed, vram_gb, rank], np.float32)


def util_variance(utils) -> float:
    """Var(U/100) of Eq. 7: population variance of utilisation fractions.
    SPEC example: [0, 1] -> 0.25."""
    u = np.asarray(utils, np.float64)
    return float(((u - u.mean()) ** 2).mean()) if u.size else 0.0


class NvmlSampler:
    """Background sampler of SM clock, power, utilisation and clock-event reasons."""

    def __init__(self, device_index: int = 0, period_s: float = 0.01):
        self.period = period_s
        self.samples = []
        self._stop = threading.Event()
        self._thr = None
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self._nv = None
            self.max_sm = None

    def energy_mj(self):
        if not self.ok:
            return None
        try:
            return self._nv.nvmlDeviceGetTotalEnergyConsumption(self._h)
        except Exception:
            return None

    def sample(self):
        nv, h = self._nv, self._h
        try:
            reasons = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            reasons = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        try:
            energy_mj = nv.nvmlDeviceGetTotalEnergyConsumption(h)
        except Exception:
            energy_mj = None
        return dict(t=time.time(), sm=nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                    power_w=nv.nvmlDeviceGetPowerUsage(h) / 1000.0,
                    util=nv.nvmlDeviceGetUtilizationRates(h).gpu / 100.0, reasons=int(reasons),
                    mem_gb=nv.nvmlDeviceGetMemoryInfo(h).used / 2 ** 30, energy_mj=energy_mj)

    def latest(self):
        """The most recent background sample (None before the first); no NVML call on the caller."""
        return self.samples[-1] if self.samples else None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.sample())
            except Exception:
                pass
            self._stop.wait(self.period)

    def start(self):
        if self.ok:
            self.samples = []
            self._stop.clear()
            self._thr = threading.Thread(target=self._run, daemon=True)
            self._thr.start()

    def stop(self):
        if self._thr is not None:
            self._stop.set()
            self._thr.join()
            self._thr = None
            try:
                self.samples.append(self.sample())
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_sm, "reasons": [], "samples": 0}
        sm = sorted(s["sm"] for s in self.samples)
        mask = 0
        for s in self.samples:
            mask |= s["reasons"]
        return {"sm_mhz": float(sm[len(sm) // 2]), "sm_max_mhz": self.max_sm, "reasons": reason_names(mask),
                "samples": len(self.samples), "power_w_max": max(s["power_w"] for s in self.samples)}


class TelemetrySource:
    """Fills this rank's float32[8] record (FIELDS) for a router tick from the background NVML
    sampler's latest sample -- power (W), utilisation (fraction), VRAM (GB), energy (J) since the
    previous tick -- plus what the executor knows: queue length, mean latency (s), completed requests.
    The tick itself makes no NVML call (the sampler thread does, every period_s)."""

    def __init__(self, sampler: "NvmlSampler", rank: int):
        self.sampler, self.rank = sampler, rank
        self._e_prev = None

    def record(self, queue_len: float = 0.0, mean_latency_s: float = 0.0, completed: float = 0.0) -> np.ndarray:
        s = self.sampler.latest() if self.sampler is not None else None
        if s is None:
            return pack_record(queue_len=queue_len, mean_latency_s=mean_latency_s, completed=completed, rank=self.rank)
        e = s.get("energy_mj")
        de = 0.0 if (e is None or self._e_prev is None) else (e - self._e_prev) / 1e3
        if e is not None:
            self._e_prev = e
        return pack_record(queue_len=queue_len, power_w=s["power_w"], util=s["util"],
                           mean_latency_s=mean_latency_s, energy_j=de, completed=completed,
                           vram_gb=s["mem_gb"], rank=self.rank)


class TelemetryExchange:
    """One all_gather_into_tensor of float32[8] per rank per router tick."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.device = device if device is not None else "cpu"
        self.send = torch.zeros(RECORD_LEN, dtype=torch.float32, device=self.device)
        self.recv = torch.zeros(self.world * RECORD_LEN, dtype=torch.float32, device=self.device)
        self.stream = torch.cuda.Stream(device=self.device) if str(self.device).startswith("cuda") else None
        # pinned staging ring: a pageable H2D copy would block the host until the side stream (which
        # waits for the step) reaches it, serialising the host's launches with the GPU every tick
        self._ring = [torch.zeros(RECORD_LEN, dtype=torch.float32).pin_memory() for _ in range(4)] \
            if self.stream is not None else None
        self._ev = [torch.cuda.Event() for _ in range(4)] if self.stream is not None else None
        # per-tick result ring: tick i gathers into recv_ring[i % 4] and copies it to a pinned host buffer;
        # records(i) waits for that copy only (a fixed lag, so every rank reads the same tick's state)
        if self.stream is not None:
            self._recv_ring = [torch.zeros(self.world * RECORD_LEN, dtype=torch.float32, device=self.device)
                               for _ in range(4)]
            self._host_ring = [torch.zeros(self.world * RECORD_LEN, dtype=torch.float32).pin_memory()
                               for _ in range(4)]
            self._hev = [torch.cuda.Event() for _ in range(4)]
        self._cpu_hist = {}
        self._k = 0
        # device time of each all-gather on the side stream (CFG5 "telemetry all-gather overhead")
        self._t = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(4)] \
            if self.stream is not None else None
        self.gather_ms = []

    def tick(self, record: np.ndarray, wait: bool = False):
        """Start the all-gather of this rank's record; returns a handle (or the gathered [world, 8] array)."""
        import torch
        rec = torch.from_numpy(np.asarray(record, np.float32))
        if self.stream is not None:
            i = self._k % len(self._ring)
            self._k += 1
            self._ev[i].synchronize()          # the copy that last read this staging buffer is done
            self._ring[i].copy_(rec)
            cur = torch.cuda.current_stream(self.device)
            self.stream.wait_stream(cur)
            if self._k > len(self._t):   # the timing events of slot i were recorded 4 ticks ago
                ta, tb = self._t[i]
                tb.synchronize()
                self.gather_ms.append(ta.elapsed_time(tb))
            self.recv = self._recv_ring[i]
            with torch.cuda.stream(self.stream):
                self.send.copy_(self._ring[i], non_blocking=True)
                self._ev[i].record(self.stream)
                self._t[i][0].record(self.stream)
                work = self.dist.all_gather_into_tensor(self.recv, self.send, group=self.group, async_op=True)
                work.wait()   # NCCL: the side stream (not the host) waits for the collective
                self._t[i][1].record(self.stream)
                self._host_ring[i].copy_(self.recv, non_blocking=True)
                self._hev[i].record(self.stream)
        else:
            self.send.copy_(rec)
            work = self.dist.all_gather_into_tensor(self.recv, self.send, group=self.group, async_op=True)
            work.wait()
            self._cpu_hist[self._k] = self.recv.clone()
            self._cpu_hist.pop(self._k - 8, None)
            self._k += 1
        if wait:
            work.wait()
            if self.stream is not None:
                self.stream.synchronize()
            return self.recv.view(self.world, RECORD_LEN).cpu().numpy()
        return work

    def ticks(self) -> int:
        """Number of ticks started so far (tick indices 0 .. ticks()-1)."""
        return self._k

    def records(self, tick: int) -> np.ndarray:
        """The [world, 8] records all-gathered at tick `tick` (one of the last 4; waits only for that
        tick's copy).  Reading a fixed number of ticks back keeps every rank on the same state."""
        if self.stream is not None:
            assert self._k - 4 <= tick < self._k, "tick outside the 4-entry ring"
            i = tick % 4
            self._hev[i].synchronize()
            return self._host_ring[i].view(self.world, RECORD_LEN).numpy().copy()
        return self._cpu_hist[tick].view(self.world, RECORD_LEN).numpy().copy()

    def gathered(self) -> np.ndarray:
        if self.stream is not None:
            self.stream.synchronize()
        return self.recv.view(self.world, RECORD_LEN).cpu().numpy()
