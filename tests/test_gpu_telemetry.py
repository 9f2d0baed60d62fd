"""GPU: the telemetry all-gather (P:90-92 router state) over a 1-rank NCCL group on
the side stream -- asynchronous ticks (pinned staging ring) deliver the latest record, and a tick
does not block the host on the GPU work it follows."""
import os
import socket
import time

import numpy as np
import pytest
import torch
import torch.distributed as dist

from paper_2510_09018_b200.telemetry import TelemetryExchange, pack_record

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_nccl_telemetry_ticks_are_async():
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        ex = TelemetryExchange(device="cuda:0")
        for k in range(10):
            ex.tick(pack_record(queue_len=k, power_w=100.0 + k, rank=0))
        g = ex.gathered()
        np.testing.assert_array_equal(g[0], pack_record(queue_len=9, power_w=109.0, rank=0))
        # a long GPU job in flight: the tick must return without waiting for it
        a = torch.randn(4096, 4096, device="cuda")
        torch.cuda.synchronize()
        for _ in range(30):
            a = a @ a * 1e-3
        t0 = time.perf_counter()
        ex.tick(pack_record(queue_len=42.0))
        dt = time.perf_counter() - t0
        torch.cuda.synchronize()
        assert ex.gathered()[0][0] == 42.0
        assert dt < 0.02, f"tick blocked the host for {dt * 1e3:.1f} ms"
        for _ in range(6):
            ex.tick(pack_record(queue_len=1.0))
        torch.cuda.synchronize()
        assert len(ex.gather_ms) >= 3 and all(t > 0 for t in ex.gather_ms)   # device time per all-gather
    finally:
        dist.destroy_process_group()
