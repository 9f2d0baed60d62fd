"""Per-segment cross-device routing -- host side on CPU:
the replicated segment plan, the exchange lists, and the collective transport over a
world-size-2/3 gloo group: every row reaches the rank that runs the request's next
segment, with split sizes every rank derived on its own."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_09018_b200 import handoff


def test_plan_policies():
    for world in (1, 2, 3, 8):
        p = handoff.plan_segments(500, world, "pipeline")
        assert (p == np.array([(s * world) // 4 for s in range(4)])).all()
        r = handoff.plan_segments(500, world, "random", seed=3)
        assert r.min() >= 0 and r.max() < world and (r == handoff.plan_segments(500, world, "random", seed=3)).all()
        st = handoff.plan_segments(500, world, "sticky")
        assert (st == st[:, :1]).all()
    r = handoff.plan_segments(4000, 2, "random")
    assert 0.45 < (r[:, 1] != r[:, 0]).mean() < 0.55   # about half of the requests change device


def test_exchange_lists_partition():
    world, n = 3, 400
    dev = handoff.plan_segments(n, world, "random", seed=9)
    for s in range(3):
        moved = np.nonzero(dev[:, s] != dev[:, s + 1])[0]
        sends = [handoff.exchange_lists(dev, s, r, world)[0] for r in range(world)]
        recvs = [handoff.exchange_lists(dev, s, r, world)[1] for r in range(world)]
        allsent = np.sort(np.concatenate([x for r in sends for x in r]))
        np.testing.assert_array_equal(allsent, moved)
        for a in range(world):
            for b in range(world):
                np.testing.assert_array_equal(sends[a][b], recvs[b][a])   # what a sends b is what b expects from a


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, row = 300, 24
        dev = handoff.plan_segments(n, world, "random", seed=21)
        ok = True
        for s in range(3):
            send, recv = handoff.exchange_lists(dev, s, rank, world)
            ids = np.concatenate(send)
            # row bytes of request i at boundary s: (i * 7 + s + k) mod 251, k < row
            send_buf = torch.from_numpy(((ids[:, None] * 7 + s + np.arange(row)) % 251).astype(np.uint8).ravel())
            rb = [len(x) * row for x in recv]
            recv_buf = torch.empty(sum(rb), dtype=torch.uint8)
            handoff.CollectiveTransport().exchange(send_buf, [len(x) * row for x in send], recv_buf, rb)
            rid = np.concatenate(recv)
            exp = ((rid[:, None] * 7 + s + np.arange(row)) % 251).astype(np.uint8).ravel()
            ok &= bool(np.array_equal(recv_buf.numpy(), exp))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_collective_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(res.values()), res
