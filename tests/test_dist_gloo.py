"""Multi-process (world_size 2, gloo on CPU) coverage of the N>1 host path:
replicated deterministic routing, request sharding, and the telemetry all-gather."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_09018_b200 import router
from paper_2510_09018_b200.telemetry import RECORD_LEN, TelemetryExchange, pack_record, util_variance


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
        out = {}
        # 1. replicated routing: every rank derives the same assignment without communication
        for pol in router.POLICIES:
            dev, tup, grp = router.route(1000, world, pol, seed=5)
            h = torch.tensor([int(np.bitwise_xor.reduce(dev * 1000003 + tup * 31 + grp))], dtype=torch.int64)
            hs = [torch.zeros_like(h) for _ in range(world)]
            dist.all_gather(hs, h)
            out[f"same_{pol}"] = all(int(x) == int(hs[0]) for x in hs)
            mine = router.shard(dev, rank)
            cnt = torch.tensor([len(mine)], dtype=torch.int64)
            dist.all_reduce(cnt)
            out[f"count_{pol}"] = int(cnt)
        # 2. telemetry all-gather of float32[8] records
        ex = TelemetryExchange(device="cpu")
        g = ex.tick(pack_record(queue_len=rank + 1, power_w=100.0 * (rank + 1), util=0.5 * rank, rank=rank), wait=True)
        out["telemetry"] = g.tolist()
        # 3. frozen PPO routing on the gathered state (one tick late): identical on both ranks, and
        #    it reads the state (a different gathered record routes differently)
        def _hash(a):
            h = torch.tensor([int(np.bitwise_xor.reduce(a[0] * 1000003 + a[1] * 31 + a[2]))], dtype=torch.int64)
            hs = [torch.zeros_like(h) for _ in range(world)]
            dist.all_gather(hs, h)
            return [int(x) for x in hs]
        rt = router.route_frozen(2000, world, g, t=3)
        out["frozen_hashes"] = _hash(rt)
        busy = g.copy(); busy[0, 0] += 5000.0                    # rank 0's queue much longer
        out["frozen_differs"] = not np.array_equal(router.route_frozen(2000, world, busy, t=3)[0], rt[0])
        out["frozen_counts"] = np.bincount(rt[0], minlength=world).tolist()
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def gloo_results():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_routing_is_replicated(gloo_results):
    for r in (0, 1):
        for pol in router.POLICIES:
            assert gloo_results[r][f"same_{pol}"]


def test_shards_partition_the_stream(gloo_results):
    for pol in router.POLICIES:
        assert gloo_results[0][f"count_{pol}"] == 1000


def test_telemetry_allgather_layout(gloo_results):
    for r in (0, 1):
        g = np.asarray(gloo_results[r]["telemetry"])
        assert g.shape == (2, RECORD_LEN)
        assert list(g[:, 0]) == [1.0, 2.0] and list(g[:, 1]) == [100.0, 200.0]
        assert list(g[:, 7]) == [0.0, 1.0]


def test_frozen_policy_routing_replicated(gloo_results):
    """--policy ppo_frozen: both ranks derive the same assignment from the all-gathered telemetry."""
    for r in (0, 1):
        h = gloo_results[r]["frozen_hashes"]
        assert h[0] == h[1]
        assert gloo_results[r]["frozen_differs"]
        assert sum(gloo_results[r]["frozen_counts"]) == 2000
    assert gloo_results[0]["frozen_hashes"] == gloo_results[1]["frozen_hashes"]


def test_util_variance_spec_example():
    assert util_variance([0.0, 1.0]) == 0.25          # SPEC util_variance example
    assert util_variance([0.3, 0.3, 0.3]) == 0.0


def test_route_policies_shapes():
    dev, tup, grp = router.route(64, 4, "table_rr")
    assert set(dev.tolist()) == {0, 1, 2, 3}
    assert np.all(tup[:4] == 0) and np.all(tup[4:8] == 1)
    dev, tup, grp = router.route(10, 3, "slim")
    assert np.all(tup == 0) and np.all(np.asarray(router.TABLE_TUPLES[0]) == 0.25)
    with pytest.raises(ValueError):
        router.route(4, 2, "ppo")
