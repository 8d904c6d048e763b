"""Multi-process host logic on CPU (gloo, world_size 2): view partition and
the data-parallel gradient all-reduce used by DataParallelTrainer and
bench.py. The CUDA kernels are not involved (no GPU here)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_13348_b200.training import allreduce_mean_, flatten, partition_views, unflatten


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # each rank's "gradients": rank-dependent values in mixed dtypes
        g64 = torch.full((5, 3), float(rank + 1), dtype=torch.float64)
        g32 = torch.arange(7, dtype=torch.float32) * (rank + 1)
        flat = flatten([g64, g32])
        allreduce_mean_(flat)
        a, b = unflatten(flat, [g64, g32])
        views = partition_views(256, rank, world)
        # total views over ranks, via an all-reduce of the counts
        cnt = torch.tensor([len(views)], dtype=torch.int64)
        dist.all_reduce(cnt)
        # max-over-ranks timing reduction as in bench.py
        t = torch.tensor([1.0 + rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        q.put((rank, a.tolist(), b.tolist(), views[:3], int(cnt), float(t)))
    finally:
        dist.destroy_process_group()


def test_allreduce_mean_and_partition_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    for rank, a, b, views, cnt, tmax in out:
        assert all(v == 1.5 for row in a for v in row)      # mean of 1 and 2
        assert b == [i * 1.5 for i in range(7)]
        assert views == [rank, rank + 2, rank + 4]
        assert cnt == 256
        assert tmax == 2.0


def test_partition_covers_every_view_once():
    for world in (1, 2, 4, 8):
        seen = sorted(v for r in range(world) for v in partition_views(256, r, world))
        assert seen == list(range(256))
    with pytest.raises(ValueError):
        partition_views(10, 3, 2)


def test_unflatten_roundtrip_and_size_check():
    ts = [torch.randn(3, 4, dtype=torch.float64), torch.randn(5)]
    back = unflatten(flatten(ts), ts)
    assert torch.allclose(back[0].double(), ts[0].float().double())
    assert torch.equal(back[1], ts[1])
    with pytest.raises(ValueError):
        unflatten(torch.zeros(3), ts)
