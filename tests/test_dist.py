"""Multi-rank host logic of the sharded path on CPU with gloo,
world_size 2 (and 3): shard bounds cover XX exactly once in order, and the
all-gather reassembles per-rank outputs in input order, including ragged and
empty shards. The per-location compute is replaced by a deterministic function
of the global row index (no GPU here)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1310_5182_b200 import gather_shards, shard_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def fake_local(lo, hi, n):
    rows = torch.arange(lo, hi, dtype=torch.int64)
    return dict(
        idx=(rows[:, None] * 7 + torch.arange(n)[None, :]).to(torch.int32),
        mean=rows.to(torch.float64) * 0.5,
        s2=rows.to(torch.float64) + 0.25,
        var=rows.to(torch.float64) * 2.0,
        flags=(rows % 3).to(torch.int32),
    )


def _worker(rank, world, port, M, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi, _ = shard_bounds(M, rank, world)
        out = gather_shards(fake_local(lo, hi, n), M)
        ref = fake_local(0, M, n)
        ok = all(torch.equal(out[k], ref[k]) for k in ref)
        q.put((rank, ok, [int(out["idx"].shape[0])]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,M", [(2, 10), (2, 11), (3, 7), (2, 1), (3, 2)])
def test_gather_shards_gloo(world, M):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, M, 5, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res), res
    assert all(sz == [M] for _, _, sz in res)


@pytest.mark.parametrize("M,world", [(10, 1), (10, 3), (10000, 8), (7, 8), (0, 4)])
def test_shard_bounds_partition(M, world):
    seen = []
    for r in range(world):
        lo, hi, per = shard_bounds(M, r, world)
        assert 0 <= lo <= hi <= M and hi - lo <= per
        seen.extend(range(lo, hi))
    assert seen == list(range(M))
    assert np.all(np.diff(seen) == 1) if seen else True
