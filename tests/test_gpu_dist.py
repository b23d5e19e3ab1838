"""The sharded product path end to end on real kernels: two ranks
(gloo process group, both on cuda:0 — one GPU in this environment) each run
laGP_alc_batch on their contiguous shard of XX and one all-gather assembles the
outputs; the result must be bit-identical to the single unsharded call (S:351:
each location depends only on its own row), for an even and a ragged split."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

KEYS = ("idx", "mean", "s2", "var", "flags")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, M, outdir):
    import torch.distributed as dist

    import paper_1310_5182_b200 as lagp
    from lagp_data import make_config

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = torch.device("cuda", 0)
        cfg = make_config("C2", M=M, N=20000)
        X, Z, XX = (torch.from_numpy(cfg[k]).to(dev) for k in ("X", "Z", "XX"))
        r = lagp.alc_batch_dist(X, Z, XX, cfg["d"], cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"])
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), **{k: r[k].cpu().numpy() for k in KEYS})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("M", [64, 77])
def test_alc_batch_dist_two_ranks_bit_identical(tmp_path, M):
    import paper_1310_5182_b200 as lagp
    from lagp_data import make_config

    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, M, str(tmp_path))) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    dev = torch.device("cuda", 0)
    cfg = make_config("C2", M=M, N=20000)
    X, Z, XX = (torch.from_numpy(cfg[k]).to(dev) for k in ("X", "Z", "XX"))
    ref = lagp.alc_batch(X, Z, XX, cfg["d"], cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"])
    for r in range(2):
        got = np.load(tmp_path / f"rank{r}.npz")
        for k in KEYS:
            assert np.array_equal(got[k], ref[k].cpu().numpy()), (r, k)
