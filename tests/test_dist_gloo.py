"""Multi-GPU decomposition checked on CPU with torch.distributed/gloo,
world size 2: each rank back-projects its contiguous block of a subset's views (the same
partition the C library's rank_views uses, mirrored by host.rank_view_block), the partial
images are summed with all_reduce, and the result must equal the full subset back-projection.
The oracle supplies the projector on both ranks; the NCCL path itself needs GPUs."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import oracle as O
    from paper_1402_4381_b200 import host
    from tests import geomutil as GU
    g = GU.small_geoms()["helical_c5"]
    M, m = 4, 1
    first, stride, count = host.subset_views(g["na"], M, m)
    rng = np.random.default_rng(0)
    p = rng.random(O.sino_shape(g, count))
    k0, n = host.rank_view_block(count, rank, ws)
    part = O.back(g, p[k0:k0 + n], first + k0 * stride, stride, n)
    # the scalar xi is likewise a sum of per-rank partials
    xi = torch.tensor([float(part.sum())], dtype=torch.float64)
    t = torch.from_numpy(part.copy())
    dist.all_reduce(t)
    dist.all_reduce(xi)
    if rank == 0:
        full = O.back(g, p, first, stride, count)
        out.put((float(np.abs(t.numpy() - full).max() / np.abs(full).max()),
                 abs(xi.item() - full.sum()) / abs(full.sum())))
    dist.destroy_process_group()


def test_view_block_partition_covers_subset():
    from paper_1402_4381_b200 import host
    for count in (1, 7, 41, 287):
        for ws in (1, 2, 3, 8):
            blocks = [host.rank_view_block(count, r, ws) for r in range(ws)]
            assert blocks[0][0] == 0
            for (a, n), (b, _) in zip(blocks, blocks[1:]):
                assert a + n == b
            assert sum(n for _, n in blocks) == count
            assert max(n for _, n in blocks) - min(n for _, n in blocks) <= 1


def test_gloo_two_rank_back_projection_sum():
    import oracle
    oracle.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] <= 1e-12 and res[1] <= 1e-12
