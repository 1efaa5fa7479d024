"""Multi-GPU decomposition checked on CPU with torch.distributed/gloo,
world sizes 2 and 3: each rank back-projects its contiguous block of a subset's views (the same
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


def _slab_worker(rank, ws, port, out):
    """One OS-LALM inner step with the slab decomposition of the SQS update (ct_abi.cu
    subset_gradient / enqueue_iteration, slab path): partial back-projections summed and
    scattered by rows, slab g-update and xi partial, xi summed, slab update from the full
    x, rows gathered.  Compared with the same step computed whole on one process."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import oracle as O
    from paper_1402_4381_b200 import host
    from tests import geomutil as GU
    g = GU.small_geoms()["fan_c2"]
    M, m, beta, delta, rho = 3, 1, 2.0 ** 10, 2e-4, 0.4
    first, stride, count = host.subset_views(g["na"], M, m)
    rng = np.random.default_rng(1)
    shape = O.img_shape(g)
    x = rng.random(shape) * 0.02
    r = rng.standard_normal(O.sino_shape(g, count))
    G, gs, dl = rng.standard_normal(shape), rng.standard_normal(shape), rng.random(shape) + 0.5
    mask = np.ones(shape, np.uint8)

    def step(rows):
        """(x+ on rows, g+ on rows, xi over rows) given full x and the summed G+."""
        gr, cu = O.reg_grad(g, beta, delta, 8, mask, x)
        s_dir = rho * G + (1 - rho) * gs
        xn = np.maximum(0.0, x - (s_dir + gr) / (rho * dl + cu))
        return xn[..., rows, :], Gp

    k0, n = host.rank_view_block(count, rank, ws)
    part = O.back(g, r[k0:k0 + n], first + k0 * stride, stride, n)
    t = torch.from_numpy(part.copy())
    dist.all_reduce(t)                      # reduce-scatter = all-reduce + own rows
    iy0, iy1, R = host.rank_slab(shape[-2], rank, ws)
    Gp = t.numpy()
    rows = slice(iy0, iy1)
    xi_part = float(((gs - Gp) * (Gp - G))[..., rows, :].sum())
    xi = torch.tensor([xi_part], dtype=torch.float64)
    dist.all_reduce(xi)
    xrows, _ = step(rows)
    pad = np.zeros(shape[:-2] + (R, shape[-1]))
    pad[..., :iy1 - iy0, :] = xrows
    bufs = [torch.zeros_like(torch.from_numpy(pad)) for _ in range(ws)]
    dist.all_gather(bufs, torch.from_numpy(pad))
    xg = np.concatenate([b.numpy() for b in bufs], axis=-2)[..., :shape[-2], :]
    if rank == 0:
        Gf = O.back(g, r, first, stride, count)
        xi_f = float(((gs - Gf) * (Gf - G)).sum())
        gr, cu = O.reg_grad(g, beta, delta, 8, mask, x)
        xf = np.maximum(0.0, x - (rho * G + (1 - rho) * gs + gr) / (rho * dl + cu))
        out.put((float(np.abs(xg - xf).max()), abs(xi.item() - xi_f) / abs(xi_f)))
    dist.destroy_process_group()


def _zslab_worker(rank, ws, port, out):
    """z-slab decomposition (NEXT-3) with the oracle as the projector on each rank: partial
    sinograms of the slabs all-reduced = the full forward projection; the back-projection onto
    the slab = the full back-projection's slices; the regulariser on the slab with the
    neighbours' boundary slices (halo) = the full one's slices (what the 26-neighbour update
    of ct_abi.cu's z-slab path computes)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import oracle as O
    from paper_1402_4381_b200 import host
    from paper_1402_4381_b200 import inputs as I
    from tests import geomutil as GU
    g = GU.small_geoms()["helical_c5"]
    rng = np.random.default_rng(2)
    x = rng.random(O.img_shape(g)) * 0.02          # oracle layout [iz][iy][ix]
    r = rng.standard_normal(O.sino_shape(g, g["na"]))
    z0, z1 = host.rank_zslab(g["nz"], rank, ws)
    gs = I.slab_geom(g, z0, z1)
    part = torch.from_numpy(O.fwd(gs, x[z0:z1]))
    dist.all_reduce(part)
    back_s = O.back(gs, r)
    # halo: the slab extended by the neighbours' boundary slices, result cropped
    e0, e1 = max(z0 - 1, 0), min(z1 + 1, g["nz"])
    ge = I.slab_geom(g, e0, e1)
    mask = np.ones((e1 - e0,) + O.img_shape(g)[1:], np.uint8)
    gr_e, cu_e = O.reg_grad(ge, 2.0 ** 10, 2e-4, 26, mask, x[e0:e1])
    gr_s = gr_e[z0 - e0:z0 - e0 + (z1 - z0)]
    if rank == 0:
        full = O.fwd(g, x)
        bf = O.back(g, r)
        grf, _ = O.reg_grad(g, 2.0 ** 10, 2e-4, 26, np.ones(O.img_shape(g), np.uint8), x)
        out.put((float(np.abs(part.numpy() - full).max() / np.abs(full).max()),
                 float(np.abs(back_s - bf[z0:z1]).max() / np.abs(bf).max()),
                 float(np.abs(gr_s - grf[z0:z1]).max() / np.abs(grf).max())))
    dist.destroy_process_group()


def _zslab_window_worker(rank, ws, port, out):
    """Windowed z-slab exchange (helical) with the oracle as the projector: each rank projects
    its slab for the views of its window (host.zslab_window), sends every other rank the views
    both windows hold, receives theirs (gloo send / recv) and sums in rank order — on its
    window this equals the full forward projection (what zwin_sum_resid_kernel forms before the
    residual)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import oracle as O
    from paper_1402_4381_b200 import host
    from paper_1402_4381_b200 import inputs as I
    from tests import geomutil as GU
    g = GU.geom("cone_helical", nx=12, nz=40, dx=0.9766, dz=0.625, ns=24, ds=1.0239, nt=6, dt=1.0964, na=144,
                turns=6.0, pitch=0.8)
    M = 4
    rng = np.random.default_rng(5)
    x = rng.random(O.img_shape(g)) * 0.02
    slabs = [host.rank_zslab(g["nz"], q, ws) for q in range(ws)]
    errs = []
    for m in range(M):
        count = O.nviews(g, m, M)
        wins = [host.zslab_window(g, M, m, *slabs[q]) for q in range(ws)]
        k0, k1 = wins[rank]
        z0, z1 = slabs[rank]
        part = torch.from_numpy(np.ascontiguousarray(O.fwd(I.slab_geom(g, z0, z1), x[z0:z1], m + k0 * M, M, k1 - k0)))
        recv, reqs = {}, []
        for q in range(ws):
            if q == rank:
                continue
            o0, o1 = max(k0, wins[q][0]), min(k1, wins[q][1])
            if o1 <= o0:
                continue
            reqs.append(dist.isend(part[o0 - k0:o1 - k0].contiguous(), q))
            recv[q] = (o0, torch.empty((o1 - o0,) + tuple(part.shape[1:]), dtype=part.dtype))
            reqs.append(dist.irecv(recv[q][1], q))
        for rq in reqs:
            rq.wait()
        tot = torch.zeros_like(part)
        for q in range(ws):
            if q == rank:
                tot += part
            elif q in recv:
                o0, buf = recv[q]
                tot[o0 - k0:o0 - k0 + buf.shape[0]] += buf
        full = O.fwd(g, x, m, M, count)[k0:k1]
        errs.append(float(np.abs(tot.numpy() - full).max() / np.abs(full).max()))
    out.put((rank, max(errs)))
    dist.destroy_process_group()


@pytest.mark.parametrize("ws", [2, 3])
def test_gloo_zslab_window_exchange(ws):
    import oracle
    oracle.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_zslab_window_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(ws)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert max(e for _, e in res) <= 1e-12, res


@pytest.mark.parametrize("ws", [2, 3])   # 3: uneven view blocks / slabs
def test_gloo_two_rank_zslab(ws):
    import oracle
    oracle.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_zslab_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert max(res) <= 1e-12, res


def test_zslab_partition():
    from paper_1402_4381_b200 import host
    from paper_1402_4381_b200 import inputs as I
    g = I.config("c5").geom
    for ws in (1, 2, 3, 8):
        sl = [host.rank_zslab(g["nz"], r, ws) for r in range(ws)]
        assert sl[0][0] == 0 and sl[-1][1] == g["nz"]
        assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))
        for z0, z1 in sl:   # slab voxel centres lie on the full grid
            gs = I.slab_geom(g, z0, z1)
            zc_full = (z0 - (g["nz"] - 1) / 2) * g["dz"] + g.get("offz", 0.0)
            zc_slab = (0 - (gs["nz"] - 1) / 2) * gs["dz"] + gs["offz"]
            assert abs(zc_full - zc_slab) <= 1e-9


def test_slab_partition_covers_rows():
    from paper_1402_4381_b200 import host
    for ny in (1, 20, 64, 512, 513):
        for ws in (1, 2, 3, 8):
            slabs = [host.rank_slab(ny, r, ws) for r in range(ws)]
            assert slabs[0][0] == 0 and slabs[-1][1] == ny
            for (a0, a1, R), (b0, b1, _) in zip(slabs, slabs[1:]):
                assert a1 == b0 and a1 - a0 <= R
            assert ws * slabs[0][2] >= ny


@pytest.mark.parametrize("ws", [2, 3])   # 3: uneven view blocks / slabs
def test_gloo_two_rank_slab_update(ws):
    import oracle
    oracle.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] <= 1e-12 and res[1] <= 1e-10


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


@pytest.mark.parametrize("ws", [2, 3])   # 3: uneven view blocks / slabs
def test_gloo_two_rank_back_projection_sum(ws):
    import oracle
    oracle.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] <= 1e-12 and res[1] <= 1e-12


def test_rank_band_contains_every_seen_slice():
    """Band-limited exchange (helical): every slice that any view of a rank's block of a subset
    sees (a non-zero oracle projection of that slice alone) lies inside host.rank_band, and the
    bands are much narrower than the volume on a long helix (the exchange saving)."""
    import numpy as np
    import oracle as O
    from paper_1402_4381_b200 import host
    from tests import geomutil as GU
    g = GU.geom("cone_helical", nx=12, nz=40, dx=0.9766, dz=0.625, ns=24, ds=1.0239, nt=6, dt=1.0964, na=144,
                turns=6.0, pitch=0.8)
    M, P = 4, 3
    widths = []
    for m in range(M):
        count = O.nviews(g, m, M)
        for r in range(P):
            k0, n = host.rank_view_block(count, r, P)
            b0, b1 = host.rank_band(g, M, m, r, P)
            widths.append(b1 - b0)
            for z in range(g["nz"]):
                x = np.zeros(O.img_shape(g))
                x[z] = 1.0
                p = O.fwd(g, x, m + k0 * M, M, n)
                if np.abs(p).max() > 0:
                    assert b0 <= z < b1, (m, r, z, b0, b1)
    assert max(widths) <= 0.75 * g["nz"]


def test_zslab_window_contains_every_reaching_view():
    """Windowed z-slab exchange (helical): every view of a subset whose oracle projection of a
    rank's slab (all ones) is non-zero lies inside host.zslab_window (the mirror of the
    library's zslab_window_of), and on a long helix the windows are shorter than a subset
    (on average; the middle slab's window spans most of a subset — the cone's z reach)."""
    import numpy as np
    import oracle as O
    from paper_1402_4381_b200 import host
    from tests import geomutil as GU
    g = GU.geom("cone_helical", nx=12, nz=40, dx=0.9766, dz=0.625, ns=24, ds=1.0239, nt=6, dt=1.0964, na=144,
                turns=6.0, pitch=0.8)
    M, P = 4, 3
    fracs = []
    for m in range(M):
        count = O.nviews(g, m, M)
        for r in range(P):
            z0, z1 = host.rank_zslab(g["nz"], r, P)
            k0, k1 = host.zslab_window(g, M, m, z0, z1)
            fracs.append((k1 - k0) / count)
            x = np.zeros(O.img_shape(g))
            x[z0:z1] = 1.0
            p = O.fwd(g, x, m, M, count).reshape(count, -1)
            hit = np.nonzero(np.abs(p).max(axis=1) > 0)[0]
            assert hit.size > 0
            assert k0 <= hit.min() and hit.max() < k1, (m, r, hit.min(), hit.max(), k0, k1)
    assert sum(fracs) / len(fracs) <= 0.7
