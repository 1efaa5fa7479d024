"""The multi-rank C++ path with P > 1 ranks, run as VIRTUAL ranks on one GPU (SURVEY §4
item 3(i); `ct_comm_init_virtual`, csrc/ct_comm.cuh) and checked against the fp64 oracle.

Every virtual rank has its own geometry handle, OS-LALM state, buffers and stream and is
driven by its own host thread; each exchange step (reduce-scatter of the partial G+ into
padded row slabs, xi all-reduce, all-gather of the updated slabs, D_L all-reduce; for the
z-slab decomposition the subset-sinogram all-reduce and the one-slice halos) is a host
rendezvous followed by device copies and fixed-order sum kernels ordered by CUDA events, so
no kernel waits on another.  This runs the real `ct_abi.cu` multi-rank code (slab padding,
off0, gupd_slab_kernel, xi_rule_kernel, z-slab halos, view blocks with empty ranks) that a
one-rank NCCL communicator cannot reach.

Bar: the oracle's OS-LALM image within 0.5 HU RMS over S with identical restart decisions
(BASELINE.json north_star), plus the support mask bit-exact.
"""
import math
import threading

import numpy as np
import pytest
import torch

from paper_1402_4381_b200 import inputs as I
from tests import geomutil as GU

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ct():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1402_4381_b200 import build, ctlib
    build.build()
    ctlib.load()
    return ctlib


@pytest.fixture(scope="module")
def O():
    import oracle
    oracle.build()
    return oracle


def run_virtual(ct, geoms, y, w, masks, M, n_iter, beta, delta, nbr, zslab=False, bb=False, exchange="auto"):
    """Drive len(geoms) virtual ranks (one thread each): D_L, then n_iter OS-LALM iterations.
    Returns per-rank (x, support, log)."""
    P = len(geoms)
    geos = [ct.Geometry(g) for g in geoms]
    ct.Geometry.comm_init_virtual(geos, zslab=zslab)
    for geo in geos:
        ct.ct_comm_set_exchange(geo.h, exchange)
    streams = [torch.cuda.Stream() for _ in range(P)]
    yc, wc = y.cuda(), w.cuda()
    S = [m.clone().cuda() for m in masks]
    dl = [torch.empty(geo.img_shape, dtype=torch.float32, device="cuda") for geo in geos]
    scr = [torch.empty(ct.ct_sqs_denom_scratch_bytes(geo.h), dtype=torch.uint8, device="cuda") for geo in geos]
    sols = [ct.OSLALM(geo, M, beta=beta, delta=delta, nbr=nbr, bb=bb) for geo in geos]
    xs = [torch.zeros(geo.img_shape, device="cuda") for geo in geos]
    torch.cuda.synchronize()
    logs, errs = [None] * P, []

    def worker(r):
        try:
            ct.ct_sqs_denom(geos[r].h, wc, S[r], dl[r], scr[r], stream=streams[r])
            sols[r].set_data(yc, wc, dl[r], S[r])
            logs[r] = np.array(sols[r].run(xs[r], n_iter, log=True, stream=streams[r]))
        except Exception as e:  # reported below
            errs.append((r, repr(e)))

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in th), "virtual ranks did not finish (rendezvous stuck)"
    assert not errs, errs
    torch.cuda.synchronize()
    return [(xs[r].cpu().numpy(), S[r].cpu().numpy(), logs[r]) for r in range(P)]


def oracle_run(O, g, y, w, m0, M, n_iter, beta, delta, nbr, bb=False):
    dlo, So = O.sqs_denom(g, I.to_oracle_sino(w), I.to_oracle_image(m0).astype(np.uint8))
    xo, logo, _, _ = O.oslalm_run(g, I.to_oracle_sino(y), I.to_oracle_sino(w), dlo, So, np.zeros(O.img_shape(g)),
                                  M=M, beta=beta, delta=delta, nbr=nbr, n_iter=n_iter, bb=bb)
    return xo, So, logo


def rms_hu(xg, xo, So):
    return math.sqrt(((xg - xo)[So > 0] ** 2).mean()) / I.HU


@pytest.mark.parametrize("P,ny", [(2, 48), (3, 48), (8, 20)])
def test_row_slab_path_2d(ct, O, P, ny):
    """2D fan (c1 geometry, 48 x ny image): views split into per-rank blocks, reduce-scatter
    into padded row slabs.  P = 8 with 20 rows leaves the last rank an empty slab (rows 21..20)
    and ranks with 1-2 views of a subset."""
    base = I.config("c1")
    cfg = I.scaled(base, "c1v", nx=48, ny=ny, na=60)
    g = cfg.geom
    d = I.synthesize(cfg)
    m0 = I.support_mask(cfg)
    outs = run_virtual(ct, [g] * P, d["y"], d["w"], [m0] * P, 4, 6, cfg.beta, cfg.delta, 8)
    xo, So, logo = oracle_run(O, g, d["y"], d["w"], m0, 4, 6, cfg.beta, cfg.delta, 8)
    for r, (x, S, log) in enumerate(outs):
        assert np.array_equal(I.to_oracle_image(S).astype(np.uint8), So), r
        assert np.array_equal(log[:, 2], logo[:, 2]), r
        e = rms_hu(I.to_oracle_image(x), xo, So)
        assert e <= 0.5, (P, r, e)
    # every rank ends with the same all-gathered image
    for r in range(1, P):
        assert np.array_equal(outs[r][0], outs[0][0])


def _small3d(name):
    g = GU.small_geoms()[name]
    ell = [(0.0, 0.0, 0.0, 4.0, 3.5, 2.5, 0.0, 0.02), (1.0, -0.5, 0.3, 1.2, 0.8, 0.9, 0.4, 0.01)]
    d = I.noisy_data(g, ell, 1e5, 0.0, 81)
    m0 = torch.ones((g["ny"], g["nx"], g["nz"]), dtype=torch.uint8)
    return g, d, m0


@pytest.mark.parametrize("P,exchange", [(2, "full"), (3, "full"), (2, "band"), (3, "band"), (4, "band")])
def test_row_slab_path_3d(ct, O, P, exchange):
    """Helical cone beam (26 neighbours, row-slab 3D update kernel) with P virtual ranks, full
    reduce-scatter / all-gather or the band-limited exchange (z-band blocks of the partial
    back-projections and of x+, boundary rows for the stencil; the default for helical scans)."""
    g, d, m0 = _small3d("helical_c4")
    base = I.config("c4")
    outs = run_virtual(ct, [g] * P, d["y"], d["w"], [m0] * P, 4, 5, base.beta, base.delta, 26, exchange=exchange)
    xo, So, logo = oracle_run(O, g, d["y"], d["w"], m0, 4, 5, base.beta, base.delta, 26)
    for r, (x, S, log) in enumerate(outs):
        assert np.array_equal(log[:, 2], logo[:, 2]), r
        e = rms_hu(I.to_oracle_image(x), xo, So)
        assert e <= 0.5, (P, r, e)


@pytest.mark.parametrize("name,P,bb", [("helical_c4", 2, False), ("helical_c5", 3, False), ("helical_c4", 4, True)])
def test_zslab_path_virtual(ct, O, name, P, bb):
    """z-slab decomposition (NEXT-3) with P virtual ranks: partial subset sinograms summed over
    the slabs, residual on every ray, slab back-projection, xi (and BB sums) all-reduced, the
    26-neighbour update with the neighbours' boundary slices (halos of x and of S)."""
    from paper_1402_4381_b200 import host
    g, d, m0 = _small3d(name)
    base = I.config("c4")
    slabs = [host.rank_zslab(g["nz"], r, P) for r in range(P)]
    geoms = [I.slab_geom(g, z0, z1) for (z0, z1) in slabs]
    masks = [m0[..., z0:z1].contiguous() for (z0, z1) in slabs]
    outs = run_virtual(ct, geoms, d["y"], d["w"], masks, 4, 5, base.beta, base.delta, 26, zslab=True, bb=bb)
    xo, So, logo = oracle_run(O, g, d["y"], d["w"], m0, 4, 5, base.beta, base.delta, 26, bb=bb)
    x = np.concatenate([o[0] for o in outs], axis=2)
    S = np.concatenate([o[1] for o in outs], axis=2)
    assert np.array_equal(I.to_oracle_image(S).astype(np.uint8), So)
    for r in range(P):
        assert np.array_equal(outs[r][2][:, 2], logo[:, 2]), r
    e = rms_hu(I.to_oracle_image(x), xo, So)
    assert e <= 0.5, (name, P, e)


@pytest.mark.parametrize("P", [3, 5])
def test_zslab_window_exchange_long_helix(ct, O, P):
    """Windowed exchange of the helical z-slab path: a 6-turn helix over 40 slices
    split into P slabs, so a view's cone reaches only some of the slabs and only the views two
    ranks' windows share travel.  2 iterations against the oracle, and the FULL exchange (an
    all-reduce of every subset sinogram) gives the same image to fp32 rounding."""
    from paper_1402_4381_b200 import host
    g = GU.geom("cone_helical", nx=16, nz=40, dx=0.9766, dz=0.625, ns=28, ds=1.0239, nt=6, dt=1.0964, na=144,
                turns=6.0, pitch=0.8)
    ell = [(0.0, 0.0, 0.0, 5.5, 4.5, 10.0, 0.0, 0.02), (1.0, -0.5, 3.0, 2.0, 1.5, 3.0, 0.4, 0.01)]
    d = I.noisy_data(g, ell, 1e5, 0.0, 87)
    m0 = torch.ones((g["ny"], g["nx"], g["nz"]), dtype=torch.uint8)
    base = I.config("c4")
    slabs = [host.rank_zslab(g["nz"], r, P) for r in range(P)]
    geoms = [I.slab_geom(g, z0, z1) for (z0, z1) in slabs]
    masks = [m0[..., z0:z1].contiguous() for (z0, z1) in slabs]
    win = run_virtual(ct, geoms, d["y"], d["w"], masks, 4, 2, base.beta, base.delta, 26, zslab=True,
                      exchange="band")
    full = run_virtual(ct, geoms, d["y"], d["w"], masks, 4, 2, base.beta, base.delta, 26, zslab=True,
                       exchange="full")
    xo, So, logo = oracle_run(O, g, d["y"], d["w"], m0, 4, 2, base.beta, base.delta, 26)
    x = np.concatenate([o[0] for o in win], axis=2)
    xf = np.concatenate([o[0] for o in full], axis=2)
    for r in range(P):
        assert np.array_equal(win[r][2][:, 2], logo[:, 2]), r
    assert rms_hu(I.to_oracle_image(x), xo, So) <= 0.5
    assert np.abs(x - xf).max() <= 1e-5 * np.abs(xf).max()


def test_band_exchange_long_helix(ct, O):
    """Band-limited exchange where the bands are much narrower than the volume: a 6-turn helix
    over 40 slices, 3 ranks (each rank's view block sees about half of the slices), 2
    iterations against the oracle, and the FULL exchange gives the same image to fp32 rounding."""
    g = GU.geom("cone_helical", nx=16, nz=40, dx=0.9766, dz=0.625, ns=28, ds=1.0239, nt=6, dt=1.0964, na=144,
                turns=6.0, pitch=0.8)
    ell = [(0.0, 0.0, 0.0, 5.5, 4.5, 10.0, 0.0, 0.02), (1.0, -0.5, 3.0, 2.0, 1.5, 3.0, 0.4, 0.01)]
    d = I.noisy_data(g, ell, 1e5, 0.0, 83)
    m0 = torch.ones((g["ny"], g["nx"], g["nz"]), dtype=torch.uint8)
    base = I.config("c4")
    band = run_virtual(ct, [g] * 3, d["y"], d["w"], [m0] * 3, 4, 2, base.beta, base.delta, 26, exchange="band")
    full = run_virtual(ct, [g] * 3, d["y"], d["w"], [m0] * 3, 4, 2, base.beta, base.delta, 26, exchange="full")
    xo, So, logo = oracle_run(O, g, d["y"], d["w"], m0, 4, 2, base.beta, base.delta, 26)
    for r in range(3):
        assert np.array_equal(band[r][2][:, 2], logo[:, 2]), r
        e = rms_hu(I.to_oracle_image(band[r][0]), xo, So)
        assert e <= 0.5, (r, e)
        assert np.abs(band[r][0] - full[r][0]).max() <= 1e-5 * np.abs(full[r][0]).max()


def test_band_exchange_eight_ranks(ct, O):
    """Eight virtual ranks (the north_star's 8-GPU split) on a 16-row helical case with the band
    exchange: every rank owns two image rows and a sixth of a helical turn's views per subset."""
    g = GU.geom("cone_helical", nx=16, nz=24, dx=0.9766, dz=0.625, ns=28, ds=1.0239, nt=6, dt=1.0964, na=192,
                turns=4.0, pitch=0.8)
    ell = [(0.0, 0.0, 0.0, 5.5, 4.5, 6.0, 0.0, 0.02), (1.0, -0.5, 1.0, 2.0, 1.5, 3.0, 0.4, 0.01)]
    d = I.noisy_data(g, ell, 1e5, 0.0, 85)
    m0 = torch.ones((g["ny"], g["nx"], g["nz"]), dtype=torch.uint8)
    base = I.config("c4")
    outs = run_virtual(ct, [g] * 8, d["y"], d["w"], [m0] * 8, 4, 3, base.beta, base.delta, 26, exchange="band")
    xo, So, logo = oracle_run(O, g, d["y"], d["w"], m0, 4, 3, base.beta, base.delta, 26)
    for r in range(8):
        assert np.array_equal(outs[r][2][:, 2], logo[:, 2]), r
        e = rms_hu(I.to_oracle_image(outs[r][0]), xo, So)
        assert e <= 0.5, (r, e)
        assert np.array_equal(outs[r][0], outs[0][0])


def test_virtual_ranks_validation(ct):
    g = GU.small_geoms()["fan_c1"]
    a, b = ct.Geometry(g), ct.Geometry(g)
    with pytest.raises(ct.CTError, match="EINVAL"):
        ct.ct_comm_init_virtual([a.h, a.h])
    with pytest.raises(ct.CTError, match="EUNSUPPORTED"):
        ct.ct_comm_init_virtual([a.h, b.h], zslab=True)
    with pytest.raises(ct.CTError, match="EUNSUPPORTED"):
        ct.ct_comm_set_exchange(a.h, "band")
