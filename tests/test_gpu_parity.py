"""GPU parity: the sm_100a kernels (through the C ABI) against the fp64 oracle on the
same seeded inputs.  Tolerances (BASELINE.json north_star):
  projection / back-projection: relative L2 <= 1e-4 (per view and overall);
  regulariser gradient / curvature: elementwise, 1e-5 of the max + 1e-4 relative;
  OS-LALM image: RMS over S <= 0.5 HU (1 HU = 2e-5 mm^-1) with identical restart decisions;
  U counts (integer): exact.
"""
import math

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


MARGINS = []


@pytest.fixture(scope="module", autouse=True)
def _write_margins():
    """Record the measured parity errors (for DESIGN.md / profiles) when run on a GPU box."""
    yield
    import json
    import os
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    if MARGINS and os.path.isdir(out):
        with open(os.path.join(out, "parity_margins.json"), "w") as f:
            json.dump(MARGINS, f, indent=1)


def rel_l2(a, b, tag=None):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    v = float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
    if tag:
        MARGINS.append({"case": tag, "rel_l2": v})
    return v


def geoms_small():
    gs = GU.small_geoms()
    # ragged tiles / offsets / non-square: extra cases
    gs["fan_offsets"] = GU.geom("fan2d", nx=30, ny=22, dx=2.0, ns=77, ds=2.5, na=50, offx=3.1, offy=-2.2, offs=0.37,
                                start=11.0)
    gs["axial_offsets"] = GU.geom("cone_axial", nx=14, ny=11, nz=9, dx=1.5, dz=1.1, ns=37, ds=1.9, nt=13, dt=1.3,
                                  na=30, offx=-0.7, offz=0.4, offs=-0.21, offt=0.33)
    # 32 < nt <= 64: the pair-row forward kernel (odd nt: the last lane's second row is off
    # the detector); fine slices (kz >= 2): its general axial form
    gs["axial_rows41"] = GU.geom("cone_axial", nx=11, ny=9, nz=28, dx=0.9766, dz=0.625, ns=23, ds=1.0239, nt=41,
                                 dt=1.0964, na=20, offz=0.3, offt=0.4)
    gs["helical_fine_kz"] = GU.geom("cone_helical", nx=10, nz=40, dx=0.9766, dz=0.25, ns=21, ds=1.0239, nt=36,
                                    dt=1.0964, na=30, turns=2.0, pitch=0.7, start=5.0)
    # steep cones (|tz| > 0.08): the exact-sqrt l_theta instances of fwd3d2 / back3d (every
    # geometry above takes the polynomial form)
    gs["axial_steep"] = GU.geom("cone_axial", nx=12, nz=10, dx=2.0, dz=2.0, ns=30, ds=4.0, nt=40, dt=4.0, na=24,
                                dso=250.0, dsd=400.0)
    gs["helical_steep"] = GU.geom("cone_helical", nx=10, nz=16, dx=2.0, dz=2.0, ns=30, ds=4.0, nt=34, dt=4.0, na=40,
                                  dso=250.0, dsd=400.0, turns=2.0, pitch=0.6, start=9.0)
    return gs


def lpoly_tz_bound(g):
    """The |tz| bound ct_geom_create gates the polynomial l_theta on (restated, not imported)."""
    rb = (g["nt"] - 1) / 2.0 + g["offt"]
    rowmax = max(abs(-0.5 - rb), abs(g["nt"] - 0.5 - rb))
    rmax = math.hypot(0.5 * (g["nx"] - 1) * g["dx"] + abs(g["offx"]) + g["dx"],
                      0.5 * (g["ny"] - 1) * g["dy"] + abs(g["offy"]) + g["dy"])
    return rowmax * g["dt"] / g["dsd"] + g["dz"] / (g["dso"] - rmax)


def test_steep_geometries_take_the_exact_ltheta():
    gs = geoms_small()
    assert lpoly_tz_bound(gs["axial_steep"]) > 0.08 and lpoly_tz_bound(gs["helical_steep"]) > 0.08
    for k in ("axial_c3", "helical_c5", "axial_rows41", "helical_fine_kz"):
        assert lpoly_tz_bound(gs[k]) <= 0.08, k


def rand_image(g, seed, shape_abi):
    rng = np.random.default_rng(seed)
    return rng.random(shape_abi).astype(np.float32)


# --------------------------------------------------------------------------- projector

@pytest.mark.parametrize("name", list(geoms_small().keys()))
def test_fwd_back_small(ct, O, name):
    g = geoms_small()[name]
    geo = ct.Geometry(g)
    x = rand_image(g, 1, geo.img_shape)
    xt = torch.from_numpy(x).cuda()
    for views in ((0, 1, g["na"]), (1, 3, (g["na"] - 1 + 2) // 3), (2, 5, 1)):
        yg = geo.fwd(xt, views).cpu().numpy()
        yo = O.fwd(g, I.to_oracle_image(x), *views)
        assert rel_l2(I.to_oracle_sino(yg), yo, f"fwd {name} {views}") <= 1e-4, name
        p = np.random.default_rng(2).random(yg.shape).astype(np.float32)
        bg = geo.back(torch.from_numpy(p).cuda(), views).cpu().numpy()
        bo = O.back(g, I.to_oracle_sino(p), *views)
        assert rel_l2(I.to_oracle_image(bg), bo, f"back {name} {views}") <= 1e-4, name


@pytest.mark.parametrize("name", ["fan_c2", "axial_c3", "helical_c5", "axial_steep", "helical_steep"])
def test_adjoint_gpu(ct, name):
    g = geoms_small()[name]
    geo = ct.Geometry(g)
    x = torch.from_numpy(rand_image(g, 3, geo.img_shape)).cuda()
    p = torch.rand(geo.sino_shape(g["na"]), device="cuda")
    lhs = (geo.fwd(x).double() * p.double()).sum().item()
    rhs = (x.double() * geo.back(p).double()).sum().item()
    assert abs(lhs - rhs) <= 1e-5 * abs(lhs)


def test_back_accumulate_and_empty_views(ct):
    g = geoms_small()["axial_c3"]
    geo = ct.Geometry(g)
    p = torch.rand(geo.sino_shape(g["na"]), device="cuda")
    full = geo.back(p)
    acc = torch.zeros_like(full)
    # virtual ranks: contiguous view blocks, partial back-projections summed
    from paper_1402_4381_b200 import host
    for r in range(3):
        k0, n = host.rank_view_block(g["na"], r, 3)
        geo.back(p[k0:k0 + n].contiguous(), (k0, 1, n), out=acc, accumulate=True)
    assert rel_l2(acc.cpu().numpy(), full.cpu().numpy()) <= 1e-6
    empty = geo.back(p[:0].contiguous(), (0, 1, 0))
    assert torch.count_nonzero(empty).item() == 0
    with pytest.raises(ct.CTError, match="CT_EINVAL"):
        geo.back(p, (5, 1, g["na"]))


def test_determinism_3d_iteration(ct):
    """Bit-reproducible OS-LALM iterations in 3D (helical, 26 neighbours): two fresh states on
    the same inputs give identical images (no float atomics anywhere on the path)."""
    g = GU.small_geoms()["helical_c5"]
    ell = [(0.0, 0.0, 0.0, 4.0, 3.5, 2.5, 0.0, 0.02)]
    d = I.noisy_data(g, ell, 1e5, 0.0, 3)
    geo = ct.Geometry(g)
    dl, S = geo.sqs_denom(d["w"].cuda(), torch.ones(geo.img_shape, dtype=torch.uint8).cuda())
    outs = []
    for _ in range(2):
        sol = ct.OSLALM(geo, 4, beta=2.0 ** 10, delta=2e-4, nbr=26)
        sol.set_data(d["y"].cuda(), d["w"].cuda(), dl, S)
        x = torch.zeros(geo.img_shape, device="cuda")
        sol.run(x, 3)
        outs.append(x)
    assert torch.equal(outs[0], outs[1])


def test_determinism(ct):
    g = I.config("c1").geom
    geo = ct.Geometry(g)
    x = torch.rand(geo.img_shape, device="cuda")
    a = geo.fwd(x); b = geo.fwd(x)
    assert torch.equal(a, b)
    p = torch.rand_like(a)
    assert torch.equal(geo.back(p), geo.back(p))


@pytest.mark.parametrize("cname,views", [
    ("c1", None),
    ("c2", (5, 24, 41)),          # one c2 subset (41 views) at full image/detector size
    ("c3", (7, 24, 41)),          # one c3 subset
    ("c4", (1000, 97, 6)),        # helical: sampled views
    ("c5", (3000, 211, 5)),
])
def test_projector_full_size(ct, O, cname, views):
    """Full BASELINE sizes in the bench's launch configuration, on sampled view lists."""
    cfg = I.config(cname)
    g = cfg.geom
    geo = ct.Geometry(g)
    views = views or (0, 1, g["na"])
    rng = np.random.default_rng(4)
    x = (rng.random(geo.img_shape).astype(np.float32) * 0.02) * I.support_mask(cfg).numpy()
    xt = torch.from_numpy(x).cuda()
    yg = geo.fwd(xt, views).cpu().numpy()
    yo = O.fwd(g, I.to_oracle_image(x), *views)
    assert rel_l2(I.to_oracle_sino(yg), yo, f"fwd full-size {cname} {views}") <= 1e-4
    for k in range(views[2]):
        assert rel_l2(I.to_oracle_sino(yg)[k], yo[k]) <= 1e-4
    p = rng.random(yg.shape).astype(np.float32)
    bg = geo.back(torch.from_numpy(p).cuda(), views).cpu().numpy()
    bo = O.back(g, I.to_oracle_sino(p), *views)
    assert rel_l2(I.to_oracle_image(bg), bo, f"back full-size {cname} {views}") <= 1e-4


@pytest.mark.parametrize("scale", [1e-6, 1e4])
def test_fan_forward_input_scale(ct, O, scale):
    """The 2D forward's 64-bit fixed-point tile sums (unit 2^-40, include/ct_oslalm.h) keep the
    1e-4 parity bound for images scaled 1e-6 and 1e4 times attenuation scale (c2 subset)."""
    cfg = I.config("c2")
    g = cfg.geom
    geo = ct.Geometry(g)
    views = (5, 24, 41)
    rng = np.random.default_rng(14)
    x = (rng.random(geo.img_shape) * 0.02 * scale * I.support_mask(cfg).numpy()).astype(np.float32)
    yg = I.to_oracle_sino(geo.fwd(torch.from_numpy(x).cuda(), views).cpu().numpy())
    yo = O.fwd(g, I.to_oracle_image(x), *views)
    e = rel_l2(yg, yo, f"fwd c2 subset, x scaled {scale:g}")
    assert e <= 1e-4, e
    for k in range(views[2]):
        assert rel_l2(yg[k], yo[k]) <= 1e-4


def test_cone_forward_two_streams(ct):
    """Cone-beam projections through ONE geometry on two streams at once (different images):
    each equals its single-stream result (per-call scratch)."""
    g = I.config("c3").geom
    geo = ct.Geometry(g)
    views = (3, 24, 41)
    x1 = torch.rand(geo.img_shape, device="cuda")
    x2 = torch.zeros(geo.img_shape, device="cuda")
    x2[200:300, 100:400, :] = torch.rand(100, 300, g["nz"], device="cuda")   # different zero columns
    r1, r2 = geo.fwd(x1, views), geo.fwd(x2, views)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    outs = []
    for _ in range(3):
        a = torch.empty_like(r1); b = torch.empty_like(r2)
        ct.ct_fwd_proj(geo.h, views, x1, a, stream=s1)
        ct.ct_fwd_proj(geo.h, views, x2, b, stream=s2)
        outs.append((a, b))
    torch.cuda.synchronize()
    for a, b in outs:
        assert torch.equal(a, r1) and torch.equal(b, r2)


@pytest.mark.parametrize("name", ["fan_c1", "axial_c3", "helical_c4", "fan_offsets"])
def test_count_vv_exact(ct, O, name):
    g = geoms_small()[name]
    geo = ct.Geometry(g)
    rng = np.random.default_rng(5)
    m = (rng.random(geo.img_shape) > 0.2).astype(np.uint8)
    assert geo.count_vv(torch.from_numpy(m).cuda()) == O.count_vv(g, I.to_oracle_image(m).astype(np.uint8))
    assert geo.count_vv(torch.from_numpy(m).cuda(), (1, 4, (g["na"] - 1 + 3) // 4)) == \
        O.count_vv(g, I.to_oracle_image(m).astype(np.uint8), 1, 4)


def test_count_vv_c2_exact(ct, O):
    cfg = I.config("c2")
    geo = ct.Geometry(cfg.geom)
    m = I.support_mask(cfg)
    assert geo.count_vv(m.cuda(), (3, 24, 41)) == O.count_vv(cfg.geom, I.to_oracle_image(m).astype(np.uint8), 3, 24)


# --------------------------------------------------------------------------- D_L, regulariser

@pytest.mark.parametrize("name", ["c1", "axial_c3", "helical_c4"])
def test_sqs_denom(ct, O, name):
    if name == "c1":
        cfg = I.config("c1"); g = cfg.geom
        m0 = I.support_mask(cfg).numpy()
        w = I.synthesize(cfg)["w"].numpy()
    else:
        g = geoms_small()[name]
        shape = (g["ny"], g["nx"], g["nz"])
        m0 = np.ones(shape, np.uint8)
        w = (np.random.default_rng(6).random((g["na"], g["ns"], g["nt"])) * 100 + 1).astype(np.float32)
    geo = ct.Geometry(g)
    dl, m = geo.sqs_denom(torch.from_numpy(w).cuda(), torch.from_numpy(m0).cuda())
    dlo, mo = O.sqs_denom(g, I.to_oracle_sino(w), I.to_oracle_image(m0).astype(np.uint8))
    assert np.array_equal(I.to_oracle_image(m.cpu().numpy()).astype(np.uint8), mo)
    assert rel_l2(I.to_oracle_image(dl.cpu().numpy()), dlo, f"D_L {name}") <= 1e-4


@pytest.mark.parametrize("name,nbr", [("fan_c2", 8), ("axial_c3", 26), ("axial_offsets", 26), ("axial_c3", 8)])
def test_reg_grad(ct, O, name, nbr):
    g = geoms_small()[name]
    geo = ct.Geometry(g)
    rng = np.random.default_rng(7)
    x = (rng.random(geo.img_shape) * 0.03).astype(np.float32)
    m = (rng.random(geo.img_shape) > 0.1).astype(np.uint8)
    beta, delta = 2.0 ** 10, 2e-4
    gr, cu = geo.reg_grad(torch.from_numpy(x).cuda(), torch.from_numpy(m).cuda(), beta, delta, nbr)
    gro, cuo = O.reg_grad(g, beta, delta, nbr, I.to_oracle_image(m).astype(np.uint8), I.to_oracle_image(x))
    gr = I.to_oracle_image(gr.cpu().numpy()); cu = I.to_oracle_image(cu.cpu().numpy())
    # 1e-5 relative elementwise; the absolute floor (1e-6 of the max) covers the
    # gradients that cancel to ~0 (26 terms of both signs, MUFU reciprocal ~1 ulp per term)
    MARGINS.append({"case": f"reg_grad {name} nbr={nbr}", "grad_rel_max": float((np.abs(gr - gro) / np.maximum(np.abs(gro), 1e-30))[np.abs(gro) > 1e-3 * np.abs(gro).max()].max()),
                    "grad_err_over_max": float(np.abs(gr - gro).max() / np.abs(gro).max()),
                    "curv_rel_max": float((np.abs(cu - cuo) / np.maximum(np.abs(cuo), 1e-30))[cuo > 0].max())})
    assert np.all(np.abs(gr - gro) <= 1e-6 * np.abs(gro).max() + 1e-5 * np.abs(gro))
    assert np.all(np.abs(cu - cuo) <= 1e-6 * np.abs(cuo).max() + 1e-5 * np.abs(cuo))


# --------------------------------------------------------------------------- OS-LALM

def _run_pair(ct, O, cfg, n_iter, M=None, mode="continuation", rho_fixed=1.0, x0=None, inner="sqs", n_inner=1):
    g = cfg.geom
    M = M or cfg.M
    d = I.synthesize(cfg)
    y, w = d["y"], d["w"]
    m0 = I.support_mask(cfg)
    geo = ct.Geometry(g)
    dl, S = geo.sqs_denom(w.cuda(), m0.cuda())
    dlo, So = O.sqs_denom(g, I.to_oracle_sino(w), I.to_oracle_image(m0).astype(np.uint8))
    assert np.array_equal(I.to_oracle_image(S.cpu().numpy()).astype(np.uint8), So)
    sol = ct.OSLALM(geo, M, mode=mode, rho_fixed=rho_fixed, beta=cfg.beta, delta=cfg.delta, nbr=cfg.nbr,
                    inner=inner, n_inner=n_inner)
    yc, wc = y.cuda(), w.cuda()
    sol.set_data(yc, wc, dl, S)
    x = torch.zeros(geo.img_shape, device="cuda") if x0 is None else x0.clone().cuda()
    log = sol.run(x, n_iter, log=True)
    xo, logo, _, _ = O.oslalm_run(g, I.to_oracle_sino(y), I.to_oracle_sino(w), dlo, So,
                                  np.zeros(O.img_shape(g)) if x0 is None else I.to_oracle_image(x0),
                                  M=M, mode=mode, rho_fixed=rho_fixed, beta=cfg.beta, delta=cfg.delta, nbr=cfg.nbr,
                                  n_iter=n_iter, inner=inner, n_inner=n_inner)
    xg = I.to_oracle_image(x.cpu().numpy())
    Sm = So > 0
    rms_hu = math.sqrt(((xg - xo)[Sm] ** 2).mean()) / I.HU
    MARGINS.append({"case": f"OS-LALM {cfg.name} M={M} {mode} rho={rho_fixed} iters={n_iter} inner={inner}x{n_inner}",
                    "rms_HU": rms_hu,
                    "restarts_gpu": int(np.array(log)[:, 2].sum()), "restarts_oracle": int(logo[:, 2].sum())})
    return xg, xo, np.array(log), logo, rms_hu


def test_oslalm_c1_full(ct, O):
    """c1 (BASELINE configs[0]): 20 iterations, M = 4, continuation: <= 0.5 HU RMS on S."""
    cfg = I.config("c1")
    xg, xo, log, logo, rms = _run_pair(ct, O, cfg, cfg.n_iter)
    assert rms <= 0.5, rms
    assert np.array_equal(log[:, 2], logo[:, 2])          # identical restart decisions
    assert np.allclose(log[:, 0], logo[:, 0], rtol=1e-12)  # identical rho trajectory
    assert np.abs(xo).max() > 0.01                         # a non-trivial reconstruction


@pytest.mark.parametrize("mode,rho", [("fixed", 1.0), ("fixed", 0.2), ("continuation", 1.0)])
def test_oslalm_modes_small(ct, O, mode, rho):
    cfg = I.scaled(I.config("c1"), "c1s", nx=48, ny=48, na=90)
    xg, xo, log, logo, rms = _run_pair(ct, O, cfg, 6, M=5 if mode == "continuation" else 4, mode=mode, rho_fixed=rho)
    assert rms <= 0.05, rms      # odd M exercises the graph's buffer-parity path
    assert np.array_equal(log[:, 2], logo[:, 2])


def test_oslalm_M1_restarts(ct, O):
    """M = 1 with continuation fires restarts (V7); decisions must match the oracle."""
    cfg = I.scaled(I.config("c1"), "c1m1", nx=32, ny=32, na=60)
    xg, xo, log, logo, rms = _run_pair(ct, O, cfg, 60, M=1)
    assert logo[:, 2].sum() >= 1
    assert np.array_equal(log[:, 2], logo[:, 2])
    assert rms <= 0.05, rms


@pytest.mark.parametrize("name", ["axial_c3", "helical_c4"])
def test_oslalm_3d_small(ct, O, name):
    g = geoms_small()[name]
    base = I.config("c3")
    cfg = I.ScanConfig(name, g, 4, 8, base.beta, base.delta, 26, 1e5, 0.0, "body3d", body_z=2.0)
    cfg.extra = {}
    # phantom scaled into the small grid: a water cylinder + inserts
    ell = [(0.0, 0.0, 0.0, 4.0, 3.5, 2.0, 0.0, 0.02), (1.0, -0.5, 0.3, 1.2, 0.8, 0.9, 0.4, 0.01)]
    d = I.noisy_data(g, ell, 1e5, 0.0, 77)
    geo = ct.Geometry(g)
    m0 = torch.ones(geo.img_shape, dtype=torch.uint8)
    dl, S = geo.sqs_denom(d["w"].cuda(), m0.cuda())
    dlo, So = O.sqs_denom(g, I.to_oracle_sino(d["w"]), I.to_oracle_image(m0).astype(np.uint8))
    sol = ct.OSLALM(geo, 4, beta=cfg.beta, delta=cfg.delta, nbr=26)
    sol.set_data(d["y"].cuda(), d["w"].cuda(), dl, S)
    x = torch.zeros(geo.img_shape, device="cuda")
    log = np.array(sol.run(x, 8, log=True))
    xo, logo, _, _ = O.oslalm_run(g, I.to_oracle_sino(d["y"]), I.to_oracle_sino(d["w"]), dlo, So,
                                  np.zeros(O.img_shape(g)), M=4, beta=cfg.beta, delta=cfg.delta, nbr=26, n_iter=8)
    xg = I.to_oracle_image(x.cpu().numpy())
    rms = math.sqrt(((xg - xo)[So > 0] ** 2).mean()) / I.HU
    assert rms <= 0.5, rms
    assert np.array_equal(log[:, 2], logo[:, 2])


def test_iter_equals_run_and_state(ct):
    cfg = I.config("c1")
    d = I.synthesize(cfg)
    geo = ct.Geometry(cfg.geom)
    dl, S = geo.sqs_denom(d["w"].cuda(), I.support_mask(cfg).cuda())
    a = ct.OSLALM(geo, 4, beta=cfg.beta, delta=cfg.delta, nbr=8)
    b = ct.OSLALM(geo, 4, beta=cfg.beta, delta=cfg.delta, nbr=8)
    for s in (a, b):
        s.set_data(d["y"].cuda(), d["w"].cuda(), dl, S)
    xa = torch.zeros(geo.img_shape, device="cuda"); xb = xa.clone()
    a.run(xa, 5)
    for _ in range(5):
        b.iterate(xb)
    torch.cuda.synchronize()
    assert torch.equal(xa, xb)
    assert a.scalars() == b.scalars()
    assert a.scalars()[2] == 20
    assert torch.equal(a.split_gradient(), b.split_gradient())


@pytest.mark.parametrize("inner", ["sqs", "fista"])
def test_exchange_path_single_rank(ct, inner):
    """The multi-GPU exchange path run with a 1-rank communicator equals the fused
    single-GPU path (2D c1).  SQS inner step: per-rank partial back-projection, NCCL
    reduce-scatter into the rank's row slab, slab g-update + xi, xi all-reduce, K4, slab
    update and all-gather of x+.  FISTA inner loop: all-reduce of G+ and the unfused g-update."""
    cfg = I.config("c1")
    d = I.synthesize(cfg)
    outs = []
    for use_comm in (False, True):
        geo = ct.Geometry(cfg.geom)
        if use_comm:
            geo.comm_init(0, 1, ct.ct_comm_get_unique_id())
        dl, S = geo.sqs_denom(d["w"].cuda(), I.support_mask(cfg).cuda())
        sol = ct.OSLALM(geo, cfg.M, beta=cfg.beta, delta=cfg.delta, nbr=cfg.nbr, inner=inner,
                        n_inner=2 if inner == "fista" else 1)
        sol.set_data(d["y"].cuda(), d["w"].cuda(), dl, S)
        x = torch.zeros(geo.img_shape, device="cuda")
        log = np.array(sol.run(x, 5, log=True))
        outs.append((x.cpu().numpy(), log))
    (xa, la), (xb, lb) = outs
    assert np.array_equal(la[:, 2], lb[:, 2])
    # xi: same terms, different fp64 summation order (block partials of another grid)
    assert np.allclose(la[:, 1], lb[:, 1], rtol=1e-5)
    assert rel_l2(xb, xa, f"exchange path c1 {inner}") <= 1e-6


def test_exchange_path_single_rank_3d(ct, O):
    """Slab exchange path on a small helical cone-beam case (26 neighbours, row-slab 3D
    update kernel), 1-rank communicator, against the fp64 oracle.  (The fused and exchange
    back-projection epilogues are separate template instances whose last-bit rounding can
    differ; OS iterations then drift apart at the 1e-5 level, so the bar is the oracle's.)"""
    g = geoms_small()["helical_c4"]
    base = I.config("c4")
    ell = [(0.0, 0.0, 0.0, 4.0, 3.5, 2.5, 0.0, 0.02), (1.0, -0.5, 0.3, 1.2, 0.8, 0.9, 0.4, 0.01)]
    d = I.noisy_data(g, ell, 1e5, 0.0, 78)
    geo = ct.Geometry(g)
    geo.comm_init(0, 1, ct.ct_comm_get_unique_id())
    m0 = torch.ones(geo.img_shape, dtype=torch.uint8)
    dl, S = geo.sqs_denom(d["w"].cuda(), m0.cuda())
    dlo, So = O.sqs_denom(g, I.to_oracle_sino(d["w"]), I.to_oracle_image(m0).astype(np.uint8))
    sol = ct.OSLALM(geo, 4, beta=base.beta, delta=base.delta, nbr=26)
    sol.set_data(d["y"].cuda(), d["w"].cuda(), dl, S)
    x = torch.zeros(geo.img_shape, device="cuda")
    log = np.array(sol.run(x, 6, log=True))
    xo, logo, _, _ = O.oslalm_run(g, I.to_oracle_sino(d["y"]), I.to_oracle_sino(d["w"]), dlo, So,
                                  np.zeros(O.img_shape(g)), M=4, beta=base.beta, delta=base.delta, nbr=26, n_iter=6)
    xg = I.to_oracle_image(x.cpu().numpy())
    rms = math.sqrt(((xg - xo)[So > 0] ** 2).mean()) / I.HU
    MARGINS.append({"case": "exchange path helical_c4 (1-rank slab) vs oracle", "rms_HU": rms})
    assert rms <= 0.5, rms
    assert np.array_equal(log[:, 2], logo[:, 2])


@pytest.mark.parametrize("n_inner", [1, 2, 5])
def test_oslalm_inner_fista(ct, O, n_inner):
    """NEXT-1: n warm-started inner FISTA iterations vs the oracle, c1 geometry."""
    cfg = I.config("c1")
    xg, xo, log, logo, rms = _run_pair(ct, O, cfg, 8, inner="fista", n_inner=n_inner)
    assert rms <= 0.5, rms
    assert np.array_equal(log[:, 2], logo[:, 2])


def test_oslalm_inner_fista_3d(ct, O):
    g = geoms_small()["axial_c3"]
    ell = [(0.0, 0.0, 0.0, 4.0, 3.5, 2.0, 0.0, 0.02), (1.0, -0.5, 0.3, 1.2, 0.8, 0.9, 0.4, 0.01)]
    d = I.noisy_data(g, ell, 1e5, 0.0, 78)
    geo = ct.Geometry(g)
    m0 = torch.ones(geo.img_shape, dtype=torch.uint8)
    dl, S = geo.sqs_denom(d["w"].cuda(), m0.cuda())
    dlo, So = O.sqs_denom(g, I.to_oracle_sino(d["w"]), I.to_oracle_image(m0).astype(np.uint8))
    beta, delta = 2.0 ** 10, 2e-4
    sol = ct.OSLALM(geo, 4, beta=beta, delta=delta, nbr=26, inner="fista", n_inner=3)
    sol.set_data(d["y"].cuda(), d["w"].cuda(), dl, S)
    x = torch.zeros(geo.img_shape, device="cuda")
    sol.run(x, 6)
    xo, _, _, _ = O.oslalm_run(g, I.to_oracle_sino(d["y"]), I.to_oracle_sino(d["w"]), dlo, So, np.zeros(O.img_shape(g)),
                               M=4, beta=beta, delta=delta, nbr=26, n_iter=6, inner="fista", n_inner=3)
    xg = I.to_oracle_image(x.cpu().numpy())
    rms = math.sqrt(((xg - xo)[So > 0] ** 2).mean()) / I.HU
    MARGINS.append({"case": "OS-LALM axial_c3 small inner=fista x3", "rms_HU": rms})
    assert rms <= 0.5, rms


def test_inner_mode_validation(ct):
    geo = ct.Geometry(I.config("c1").geom)
    with pytest.raises(ct.CTError, match="CT_EINVAL"):
        ct.OSLALM(geo, 4, beta=1.0, delta=1e-3, nbr=8, inner="sqs", n_inner=2)
    with pytest.raises(ct.CTError, match="CT_EINVAL"):
        ct.OSLALM(geo, 4, beta=1.0, delta=1e-3, nbr=8, inner="fista", n_inner=0)


# --------------------------------------------------------------------------- BB (NEXT-2)

@pytest.mark.parametrize("M,n_iter,comm", [(4, 12, False), (1, 30, False), (4, 10, True)])
def test_oslalm_bb_c1(ct, O, M, n_iter, comm):
    """Barzilai-Borwein scaling H_k = alpha_k D_L (reading B-BB) against
    the fp64 oracle: alpha per outer iteration, restart decisions and the image (<= 0.5 HU).
    comm = True runs the 1-rank slab exchange path (BB sums all-reduced)."""
    cfg = I.config("c1")
    g = cfg.geom
    d = I.synthesize(cfg)
    geo = ct.Geometry(g)
    if comm:
        geo.comm_init(0, 1, ct.ct_comm_get_unique_id())
    m0 = I.support_mask(cfg)
    dl, S = geo.sqs_denom(d["w"].cuda(), m0.cuda())
    sol = ct.OSLALM(geo, M, beta=cfg.beta, delta=cfg.delta, nbr=8, bb=True)
    sol.set_data(d["y"].cuda(), d["w"].cuda(), dl, S)
    x = torch.zeros(geo.img_shape, device="cuda")
    alphas, logs = [1.0], []
    for k in range(n_iter):
        logs.append(np.array(sol.run(x, 1, log=True)))
        alphas.append(sol.alpha())
    log = np.concatenate(logs)
    dlo, So = O.sqs_denom(g, I.to_oracle_sino(d["w"]), I.to_oracle_image(m0).astype(np.uint8))
    ao = np.zeros(n_iter)
    xo, logo, _, _ = O.oslalm_run(g, I.to_oracle_sino(d["y"]), I.to_oracle_sino(d["w"]), dlo, So,
                                  np.zeros(O.img_shape(g)), M=M, beta=cfg.beta, delta=cfg.delta, nbr=8,
                                  n_iter=n_iter, bb=True, alpha_out=ao)
    a_gpu = np.array(alphas[:n_iter])
    assert (ao[2:] < 1.0).any()
    assert np.allclose(a_gpu, ao, rtol=2e-3), (a_gpu, ao)
    assert np.array_equal(log[:, 2], logo[:, 2])
    xg = I.to_oracle_image(x.cpu().numpy())
    rms = math.sqrt(((xg - xo)[So > 0] ** 2).mean()) / I.HU
    MARGINS.append({"case": f"OS-LALM+BB c1 M={M} iters={n_iter} comm={comm}", "rms_HU": rms,
                    "alpha_max_rel": float(np.abs(a_gpu / ao - 1).max())})
    assert rms <= 0.5, rms
    assert np.abs(xo).max() > 0.005   # a non-trivial image (BB with OS can transiently collapse to 0)


# --------------------------------------------------------------------------- FBP (NEXT-4)

@pytest.mark.parametrize("name", ["fan_c1", "fan_c2", "fan_offsets", "axial_c3", "axial_offsets"])
def test_fbp_small(ct, O, name):
    """GPU FBP / FDK (ct_fbp) vs the fp64 oracle on random sinograms: relative L2 <= 1e-4."""
    g = geoms_small()[name]
    geo = ct.Geometry(g)
    rng = np.random.default_rng(5)
    y = rng.random(geo.sino_shape(g["na"])).astype(np.float32)
    xg = geo.fbp(torch.from_numpy(y).cuda()).cpu().numpy()
    xo = O.fbp(g, I.to_oracle_sino(y))
    assert rel_l2(I.to_oracle_image(xg), xo, f"fbp {name}") <= 1e-4


def test_fbp_full_size_c2_and_partial_orbit_rejected(ct, O):
    """c2 FBP of the synthetic scan vs the oracle (rel L2 <= 1e-4); a circular orbit that is
    not one full turn -> CT_EUNSUPPORTED."""
    cfg = I.config("c2")
    d = I.synthesize(cfg)
    geo = ct.Geometry(cfg.geom)
    xg = geo.fbp(d["y"].cuda()).cpu().numpy()
    xo = O.fbp(cfg.geom, I.to_oracle_sino(d["y"]))
    assert rel_l2(I.to_oracle_image(xg), xo, "fbp full-size c2") <= 1e-4
    half = GU.geom("cone_axial", nx=12, nz=6, dx=0.9766, dz=0.625, ns=24, ds=1.0239, nt=8, dt=1.0964, na=24, turns=0.5)
    with pytest.raises(ct.CTError, match="EUNSUPPORTED"):
        ct.Geometry(half).fbp(torch.zeros(ct.Geometry(half).sino_shape(24), device="cuda"))


@pytest.mark.parametrize("name", ["helical_c4", "helical_c5", "c5_coarse"])
def test_fbp_helical(ct, O, name):
    """Helical FBP initial image (reading B-FBP-H: back-projection over the views that see the
    voxel, normalised by their number) vs the oracle: small helical geometries on random data,
    and the c5 scan (full detector and 6888 views) on the central 128^2 x 16 voxels with its data."""
    if name == "c5_coarse":
        g = I.slab_geom(dict(I.config("c5").geom, nx=128, ny=128), 152, 168)   # central 125 mm x 10 mm
        cfg = I.ScanConfig("c5", g, 24, 1, 1.0, 1.0, 26, 5e4, 0.0, "body3d", body_z=70.0)
        y = I.synthesize(cfg, device="cuda", views_per_chunk=8)["y"]
    else:
        g = geoms_small()[name]
        y = torch.rand((g["na"], g["ns"], g["nt"]), device="cuda", generator=torch.Generator("cuda").manual_seed(5))
    geo = ct.Geometry(g)
    xg = geo.fbp(y).cpu().numpy()
    xo = O.fbp(g, I.to_oracle_sino(y.cpu()))
    assert np.abs(xo).max() > 0
    assert rel_l2(I.to_oracle_image(xg), xo, f"fbp helical {name}") <= 1e-4

def test_oslalm_from_fbp_init(ct, O):
    """OS-LALM started from the FBP image matches the oracle started from its own FBP."""
    cfg = I.config("c1")
    g = cfg.geom
    d = I.synthesize(cfg)
    geo = ct.Geometry(g)
    m0 = I.support_mask(cfg)
    dl, S = geo.sqs_denom(d["w"].cuda(), m0.cuda())
    x = geo.fbp(d["y"].cuda())
    sol = ct.OSLALM(geo, cfg.M, beta=cfg.beta, delta=cfg.delta, nbr=8)
    sol.set_data(d["y"].cuda(), d["w"].cuda(), dl, S)
    log = np.array(sol.run(x, 8, log=True))
    dlo, So = O.sqs_denom(g, I.to_oracle_sino(d["w"]), I.to_oracle_image(m0).astype(np.uint8))
    x0 = O.fbp(g, I.to_oracle_sino(d["y"]))
    xo, logo, _, _ = O.oslalm_run(g, I.to_oracle_sino(d["y"]), I.to_oracle_sino(d["w"]), dlo, So, x0,
                                  M=cfg.M, beta=cfg.beta, delta=cfg.delta, nbr=8, n_iter=8)
    xg = I.to_oracle_image(x.cpu().numpy())
    rms = math.sqrt(((xg - xo)[So > 0] ** 2).mean()) / I.HU
    MARGINS.append({"case": "OS-LALM c1 from FBP x0, 8 iters", "rms_HU": rms})
    assert rms <= 0.5, rms
    assert np.array_equal(log[:, 2], logo[:, 2])


# --------------------------------------------------------------------------- edge cases

def test_axis_aligned_and_diagonal_views(ct, O):
    """Views at multiples of 45 degrees: pixel edges parallel to the centre ray (zero rise or
    fall width, degenerate trapezoids) and diagonal views (zero flat part); 2D and 3D."""
    for g in (GU.geom("fan2d", nx=20, dx=4.0, ns=40, ds=8.1912, na=8),
              GU.geom("cone_axial", nx=12, nz=6, dx=0.9766, dz=0.625, ns=24, ds=1.0239, nt=8, dt=1.0964, na=8)):
        geo = ct.Geometry(g)
        x = rand_image(g, 3, geo.img_shape)
        yg = geo.fwd(torch.from_numpy(x).cuda(), (0, 1, g["na"])).cpu().numpy()
        yo = O.fwd(g, I.to_oracle_image(x), 0, 1, g["na"])
        assert np.isfinite(yg).all()
        assert rel_l2(I.to_oracle_sino(yg), yo, f"fwd 45deg {g['kind']}") <= 1e-4
        p = np.random.default_rng(4).random(geo.sino_shape(g["na"])).astype(np.float32)
        bg = geo.back(torch.from_numpy(p).cuda()).cpu().numpy()
        bo = O.back(g, I.to_oracle_sino(p), 0, 1, g["na"])
        assert rel_l2(I.to_oracle_image(bg), bo, f"back 45deg {g['kind']}") <= 1e-4


def test_empty_forward_and_one_view_subsets(ct, O):
    """count = 0 forward projection is a no-op; M = na (one view per subset) OS-LALM matches
    the oracle."""
    g = geoms_small()["fan_c1"]
    geo = ct.Geometry(g)
    y = torch.full(geo.sino_shape(1), 7.0, device="cuda")
    ct.ct_fwd_proj(geo.h, (0, 1, 0), torch.zeros(geo.img_shape, device="cuda"), y)
    assert (y == 7.0).all()
    ell = [(0.0, 0.0, 0.0, 30.0, 25.0, float("inf"), 0.2, 0.02)]
    d = I.noisy_data(g, ell, 1e5, 0.0, 9)
    m0 = torch.ones(geo.img_shape, dtype=torch.uint8)
    dl, S = geo.sqs_denom(d["w"].cuda(), m0.cuda())
    M = g["na"]
    sol = ct.OSLALM(geo, M, beta=2.0 ** 8, delta=2e-4, nbr=8)
    sol.set_data(d["y"].cuda(), d["w"].cuda(), dl, S)
    x = torch.zeros(geo.img_shape, device="cuda")
    log = np.array(sol.run(x, 2, log=True))
    dlo, So = O.sqs_denom(g, I.to_oracle_sino(d["w"]), I.to_oracle_image(m0).astype(np.uint8))
    xo, logo, _, _ = O.oslalm_run(g, I.to_oracle_sino(d["y"]), I.to_oracle_sino(d["w"]), dlo, So,
                                  np.zeros(O.img_shape(g)), M=M, beta=2.0 ** 8, delta=2e-4, nbr=8, n_iter=2)
    xg = I.to_oracle_image(x.cpu().numpy())
    rms = math.sqrt(((xg - xo)[So > 0] ** 2).mean()) / I.HU
    assert rms <= 0.5, rms
    assert np.array_equal(log[:, 2], logo[:, 2])


# --------------------------------------------------------------------------- z-slabs (NEXT-3)

@pytest.mark.parametrize("name", ["axial_c3", "helical_c4", "helical_c5"])
def test_zslab_decomposition(ct, name):
    """A x is separable over voxels: the slab geometries' forward projections sum to the full
    one, and their back-projections are the full back-projection's slices (NEXT-3)."""
    from paper_1402_4381_b200 import host
    g = geoms_small()[name]
    geo = ct.Geometry(g)
    rng = np.random.default_rng(8)
    x = torch.from_numpy(rng.random(geo.img_shape).astype(np.float32)).cuda()
    y = torch.from_numpy(rng.random(geo.sino_shape(g["na"])).astype(np.float32)).cuda()
    yf, bf = geo.fwd(x), geo.back(y)
    ysum = torch.zeros_like(yf)
    for r in range(3):
        z0, z1 = host.rank_zslab(g["nz"], r, 3)
        gs = ct.Geometry(I.slab_geom(g, z0, z1))
        ysum += gs.fwd(x[..., z0:z1].contiguous())
        bs = gs.back(y)
        assert rel_l2(bs.cpu().numpy(), bf[..., z0:z1].cpu().numpy(), f"zslab back {name} slab {r}") <= 1e-6
    assert rel_l2(ysum.cpu().numpy(), yf.cpu().numpy(), f"zslab fwd sum {name}") <= 1e-6


def test_zslab_path_single_rank(ct, O):
    """The z-slab exchange path (partial sinograms all-reduced, residual on every ray,
    back-projection onto the slab, xi all-reduced) on a 1-rank communicator: D_L equals the
    plain D_L and OS-LALM (26 neighbours, BB on) matches the fp64 oracle."""
    g = geoms_small()["helical_c4"]
    base = I.config("c4")
    ell = [(0.0, 0.0, 0.0, 4.0, 3.5, 2.5, 0.0, 0.02), (1.0, -0.5, 0.3, 1.2, 0.8, 0.9, 0.4, 0.01)]
    d = I.noisy_data(g, ell, 1e5, 0.0, 79)
    m0 = torch.ones((g["ny"], g["nx"], g["nz"]), dtype=torch.uint8)
    plain = ct.Geometry(g)
    dl0, _ = plain.sqs_denom(d["w"].cuda(), m0.cuda())
    geo = ct.Geometry(g)
    geo.comm_init(0, 1, ct.ct_comm_get_unique_id(), zslab=True)
    dl, S = geo.sqs_denom(d["w"].cuda(), m0.cuda())
    assert rel_l2(dl.cpu().numpy(), dl0.cpu().numpy(), "zslab D_L") <= 1e-6
    sol = ct.OSLALM(geo, 4, beta=base.beta, delta=base.delta, nbr=26, bb=True)
    sol.set_data(d["y"].cuda(), d["w"].cuda(), dl, S)
    x = torch.zeros(geo.img_shape, device="cuda")
    log = np.array(sol.run(x, 6, log=True))
    dlo, So = O.sqs_denom(g, I.to_oracle_sino(d["w"]), I.to_oracle_image(m0).astype(np.uint8))
    xo, logo, _, _ = O.oslalm_run(g, I.to_oracle_sino(d["y"]), I.to_oracle_sino(d["w"]), dlo, So,
                                  np.zeros(O.img_shape(g)), M=4, beta=base.beta, delta=base.delta, nbr=26, n_iter=6,
                                  bb=True)
    xg = I.to_oracle_image(x.cpu().numpy())
    rms = math.sqrt(((xg - xo)[So > 0] ** 2).mean()) / I.HU
    MARGINS.append({"case": "z-slab path helical_c4 (1 rank, BB) vs oracle", "rms_HU": rms})
    assert rms <= 0.5, rms
    assert np.array_equal(log[:, 2], logo[:, 2])
    with pytest.raises(ct.CTError, match="EUNSUPPORTED"):
        ct.OSLALM(geo, 4, beta=base.beta, delta=base.delta, nbr=26, inner="fista", n_inner=2)


def test_fwd_more_views_than_grid_rows(ct, O):
    """A 3D forward projection of > 65535 views (the CUDA grid's y limit) is launched in view
    chunks: every view matches the oracle (tiny image and detector, 70000-view helix)."""
    g = GU.geom("cone_helical", nx=4, nz=6, dx=0.9766, dz=0.625, ns=6, ds=1.0239, nt=4, dt=1.0964, na=70000,
                turns=20.0, pitch=1.0)
    geo = ct.Geometry(g)
    x = rand_image(g, 5, geo.img_shape)
    yg = geo.fwd(torch.from_numpy(x).cuda()).cpu().numpy()
    yo = O.fwd(g, I.to_oracle_image(x), 0, 1, g["na"])
    assert rel_l2(I.to_oracle_sino(yg), yo, "fwd 70000 views") <= 1e-4
    tail = (65530, 1, 12)   # a view list straddling the chunk boundary
    yt = geo.fwd(torch.from_numpy(x).cuda(), tail).cpu().numpy()
    assert np.array_equal(yt, yg[65530:65542])


DEGENERATE = {
    # one slice, one detector row: the cone path reduces to a single-row fan
    "axial_nz1_nt1": GU.geom("cone_axial", nx=9, nz=1, dx=1.2, dz=1.0, ns=17, ds=1.7, nt=1, dt=1.1, na=14),
    # one slice seen by many rows (kz small) and a thick-slice stack (one row per slice pair)
    "axial_nz1_nt64": GU.geom("cone_axial", nx=7, nz=1, dx=1.0, dz=3.0, ns=13, ds=1.4, nt=64, dt=0.3, na=10),
    "axial_nz3_nt2": GU.geom("cone_axial", nx=8, ny=5, nz=3, dx=1.0, dz=0.4, ns=11, ds=1.6, nt=2, dt=2.0, na=12),
    # helical with two slices and two rows; one-channel detector
    "helical_nz2_nt2": GU.geom("cone_helical", nx=6, nz=2, dx=1.0, dz=0.7, ns=9, ds=1.5, nt=2, dt=1.0, na=40,
                               turns=2.0, pitch=1.0),
    "fan_ns1": GU.geom("fan2d", nx=6, dx=0.8, ns=1, ds=4.0, na=25),
    "axial_ns1": GU.geom("cone_axial", nx=5, nz=4, dx=0.8, dz=0.8, ns=1, ds=9.0, nt=3, dt=1.0, na=16),
}


@pytest.mark.parametrize("name", list(DEGENERATE))
def test_degenerate_shapes(ct, O, name):
    """Single slice / row / channel geometries and tiny volumes: forward and back match the
    oracle and stay adjoint (every kernel's tile is almost entirely ragged)."""
    g = DEGENERATE[name]
    geo = ct.Geometry(g)
    x = rand_image(g, 11, geo.img_shape)
    yg = geo.fwd(torch.from_numpy(x).cuda()).cpu().numpy()
    yo = O.fwd(g, I.to_oracle_image(x), 0, 1, g["na"])
    assert np.isfinite(yg).all()
    assert rel_l2(I.to_oracle_sino(yg), yo, f"fwd degenerate {name}") <= 1e-4
    p = np.random.default_rng(12).random(yg.shape).astype(np.float32)
    bg = geo.back(torch.from_numpy(p).cuda()).cpu().numpy()
    bo = O.back(g, I.to_oracle_sino(p), 0, 1, g["na"])
    assert rel_l2(I.to_oracle_image(bg), bo, f"back degenerate {name}") <= 1e-4


def test_fan_pixel_much_finer_than_channel_is_rejected(ct):
    """The fan forward tile kernel needs consecutive pixels >= 1/8 channel apart (lane-parity
    buffers): a finer grid is refused at create with CT_EUNSUPPORTED, not run."""
    with pytest.raises(ct.CTError, match="CT_EUNSUPPORTED"):
        ct.Geometry(GU.geom("fan2d", nx=6, dx=0.8, ns=1, ds=9.0, na=25))


def test_binding_rejects_short_buffers(ct):
    """The C ABI takes bare pointers; the binding checks every buffer's size against the
    geometry before the call (no out-of-bounds device writes from a short tensor)."""
    g = geoms_small()["axial_c3"]
    geo = ct.Geometry(g)
    x = torch.zeros(geo.img_shape, device="cuda")
    y = torch.zeros(geo.sino_shape(4), device="cuda")
    ct.ct_fwd_proj(geo.h, (0, 1, 4), x, y)
    with pytest.raises(ct.CTError, match="elements"):
        ct.ct_fwd_proj(geo.h, (0, 1, 5), x, y)            # 5 views into a 4-view sinogram
    with pytest.raises(ct.CTError, match="elements"):
        ct.ct_back_proj(geo.h, (0, 1, 4), y, x[:-1])     # image one row short
    w = torch.ones(geo.sino_shape(g["na"] - 1), device="cuda")
    mask = torch.ones(geo.img_shape, dtype=torch.uint8, device="cuda")
    scratch = torch.empty(ct.ct_sqs_denom_scratch_bytes(geo.h), dtype=torch.uint8, device="cuda")
    with pytest.raises(ct.CTError, match="elements"):
        ct.ct_sqs_denom(geo.h, w, mask, x, scratch)       # weights one view short
