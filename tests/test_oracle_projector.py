"""Pins for the oracle's SF-TR projector ("A is the
system matrix of a CT scan").  Each test checks the oracle against something
other than itself: the adjoint identity, the exact parallel-beam limit,
closed-form chords, brute-force ray–box integrals, a textbook Siddon projector,
and symmetry invariants.
"""
import math

import numpy as np
import pytest

import oracle as O
from tests import geomutil as GU


@pytest.mark.parametrize("name", list(GU.small_geoms().keys()))
def test_adjoint_identity(name):
    """<Ax, y> = <x, A'y> for random positive x, y (matched pair, SURVEY pins table)."""
    g = GU.small_geoms()[name]
    rng = np.random.default_rng(7)
    x = rng.random(O.img_shape(g))
    y = rng.random(O.sino_shape(g, g["na"]))
    lhs = float((O.fwd(g, x) * y).sum())
    rhs = float((x * O.back(g, y)).sum())
    assert lhs > 0
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)
    # a subset (interleaved views m mod M) is also an adjoint pair
    ys = rng.random(O.sino_shape(g, O.nviews(g, 1, 3)))
    lhs = float((O.fwd(g, x, 1, 3) * ys).sum())
    rhs = float((x * O.back(g, ys, 1, 3)).sum())
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)


def _exact_parallel_bin(g, v, ix_off, iy_off, c):
    """Exact bin-averaged parallel-beam projection of one unit pixel (slab clipping).

    In the limit dso -> inf with dsd = 2 dso, detector arc position s corresponds to the
    object-space offset u = s dso / dsd along e_perp; the bin average of the chord length
    over [u_lo, u_hi] is integrated exactly (chord is piecewise linear in u between the
    projected corners)."""
    b = GU.view_angle(g, v)
    ec = np.array([math.sin(b), -math.cos(b)])
    ep = np.array([math.cos(b), math.sin(b)])
    m = g["dso"] / g["dsd"]
    s = GU.chan_s(g, c)
    ulo, uhi = (s - g["ds"] / 2) * m, (s + g["ds"] / 2) * m
    half = g["dx"] / 2
    corners = [np.array([ix_off + a, iy_off + bb]) for a in (-half, half) for bb in (-half, half)]
    bps = sorted([float(p @ ep) for p in corners] + [ulo, uhi])
    pts = [u for u in bps if ulo <= u <= uhi]

    def chord(u):
        S = u * ep - 1e3 * ec
        return GU.box_chord(S, ec, np.array([ix_off - half, iy_off - half]), np.array([ix_off + half, iy_off + half]))

    tot = 0.0
    for a, bb in zip(pts[:-1], pts[1:]):
        if bb > a:  # chord is linear on each open piece: the midpoint rule is exact
            tot += chord(0.5 * (a + bb)) * (bb - a)
    return tot / (uhi - ulo)


def _parallel_limit_error(dso):
    g = GU.geom("fan2d", nx=1, dx=1.0, ns=16, ds=0.3, na=24, dso=dso, dsd=2 * dso, offx=0.37, offy=-0.23)
    p = O.fwd(g, np.ones((1, 1, 1)))[:, 0, :]
    ref = np.array([[_exact_parallel_bin(g, v, 0.37, -0.23, c) for c in range(g["ns"])] for v in range(g["na"])])
    return np.abs(p - ref).max() / ref.max()


def test_parallel_beam_limit():
    """SF-TR becomes the exact pixel projection as dso -> inf; error first order in dx/dso (V1)."""
    # max error / max value, times dso / dx: must be a constant (first order) and O(1),
    # i.e. the SF-TR weights converge to the exact pixel projection as 1/dso.
    k = [_parallel_limit_error(d) * d for d in (1e4, 1e6, 1e8)]
    assert k[2] <= 2.0
    assert abs(k[0] - k[2]) <= 1e-3 * k[2] and abs(k[1] - k[2]) <= 1e-4 * k[2]


def _disk_case(nx, dx, views):
    g = GU.geom("fan2d", nx=nx, dx=dx, ns=888, ds=1.0239, na=984)
    R, mu = 100.0, 0.02
    out = []
    for (cx, cy) in ((0.0, 0.0), (60.0, -20.0)):
        # area-fraction voxelisation with 8x8 supersampling
        o = (np.arange(8) + 0.5) / 8 - 0.5
        xc = (np.arange(nx) - (nx - 1) / 2.0) * dx
        X = xc[None, :, None, None] + o[None, None, None, :] * dx
        Y = xc[:, None, None, None] + o[None, None, :, None] * dx
        img = (((X - cx) ** 2 + (Y - cy) ** 2) <= R * R).mean(axis=(2, 3)) * mu
        for v in views:
            p = O.fwd(g, img[None], v, 1, 1)[0, 0]
            S, _ = GU.ray(g, v, 0.0, 0.0)
            d = []
            for c in range(g["ns"]):
                S, u = GU.ray(g, v, GU.chan_s(g, c), 0.0)
                w = np.array([cx, cy]) - S[:2]
                d.append(abs(w[0] * u[1] - w[1] * u[0]))
            d = np.array(d)
            sel = d < R - 2 * dx
            ref = mu * 2 * np.sqrt(R * R - d[sel] ** 2)
            out.append((p[sel] - ref) / ref)
    e = np.concatenate(out)
    return math.sqrt((e * e).mean()), np.abs(e).max()


def test_disk_chords_c2_geometry():
    """Uniform disk R=100 mm: SF projection vs closed-form chord 2 mu sqrt(R^2-d^2) (V3)."""
    views = [0, 123, 246, 500, 777]
    rms1, mx1 = _disk_case(512, 0.9766, views)
    rms2, mx2 = _disk_case(1024, 0.9766 / 2, views)
    assert rms1 <= 5e-3 and mx1 <= 3e-2
    assert rms2 <= rms1 / 2


def test_ellipsoid_chords_c3_geometry():
    """Uniform ellipsoid, cone-beam axial c3 geometry: SF projection of the 4x4x4-supersampled
    voxelisation vs the closed-form ray–ellipsoid chord, on rays whose closest approach (in
    the ellipsoid's unit-sphere coordinates) stays 2 voxels inside the surface."""
    g = GU.geom("cone_axial", nx=160, nz=64, dx=0.9766, dz=0.625, ns=888, ds=1.0239, nt=64, dt=1.0964, na=984)
    a = np.array([60.0, 40.0, 15.0]); c0 = np.array([8.0, -5.0, 1.0]); mu = 0.02
    nx, nz = g["nx"], g["nz"]
    o = (np.arange(4) + 0.5) / 4 - 0.5
    xc = (np.arange(nx) - (nx - 1) / 2.0) * g["dx"]
    zc = (np.arange(nz) - (nz - 1) / 2.0) * g["dz"]
    img = np.zeros((nz, nx, nx))
    for oz in o:
        for oy in o:
            for ox in o:
                Z = (zc[:, None, None] + oz * g["dz"] - c0[2]) / a[2]
                Y = (xc[None, :, None] + oy * g["dx"] - c0[1]) / a[1]
                X = (xc[None, None, :] + ox * g["dx"] - c0[0]) / a[0]
                img += (X * X + Y * Y + Z * Z) <= 1
    img *= mu / 64
    margin = 1.0 - 2 * max(g["dx"] / a[0], g["dy"] / a[1], g["dz"] / a[2])
    errs = []
    for v in (0, 200, 411):
        p = O.fwd(g, img, v, 1, 1)[0]
        for r in range(g["nt"]):
            for c in range(0, g["ns"], 3):
                S, u = GU.ray(g, v, GU.chan_s(g, c), GU.row_t(g, r))
                q0 = (S - c0) / a; q1 = u / a
                A = q1 @ q1; B = 2 * q0 @ q1; C = q0 @ q0 - 1
                closest = math.sqrt(max(0.0, C + 1 - B * B / (4 * A)))
                if closest > margin:
                    continue
                chord = math.sqrt(B * B - 4 * A * C) / A
                errs.append((p[r, c] - mu * chord) / (mu * chord))
    e = np.array(errs)
    assert len(e) > 500
    assert math.sqrt((e * e).mean()) <= 5e-3
    assert np.abs(e).max() <= 3e-2


def test_single_voxel_bruteforce_3d():
    """SF-TR weights of one voxel vs brute-force bin-averaged ray–box chords, 48x48 sub-rays per cell (V4)."""
    g = GU.geom("cone_axial", nx=512, nz=64, dx=0.9766, dz=0.625, ns=888, ds=1.0239, nt=64, dt=1.0964, na=984)
    rng = np.random.default_rng(3)
    for trial in range(6):
        ix, iy, iz = rng.integers(100, 412), rng.integers(100, 412), rng.integers(8, 56)
        v = int(rng.integers(0, g["na"]))
        xc = (ix - (g["nx"] - 1) / 2.0) * g["dx"]; yc = (iy - (g["ny"] - 1) / 2.0) * g["dy"]
        zc = (iz - (g["nz"] - 1) / 2.0) * g["dz"]
        lo = np.array([xc - g["dx"] / 2, yc - g["dy"] / 2, zc - g["dz"] / 2])
        hi = lo + np.array([g["dx"], g["dy"], g["dz"]])
        # candidate cells: the SF footprint plus a 2-cell margin
        tr = O.transaxial(g, v, ix, iy)
        base = -(g["ns"] - 1) / 2.0
        c_lo = int(math.floor(tr[0] / g["ds"] - base - 0.5)) - 2
        c_hi = int(math.floor(tr[3] / g["ds"] - base + 0.5)) + 2
        mag = g["dsd"] / tr[5]
        tl, th = (zc - g["dz"] / 2) * mag, (zc + g["dz"] / 2) * mag
        tb = -(g["nt"] - 1) / 2.0
        r_lo = int(math.floor(tl / g["dt"] - tb - 0.5)) - 2
        r_hi = int(math.floor(th / g["dt"] - tb + 0.5)) + 2
        sf, bf = [], []
        o = (np.arange(48) + 0.5) / 48 - 0.5
        for r in range(r_lo, r_hi + 1):
            for c in range(c_lo, c_hi + 1):
                sf.append(O.weight(g, v, ix, iy, iz, r, c))
                Ss, Us = [], []
                for os_ in o:
                    for ot in o:
                        S, u = GU.ray(g, v, GU.chan_s(g, c) + os_ * g["ds"], GU.row_t(g, r) + ot * g["dt"])
                        Ss.append(S); Us.append(u)
                bf.append(GU.box_chords_vec(np.array(Ss), np.array(Us), lo, hi).mean())
        sf, bf = np.array(sf), np.array(bf)
        assert abs(sf.sum() - bf.sum()) <= 5e-3 * bf.sum()
        assert np.linalg.norm(sf - bf) <= 2e-2 * np.linalg.norm(bf)


def _siddon_case(g, img, views, nsub=32):
    """Exact bin-averaged projection of the pixel-basis image, nsub sub-rays per channel."""
    out = np.zeros((len(views), g["ns"]))
    flat = img.reshape(-1)
    o = (np.arange(nsub) + 0.5) / nsub - 0.5
    for k, v in enumerate(views):
        S_list, U_list, owner = [], [], []
        for c in range(g["ns"]):
            for os_ in o:
                S, u = GU.ray(g, v, GU.chan_s(g, c) + os_ * g["ds"], 0.0)
                S_list.append(S[:2]); U_list.append(u[:2] / np.linalg.norm(u[:2])); owner.append(c)
        rr, cc, ll = GU.pixel_grid_chords(np.array(S_list), np.array(U_list), g)
        ray_sum = np.bincount(rr, weights=ll * flat[cc], minlength=len(S_list))
        out[k] = np.bincount(np.array(owner), weights=ray_sum, minlength=g["ns"]) / nsub
    return out


@pytest.mark.parametrize("case", ["c1", "c2res"])
def test_sf_vs_exact_pixel_projection(case):
    """SF vs exact (Siddon, 32 sub-rays/channel) projection of the same pixel image (V8)."""
    if case == "c1":
        g = GU.geom("fan2d", nx=64, dx=4.0, ns=96, ds=8.1912, na=120)
        views = list(range(0, 120, 4))
        tol = 1e-3
    else:
        g = GU.geom("fan2d", nx=96, dx=0.9766, ns=200, ds=1.0239, na=984)
        views = [0, 41, 100, 123, 300, 501, 700, 999 % 984]
        tol = 1e-4
    n = g["nx"]
    xc = (np.arange(n) - (n - 1) / 2.0) * g["dx"]
    X, Y = np.meshgrid(xc, xc, indexing="xy")
    R = n * g["dx"] / 2
    img = 0.02 * ((X / (0.8 * R)) ** 2 + (Y / (0.6 * R)) ** 2 <= 1) \
        + 0.01 * (((X - 0.2 * R) / (0.2 * R)) ** 2 + ((Y + 0.1 * R) / (0.3 * R)) ** 2 <= 1)
    ref = _siddon_case(g, img, views)
    sf = np.stack([O.fwd(g, img[None], v, 1, 1)[0, 0] for v in views])
    sel = ref >= 0.05 * ref.max()
    e = (sf[sel] - ref[sel]) / ref[sel]
    assert math.sqrt((e * e).mean()) <= tol


def test_mass_and_nonnegativity():
    """sum_c a_ij ds = l_phi (t3 + t2 - t1 - t0)/2 when the footprint is on the detector; a_ij >= 0."""
    g = GU.small_geoms()["fan_c2"]
    for v in (0, 5, 9, 17):
        for (ix, iy) in ((3, 4), (12, 10), (20, 2)):
            x = np.zeros(O.img_shape(g)); x[0, iy, ix] = 1.0
            p = O.fwd(g, x, v, 1, 1)[0, 0]
            assert (p >= 0).all()
            tr = O.transaxial(g, v, ix, iy)
            assert abs(p.sum() * g["ds"] - tr[4] * (tr[3] + tr[2] - tr[1] - tr[0]) / 2) <= 1e-12 * p.sum() * g["ds"]


def test_reflection_invariant():
    """proj(flip_x(x), -beta)[c] = proj(x, beta)[ns-1-c]  (-beta_v = beta_{na-v})."""
    g = GU.geom("fan2d", nx=14, ny=10, dx=3.0, ns=30, ds=4.0, na=36)
    rng = np.random.default_rng(5)
    x = rng.random((1, 10, 14))
    p = O.fwd(g, x)[:, 0, :]
    pf = O.fwd(g, x[:, :, ::-1].copy())[:, 0, :]
    for v in range(g["na"]):
        vm = (g["na"] - v) % g["na"]
        assert np.abs(pf[vm] - p[v, ::-1]).max() <= 1e-12 * p.max()


def test_rotation_invariant():
    """proj(rot90(x), beta + pi/2) = proj(x, beta): square grid, na divisible by 4."""
    g = GU.geom("fan2d", nx=12, dx=3.0, ns=30, ds=4.0, na=40)
    rng = np.random.default_rng(6)
    x = rng.random((12, 12))
    # x'(p) = x(R_{-90} p):  x'[iy][ix] = x[n-1-ix][iy]
    n = 12
    xr = np.empty_like(x)
    for iy in range(n):
        for ix in range(n):
            xr[iy, ix] = x[n - 1 - ix, iy]
    p = O.fwd(g, x[None])[:, 0, :]
    pr = O.fwd(g, xr[None])[:, 0, :]
    q = g["na"] // 4
    for v in range(g["na"]):
        assert np.abs(pr[(v + q) % g["na"]] - p[v]).max() <= 1e-12 * p.max()


def test_fan_beta_plus_pi_is_not_a_mirror():
    """beta -> beta + pi is NOT a channel mirror in fan beam (conjugate rays are at beta+pi+2gamma)."""
    g = GU.geom("fan2d", nx=12, dx=3.0, ns=30, ds=4.0, na=40)
    rng = np.random.default_rng(8)
    x = rng.random((1, 12, 12))
    p = O.fwd(g, x)[:, 0, :]
    assert np.abs(p[20] - p[0, ::-1]).max() > 1e-3 * p.max()


def test_view_geometry_pins():
    """O1 pins: FOV radii (c1 217.8 mm, c2 249.4 mm) and helical feed 20.0 mm/turn (c4, c5)."""
    from paper_1402_4381_b200 import inputs as I
    assert abs(I.fov_radius(I.config("c2").geom) - 249.4) < 0.05
    assert abs(I.fov_radius(I.config("c1").geom) - 217.8) < 0.05
    for c in ("c4", "c5"):
        g = I.config(c).geom
        per_turn = g["na"] / (g["orbit_deg"] / 360.0)
        feed = O.source_z(g, int(per_turn)) - O.source_z(g, 0)
        assert abs(feed - 20.0) < 0.01
        assert abs(O.source_z(g, 0) + O.source_z(g, g["na"] - 1)) < 1e-9   # centred helix (G17)


@pytest.mark.parametrize("name", ["fan_c2", "axial_c3", "helical_c4"])
def test_count_vv_is_support_of_A(name):
    """U = #(view, voxel in S) pairs with a non-empty footprint, which must equal
    the number of (view, voxel) pairs whose column of A_view has a nonzero entry."""
    g = GU.small_geoms()[name]
    shape = O.img_shape(g)
    rng = np.random.default_rng(9)
    mask = (rng.random(shape) > 0.3).astype(np.uint8)
    n = int(np.prod(shape))
    ref = 0
    for j in range(n):
        if not mask.reshape(-1)[j]:
            continue
        e = np.zeros(n); e[j] = 1.0
        p = O.fwd(g, e.reshape(shape))
        ref += int((p.reshape(g["na"], -1) > 0).any(axis=1).sum())
    assert O.count_vv(g, mask) == ref
