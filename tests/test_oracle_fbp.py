"""Pins for the oracle's FBP / FDK initial image (NEXT-4; "initialized with a
standard filtered back-projection (FBP)"; reading B-FBP in DESIGN.md).

FBP inverts the Radon transform, so on exact (analytic, noise-free) line integrals of a
uniform disk / ellipsoid it must return the density inside the object and ~0 outside
(closed form), and be linear in the data.  Helical scans (P:573, P:586, P:1495 start from an
FBP image; reading B-FBP-H): the view-normalised helical FDK must reconstruct a thin ellipsoid
at its height (closed-form density inside, ~0 above and below) and coincide with the
circular-orbit FDK as the pitch goes to 0."""
import numpy as np
import pytest

import oracle as O
from paper_1402_4381_b200 import inputs as I
from tests import geomutil as GU


def _grid(g):
    xs = (np.arange(g["nx"]) - (g["nx"] - 1) / 2) * g["dx"] + g.get("offx", 0.0)
    ys = (np.arange(g["ny"]) - (g["ny"] - 1) / 2) * g["dy"] + g.get("offy", 0.0)
    return np.meshgrid(xs, ys)      # [iy][ix]


def test_fbp_fan_disk_c2_geometry():
    """Uniform disk (R = 100 mm, mu = 0.02/mm, centre (20, -10) mm) in c2 geometry, exact
    projections: interior mean within 0.1 %, interior RMS <= 0.5 %, and near-zero outside."""
    g = I.config("c2").geom
    mu = 0.02
    p = I.line_integrals(g, [(20.0, -10.0, 0.0, 100.0, 100.0, float("inf"), 0.0, mu)], list(range(g["na"])))
    x = O.fbp(g, I.to_oracle_sino(p.numpy()))[0]
    X, Y = _grid(g)
    r = np.hypot(X - 20.0, Y + 10.0)
    inner = x[r < 80.0]
    assert abs(inner.mean() / mu - 1) <= 1e-3
    assert np.sqrt(((inner - mu) ** 2).mean()) / mu <= 5e-3
    outer = x[(r > 130.0) & (np.hypot(X, Y) < I.fov_radius(g) - 5.0)]
    # zero on average outside; the Ram-Lak filter + linear interpolation leave a fine
    # zero-mean streak texture at ~1-3 % of mu
    assert abs(outer.mean()) <= 1e-3 * mu and np.sqrt((outer ** 2).mean()) <= 0.03 * mu


def test_fdk_axial_ellipsoid_central_slices():
    """Axial cone beam (c3 detector and orbit, coarser image): a uniform ellipsoid thin in z
    is reconstructed to within 1 % in its central slices (cone angle ~2 degrees)."""
    g = GU.geom("cone_axial", nx=96, dx=3.0, nz=16, dz=0.625, ns=888, ds=1.0239, nt=64, dt=1.0964, na=492)
    mu = 0.02
    p = I.line_integrals(g, [(0.0, 0.0, 0.0, 90.0, 90.0, 4.0, 0.0, mu)], list(range(g["na"])))
    x = O.fbp(g, I.to_oracle_sino(p.numpy()))      # [iz][iy][ix]
    X, Y = _grid(g)
    zs = (np.arange(g["nz"]) - (g["nz"] - 1) / 2) * g["dz"]
    for iz in np.nonzero(np.abs(zs) < 1.5)[0]:
        inner = x[iz][np.hypot(X, Y) < 70.0]
        assert abs(inner.mean() / mu - 1) <= 1e-2, (iz, inner.mean())


def test_fbp_is_linear_and_rejects_partial_orbits():
    rng = np.random.default_rng(3)
    for g in (GU.small_geoms()["fan_c2"], GU.small_geoms()["helical_c4"]):
        p1, p2 = rng.random(O.sino_shape(g, g["na"])), rng.random(O.sino_shape(g, g["na"]))
        lhs = O.fbp(g, 2.0 * p1 - 0.5 * p2)
        rhs = 2.0 * O.fbp(g, p1) - 0.5 * O.fbp(g, p2)
        assert np.abs(lhs - rhs).max() <= 1e-12 * np.abs(rhs).max()
    half = GU.geom("cone_axial", nx=12, nz=6, dx=0.9766, dz=0.625, ns=24, ds=1.0239, nt=8, dt=1.0964, na=24, turns=0.5)
    with pytest.raises(ValueError):
        O.fbp(half, np.zeros(O.sino_shape(half, 24)))


def _helical_fbp_geom(pitch, turns, na_per_turn=984):
    return GU.geom("cone_helical", nx=64, dx=3.0, nz=24, dz=1.25, ns=888, ds=1.0239, nt=64, dt=1.0964,
                   na=int(round(turns * na_per_turn)), turns=turns, pitch=pitch)


def test_fbp_helical_thin_ellipsoid_height():
    """Helical scan with the c5 detector and pitch (0.5, 20 mm feed) over 3 turns: a uniform
    ellipsoid 16 mm thick centred at z = +3 mm is reconstructed at its height -- mean within 2 %
    of mu well inside it, ~0 (< 5 % of mu) in the slices more than 6 mm above or below it.  A
    wrong sign or offset of z_s in the back-projection moves or smears the slab."""
    g = _helical_fbp_geom(0.5, 3.0)
    mu, cz = 0.02, 3.0
    p = I.line_integrals(g, [(0.0, 0.0, cz, 70.0, 70.0, 8.0, 0.0, mu)], list(range(g["na"])))
    x = O.fbp(g, I.to_oracle_sino(p.numpy()))      # [iz][iy][ix]
    X, Y = _grid(g)
    zs = (np.arange(g["nz"]) - (g["nz"] - 1) / 2) * g["dz"]
    inside = np.hypot(X, Y) < 45.0
    for iz in range(g["nz"]):
        m = x[iz][inside].mean()
        if abs(zs[iz] - cz) < 4.0:
            assert abs(m / mu - 1) <= 2e-2, (zs[iz], m / mu)
        elif abs(zs[iz] - cz) > 14.0:
            assert abs(m) <= 5e-2 * mu, (zs[iz], m / mu)


def test_fbp_helical_small_pitch_equals_circular_fdk():
    """Pitch -> 0: one turn with pitch 1e-6 (source heights within +-2e-5 mm) is the circular
    orbit; the view-normalised helical FDK then equals the circular-orbit FDK (every view sees
    the central slices, so the normalisation is 1/na) -- on a random sinogram, to 1e-4 of the
    signal (the difference scales with the pitch: 1.7e-3 relative at pitch 1e-3)."""
    gh = GU.geom("cone_helical", nx=32, dx=6.0, nz=24, dz=1.25, ns=888, ds=1.0239, nt=64, dt=1.0964, na=492,
                 turns=1.0, pitch=1e-6)
    ga = dict(gh, kind="cone_axial", pitch=0.0)
    p = np.random.default_rng(0).random(O.sino_shape(ga, ga["na"]))
    xh, xa = O.fbp(gh, p), O.fbp(ga, p)
    c = slice(8, 16)   # central slices (|z| < 5 mm): seen by every view
    assert np.abs(xh[c] - xa[c]).max() <= 1e-4 * np.abs(xa[c]).max()
