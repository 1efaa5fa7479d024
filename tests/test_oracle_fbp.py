"""Pins for the oracle's FBP / FDK initial image (NEXT-4; "initialized with a
standard filtered back-projection (FBP)"; reading B-FBP in DESIGN.md).

FBP inverts the Radon transform, so on exact (analytic, noise-free) line integrals of a
uniform disk / ellipsoid it must return the density inside the object and ~0 outside
(closed form), and be linear in the data.  Helical scans are not supported (no FDK over a
helix here)."""
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


def test_fbp_is_linear_and_rejects_helical():
    g = GU.small_geoms()["fan_c2"]
    rng = np.random.default_rng(3)
    p1, p2 = rng.random(O.sino_shape(g, g["na"])), rng.random(O.sino_shape(g, g["na"]))
    lhs = O.fbp(g, 2.0 * p1 - 0.5 * p2)
    rhs = 2.0 * O.fbp(g, p1) - 0.5 * O.fbp(g, p2)
    assert np.abs(lhs - rhs).max() <= 1e-12 * np.abs(rhs).max()
    with pytest.raises(ValueError):
        O.fbp(GU.small_geoms()["helical_c4"], np.zeros(O.sino_shape(GU.small_geoms()["helical_c4"], 48)))
