"""Pins for the oracle's HELICAL branch (SURVEY §8(c) O1/O2 with z_s != 0; reading G17).

The helical scans of the paper ("helical shoulder scan ... pitch 0.5",
P:1495 "helical ... pitch 1.0") make the source height z_s(v) enter the axial footprint
(the rect [t-, t+] = (z_j -+ dz/2 - z_s) dsd / rho_h) and the amplitude
l_theta = sqrt(1 + ((z_j - z_s) / rho_h)^2) of `oracle.c::axial_rect`.  The axial pins
(z_s = 0) cannot see a wrong sign or offset of z_s there, so these tests compare the
oracle at views with |z_s| >= 30 mm against things it does not compute itself:

* closed-form ray-ellipsoid chords (c4 and c5 geometries; the reference rays come from
  `tests/geomutil.py`, which derives z_s from the scan parameters independently);
* brute-force bin-averaged ray-box chords of a single voxel (c5 geometry), and, at a
  steep cone angle where l_theta is several percent, the footprint mass.

Each test also evaluates the reference with a plausible mistake injected on the
reference side (z_s sign flipped, z_s offset by half a slice, l_theta dropped) and
checks that the mistake would be caught by the same tolerance.
"""
import math

import numpy as np
import pytest

import oracle as O
from tests import geomutil as GU


def _helical(cfg):
    if cfg == "c4":   # BASELINE configs[3]: 888 x 32, 2952 views / 3 turns, pitch 1.0
        return dict(nt=32, na=2952, turns=3.0, pitch=1.0)
    return dict(nt=64, na=6888, turns=7.0, pitch=0.5)   # configs[4]: 888 x 64, 6888 views / 7 turns, pitch 0.5


def _view_at(g, zs):
    """Nearest view whose source height is zs (independent formula, geomutil.source_z)."""
    per_turn = g["na"] / (g["orbit_deg"] / 360.0)
    h = g["pitch"] * g["nt"] * g["dt"] * g["dso"] / g["dsd"]
    return int(round(zs * per_turn / h + (g["na"] - 1) / 2.0))


def _voxelise_ellipsoid(g, c0, a, mu, ss=4):
    nx, nz = g["nx"], g["nz"]
    o = (np.arange(ss) + 0.5) / ss - 0.5
    xc = (np.arange(nx) - (nx - 1) / 2.0) * g["dx"] + g["offx"]
    yc = (np.arange(nx) - (nx - 1) / 2.0) * g["dy"] + g["offy"]
    zc = (np.arange(nz) - (nz - 1) / 2.0) * g["dz"] + g["offz"]
    img = np.zeros((nz, nx, nx))
    for oz in o:
        Z = ((zc[:, None, None] + oz * g["dz"] - c0[2]) / a[2]) ** 2
        for oy in o:
            Y = ((yc[None, :, None] + oy * g["dy"] - c0[1]) / a[1]) ** 2
            for ox in o:
                X = ((xc[None, None, :] + ox * g["dx"] - c0[0]) / a[0]) ** 2
                img += (X + Y + Z) <= 1
    return img * (mu / ss ** 3)


def _chord_errors(g, p, v, c0, a, mu, dzs=0.0, flip=False):
    """Relative errors of the projection p[row][channel] of view v against the closed-form
    chords, on rays that stay 2 voxels inside the surface.  dzs / flip perturb the
    REFERENCE source height (mutation check)."""
    margin = 1.0 - 2 * max(g["dx"] / a[0], g["dy"] / a[1], g["dz"] / a[2])
    errs = []
    for r in range(g["nt"]):
        for c in range(0, g["ns"], 2):
            S, u = GU.ray(g, v, GU.chan_s(g, c), GU.row_t(g, r))
            S = S.copy()
            if flip:
                S[2] = -S[2]
            S[2] += dzs
            q0 = (S - c0) / a
            q1 = u / a
            A = q1 @ q1; B = 2 * q0 @ q1; C = q0 @ q0 - 1
            closest = math.sqrt(max(0.0, C + 1 - B * B / (4 * A)))
            if closest > margin:
                continue
            chord = math.sqrt(B * B - 4 * A * C) / A
            errs.append((p[r, c] - mu * chord) / (mu * chord))
    return np.array(errs)


@pytest.mark.parametrize("cfg", ["c4", "c5"])
def test_ellipsoid_chords_helical(cfg):
    """Uniform ellipsoids centred at z = +-36 mm, projected at helical views with the source
    at |z_s| in [30, 42] mm (several turns from the helix centre): SF projection of the
    4x4x4-supersampled voxelisation vs the closed-form chords (RMS <= 0.5 %, max <= 3 %, the
    tolerances of the axial pin).  Catches: a sign error of z_s in the axial rect (the
    ellipsoid would be projected from the mirrored height), and an offset of z_s by half a
    slice (0.3125 mm)."""
    h = _helical(cfg)
    for zc in (36.0, -36.0):
        g = GU.geom("cone_helical", nx=128, nz=64, dx=0.9766, dz=0.625, ns=888, ds=1.0239, nt=h["nt"], dt=1.0964,
                    na=h["na"], turns=h["turns"], pitch=h["pitch"], offz=zc)
        c0 = np.array([6.0, -4.0, zc + 1.0]); a = np.array([45.0, 35.0, 14.0]); mu = 0.02
        img = _voxelise_ellipsoid(g, c0, a, mu)
        all_e, flip_e, off_e = [], [], []
        for dz_src in (-6.0, 0.0, 6.0):
            v = _view_at(g, zc + dz_src)
            zs = O.source_z(g, v)
            assert abs(zs) >= 29.0 and abs(zs - GU.source_z(g, v)) < 1e-9
            p = O.fwd(g, img, v, 1, 1)[0]
            all_e.append(_chord_errors(g, p, v, c0, a, mu))
            flip_e.append(_chord_errors(g, p, v, c0, a, mu, flip=True))
            off_e.append(_chord_errors(g, p, v, c0, a, mu, dzs=0.5 * g["dz"]))
        e = np.concatenate(all_e)
        assert len(e) > 500
        rms = math.sqrt((e * e).mean())
        assert rms <= 5e-3 and np.abs(e).max() <= 3e-2, (cfg, zc, rms, np.abs(e).max())
        # the same tolerance rejects the mirrored and the half-slice-shifted source height
        ef = np.concatenate(flip_e)
        assert len(ef) == 0 or math.sqrt((ef * ef).mean()) > 5e-3 or np.abs(ef).max() > 3e-2
        eo = np.concatenate(off_e)
        assert math.sqrt((eo * eo).mean()) > 5e-3 or np.abs(eo).max() > 3e-2


def _bruteforce_cells(g, v, lo, hi, cells, nsub=48, dzs=0.0, nsub_t=None):
    o = (np.arange(nsub) + 0.5) / nsub - 0.5
    nt_ = nsub if nsub_t is None else nsub_t
    ot_ = (np.arange(nt_) + 0.5) / nt_ - 0.5
    out = []
    for (r, c) in cells:
        Ss, Us = [], []
        for os_ in o:
            for ot in ot_:
                S, u = GU.ray(g, v, GU.chan_s(g, c) + os_ * g["ds"], GU.row_t(g, r) + ot * g["dt"])
                S = S.copy()
                S[2] += dzs
                Ss.append(S); Us.append(u)
        out.append(GU.box_chords_vec(np.array(Ss), np.array(Us), lo, hi).mean())
    return np.array(out)


def _voxel_cells(g, v, ix, iy, zc):
    tr = O.transaxial(g, v, ix, iy)
    base = -(g["ns"] - 1) / 2.0
    c_lo = int(math.floor(tr[0] / g["ds"] - base - 0.5)) - 2
    c_hi = int(math.floor(tr[3] / g["ds"] - base + 0.5)) + 2
    zs = GU.source_z(g, v)
    # rows from the independent geometry (geomutil), generously padded
    rh = math.hypot(*((np.array([(ix - (g["nx"] - 1) / 2.0) * g["dx"], (iy - (g["ny"] - 1) / 2.0) * g["dy"]])
                       - GU.ray(g, v, 0.0, 0.0)[0][:2])))
    mag = g["dsd"] / rh
    tl, th = (zc - g["dz"] / 2 - zs) * mag, (zc + g["dz"] / 2 - zs) * mag
    tb = -(g["nt"] - 1) / 2.0
    r_lo = max(0, int(math.floor(min(tl, th) / g["dt"] - tb - 0.5)) - 2)
    r_hi = min(g["nt"] - 1, int(math.floor(max(tl, th) / g["dt"] - tb + 0.5)) + 2)
    return [(r, c) for r in range(r_lo, r_hi + 1) for c in range(c_lo, c_hi + 1)]


def test_single_voxel_bruteforce_helical_c5():
    """c5 geometry, views with |z_s| >= 30 mm, a voxel up to 15 mm above or below the source
    plane: SF-TR weights vs brute-force bin-averaged ray-box chords (48 x 48 sub-rays per cell;
    footprint sum <= 0.5 %, per-cell L2 <= 2 %, the axial pin's tolerances).  The same
    tolerance rejects the brute force taken from a source shifted by half a slice."""
    h = _helical("c5")
    g = GU.geom("cone_helical", nx=512, nz=320, dx=0.9766, dz=0.625, ns=888, ds=1.0239, nt=h["nt"], dt=1.0964,
                na=h["na"], turns=h["turns"], pitch=h["pitch"])
    rng = np.random.default_rng(31)
    caught = 0
    for trial in range(6):
        zs_target = rng.uniform(30.0, 60.0) * (1 if trial % 2 == 0 else -1)
        v = _view_at(g, zs_target)
        zs = GU.source_z(g, v)
        assert abs(zs) >= 29.9
        ix, iy = int(rng.integers(120, 392)), int(rng.integers(120, 392))
        zoff = rng.uniform(-15.0, 15.0)
        iz = int(round((zs + zoff) / g["dz"] + (g["nz"] - 1) / 2.0))
        zc = (iz - (g["nz"] - 1) / 2.0) * g["dz"]
        xc = (ix - (g["nx"] - 1) / 2.0) * g["dx"]; yc = (iy - (g["ny"] - 1) / 2.0) * g["dy"]
        lo = np.array([xc - g["dx"] / 2, yc - g["dy"] / 2, zc - g["dz"] / 2])
        hi = lo + np.array([g["dx"], g["dy"], g["dz"]])
        cells = _voxel_cells(g, v, ix, iy, zc)
        sf = np.array([O.weight(g, v, ix, iy, iz, r, c) for (r, c) in cells])
        bf = _bruteforce_cells(g, v, lo, hi, cells)
        assert bf.sum() > 0
        assert abs(sf.sum() - bf.sum()) <= 5e-3 * bf.sum(), (trial, sf.sum(), bf.sum())
        assert np.linalg.norm(sf - bf) <= 2e-2 * np.linalg.norm(bf), (trial, np.linalg.norm(sf - bf) / np.linalg.norm(bf))
        bfo = _bruteforce_cells(g, v, lo, hi, cells, nsub=24, dzs=0.5 * g["dz"])
        caught += np.linalg.norm(sf - bfo) > 2e-2 * np.linalg.norm(bfo)
    assert caught == 6


def test_ltheta_steep_cone_helical():
    """l_theta = sqrt(1 + ((z_j - z_s)/rho_h)^2) with z_s != 0: a helical scan with a tall
    detector (64 rows x 6 mm, cone half-angle ~11 deg; 24 x 192 sub-rays per cell) and voxels ~0.19 rho_h above / below
    the source, where l_theta - 1 is ~1.8 %.  The footprint mass (sum of a_ij over the cells)
    matches the brute-force ray-box chords to <= 0.5 %, and the same comparison with
    l_theta dropped from the oracle's weights misses by > 1.2 % (l_theta of the voxel centre,
    recomputed here from geomutil's source height)."""
    g = GU.geom("cone_helical", nx=96, nz=256, dx=0.9766, dz=1.25, ns=400, ds=1.0239, nt=64, dt=6.0,
                na=1200, turns=1.0, pitch=0.3)
    rng = np.random.default_rng(41)
    for trial in range(4):
        v = int(rng.integers(0, 300)) if trial < 2 else int(rng.integers(900, 1200))
        zs = GU.source_z(g, v)
        assert abs(zs) >= 15.0
        ix, iy = int(rng.integers(20, 76)), int(rng.integers(20, 76))
        xc = (ix - (g["nx"] - 1) / 2.0) * g["dx"]; yc = (iy - (g["ny"] - 1) / 2.0) * g["dy"]
        S, _ = GU.ray(g, v, 0.0, 0.0)
        rh = math.hypot(xc - S[0], yc - S[1])
        sgn = 1 if trial % 2 == 0 else -1
        iz = int(round((zs + sgn * 0.19 * rh) / g["dz"] + (g["nz"] - 1) / 2.0))
        assert 0 <= iz < g["nz"]
        zc = (iz - (g["nz"] - 1) / 2.0) * g["dz"]
        lth = math.sqrt(1.0 + ((zc - zs) / rh) ** 2)
        assert lth > 1.015
        lo = np.array([xc - g["dx"] / 2, yc - g["dy"] / 2, zc - g["dz"] / 2])
        hi = lo + np.array([g["dx"], g["dy"], g["dz"]])
        cells = _voxel_cells(g, v, ix, iy, zc)
        sf = np.array([O.weight(g, v, ix, iy, iz, r, c) for (r, c) in cells])
        bf = _bruteforce_cells(g, v, lo, hi, cells, nsub=24, nsub_t=192)
        assert bf.sum() > 0
        assert abs(sf.sum() - bf.sum()) <= 5e-3 * bf.sum(), (trial, sf.sum() / bf.sum())
        assert abs(sf.sum() / lth - bf.sum()) > 1.2e-2 * bf.sum()
