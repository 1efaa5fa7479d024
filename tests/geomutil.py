"""Small test geometries and independent reference routines used by the pins.

Nothing here calls the oracle's arithmetic: these are textbook computations
(ray–box chords by slab clipping, ray–pixel chords by grid-line crossing,
closed-form disk chords) written from scratch for the tests.
"""
from __future__ import annotations

import math

import numpy as np


def geom(kind="fan2d", nx=16, ny=None, nz=1, dx=8.0, dz=1.0, ns=24, ds=14.0, nt=1, dt=1.0,
         na=36, dso=541.0, dsd=949.0, turns=1.0, pitch=0.0, start=0.0, offx=0.0, offy=0.0, offz=0.0,
         offs=0.0, offt=0.0):
    return dict(kind=kind, nx=nx, ny=nx if ny is None else ny, nz=nz, dx=dx, dy=dx, dz=dz,
                offx=offx, offy=offy, offz=offz, ns=ns, nt=nt, ds=ds, dt=dt, offs=offs, offt=offt,
                dso=dso, dsd=dsd, na=na, orbit_deg=360.0 * turns, orbit_start_deg=start, pitch=pitch)


def small_geoms():
    """Scaled-down versions of the five BASELINE geometries (fan, axial, helical)."""
    return {
        "fan_c1": geom("fan2d", nx=20, dx=4.0, ns=40, ds=8.1912, na=30),
        "fan_c2": geom("fan2d", nx=24, ny=20, dx=0.9766, ns=48, ds=1.0239, na=36, offx=1.3, offy=-0.7),
        "axial_c3": geom("cone_axial", nx=12, nz=6, dx=0.9766, dz=0.625, ns=24, ds=1.0239, nt=8, dt=1.0964, na=24),
        "helical_c4": geom("cone_helical", nx=12, nz=10, dx=0.9766, dz=0.625, ns=24, ds=1.0239, nt=4,
                           dt=1.0964, na=48, turns=3.0, pitch=1.0),
        "helical_c5": geom("cone_helical", nx=10, nz=12, dx=0.9766, dz=0.625, ns=20, ds=1.0239, nt=6,
                           dt=1.0964, na=42, turns=2.0, pitch=0.5, start=17.0),
    }


def view_angle(g, v):
    return math.radians(g["orbit_start_deg"]) + 2 * math.pi * (g["orbit_deg"] / 360.0) * v / g["na"]


def source_z(g, v):
    if g["kind"] != "cone_helical":
        return 0.0
    turns = g["orbit_deg"] / 360.0
    h = g["pitch"] * g["nt"] * g["dt"] * g["dso"] / g["dsd"]
    return (v - (g["na"] - 1) / 2.0) * h / (g["na"] / turns)


def ray(g, v, s_arc, t_row):
    """Source point and unit direction of the ray hitting arc position s_arc, row height t_row."""
    b = view_angle(g, v)
    ec = np.array([math.sin(b), -math.cos(b)])
    ep = np.array([math.cos(b), math.sin(b)])
    S = np.array([-g["dso"] * math.sin(b), g["dso"] * math.cos(b), source_z(g, v)])
    gam = s_arc / g["dsd"]
    dxy = g["dsd"] * (math.cos(gam) * ec + math.sin(gam) * ep)
    d = np.array([dxy[0], dxy[1], t_row])
    return S, d / np.linalg.norm(d)


def chan_s(g, c):
    return (c - (g["ns"] - 1) / 2.0 - g["offs"]) * g["ds"]


def row_t(g, r):
    nt = 1 if g["kind"] == "fan2d" else g["nt"]
    return (r - (nt - 1) / 2.0 - g["offt"]) * g["dt"]


def box_chord(S, u, lo, hi):
    """Length of the segment of the line S + t u inside the axis-aligned box [lo, hi] (slab clipping)."""
    t0, t1 = -np.inf, np.inf
    for k in range(len(lo)):
        if abs(u[k]) < 1e-300:
            if S[k] < lo[k] or S[k] > hi[k]:
                return 0.0
            continue
        a = (lo[k] - S[k]) / u[k]
        b = (hi[k] - S[k]) / u[k]
        t0 = max(t0, min(a, b))
        t1 = min(t1, max(a, b))
    return max(0.0, t1 - t0)


def box_chords_vec(S, U, lo, hi):
    """Vectorised slab clipping: S [n,d], U [n,d] unit, lo/hi [d] -> chord [n]."""
    with np.errstate(divide="ignore", invalid="ignore"):
        a = (lo[None, :] - S) / U
        b = (hi[None, :] - S) / U
    tmin = np.where(np.abs(U) < 1e-300, np.where((S >= lo) & (S <= hi), -np.inf, np.inf), np.minimum(a, b))
    tmax = np.where(np.abs(U) < 1e-300, np.where((S >= lo) & (S <= hi), np.inf, -np.inf), np.maximum(a, b))
    t0 = tmin.max(axis=1)
    t1 = tmax.min(axis=1)
    return np.maximum(0.0, t1 - t0)


def pixel_grid_chords(S, U, g):
    """Exact ray–pixel intersection lengths for 2D rays (textbook grid-crossing / Siddon).

    S [n,2], U [n,2] unit directions.  Returns list of (ray index, pixel flat index iy*nx+ix, length).
    Implemented by collecting every crossing parameter with the x- and y- grid lines,
    sorting, and assigning each sub-segment to the pixel containing its midpoint.
    """
    nx, ny, dx, dy = g["nx"], g["ny"], g["dx"], g["dy"]
    x0 = -(nx / 2.0) * dx + g["offx"]
    y0 = -(ny / 2.0) * dy + g["offy"]
    xs = x0 + dx * np.arange(nx + 1)
    ys = y0 + dy * np.arange(ny + 1)
    rows, cols, vals = [], [], []
    for i in range(S.shape[0]):
        s, u = S[i], U[i]
        ts = []
        if abs(u[0]) > 1e-300:
            ts.append((xs - s[0]) / u[0])
        if abs(u[1]) > 1e-300:
            ts.append((ys - s[1]) / u[1])
        t = np.sort(np.concatenate(ts))
        mid = 0.5 * (t[1:] + t[:-1])
        L = t[1:] - t[:-1]
        px = s[0] + mid * u[0]
        py = s[1] + mid * u[1]
        ix = np.floor((px - x0) / dx).astype(np.int64)
        iy = np.floor((py - y0) / dy).astype(np.int64)
        ok = (ix >= 0) & (ix < nx) & (iy >= 0) & (iy < ny) & (L > 0)
        rows.append(np.full(ok.sum(), i))
        cols.append(iy[ok] * nx + ix[ok])
        vals.append(L[ok])
    return np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)
