"""Seeded synthetic inputs and scan configurations (c1..c5).

This module is the ONLY code shared by the CUDA path's tests/bench and the
fp64 oracle's tests.  It holds none of the method's arithmetic: no system
matrix, no projector, no regulariser, no update.  It produces

* the scan geometry parameters of BASELINE.json ``configs[0..4]`` as plain dicts
  (readings O1, G3, G17 in DESIGN.md),
* analytic ellipse / ellipsoid phantoms and their *exact* line integrals along
  each detector cell's centre ray (ray–quadric chord length x density),
* transmission noise: counts Y ~ Poisson(I0 exp(-p)) + N(0, sigma^2),
  Y~ = max(Y, 1), y = ln(I0 / Y~), W = Y~^2 / (Y~ + sigma^2)   (
  with sigma = 0 this is W = counts),
* the FOV support mask S0 = {r_xy <= r_FOV - dx}.

The paper's data are proprietary GE scans that are absent; these
synthetic inputs stand in for them with the same sinogram shapes (P:573, P:620,
P:1495).  Everything is seeded: phantom parameters from numpy PCG64
(seed 1000 + c), noise from a torch.Generator (seed 2000 + c) on the device the
data are generated on.

Layouts produced here (the C-ABI layout, z / row fastest):
  image    [ny][nx][nz]          sinogram  [na][ns][nt]
``to_oracle_image`` / ``to_oracle_sino`` permute to the oracle's textbook layout.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

MU_WATER = 0.02          # mm^-1 (reading G16: 1 HU = 2e-5 mm^-1)
HU = MU_WATER / 1000.0
DSO, DSD = 541.0, 949.0


@dataclass
class ScanConfig:
    name: str
    geom: dict
    M: int
    n_iter: int
    beta: float
    delta: float
    nbr: int
    I0: float
    sigma: float
    recipe: str
    body_z: float = 0.0            # ellipsoid body z semi-axis (3D)
    extra: dict = field(default_factory=dict)

    @property
    def is2d(self) -> bool:
        return self.geom["kind"] == "fan2d"

    @property
    def img_shape(self):
        g = self.geom
        return (g["ny"], g["nx"], 1 if self.is2d else g["nz"])

    def sino_shape(self, count=None):
        g = self.geom
        return (g["na"] if count is None else count, g["ns"], 1 if self.is2d else g["nt"])


def _geom(kind, nx, dx, nz, dz, ns, ds, nt, dt, na, turns, pitch):
    return dict(kind=kind, nx=nx, ny=nx, nz=nz, dx=dx, dy=dx, dz=dz, offx=0.0, offy=0.0, offz=0.0,
                ns=ns, nt=nt, ds=ds, dt=dt, offs=0.0, offt=0.0, dso=DSO, dsd=DSD, na=na,
                orbit_deg=360.0 * turns, orbit_start_deg=0.0, pitch=pitch)


def config(name: str) -> ScanConfig:
    """BASELINE.json configs[0..4] (c1..c5) with SURVEY §8(d)'s synthetic recipe."""
    d10 = 10 * HU  # delta = 10 HU = 2e-4 mm^-1 (G3)
    if name == "c1":
        return ScanConfig("c1", _geom("fan2d", 64, 4.0, 1, 1.0, 96, 1.0239 * 8, 1, 1.0, 120, 1, 0.0),
                          M=4, n_iter=20, beta=2.0 ** 8, delta=d10, nbr=8, I0=1e5, sigma=0.0, recipe="c1")
    if name == "c2":
        return ScanConfig("c2", _geom("fan2d", 512, 0.9766, 1, 1.0, 888, 1.0239, 1, 1.0, 984, 1, 0.0),
                          M=24, n_iter=30, beta=2.0 ** 13, delta=d10, nbr=8, I0=1e5, sigma=5.0, recipe="body2d")
    if name == "c3":
        return ScanConfig("c3", _geom("cone_axial", 512, 0.9766, 64, 0.625, 888, 1.0239, 64, 1.0964, 984, 1, 0.0),
                          M=24, n_iter=20, beta=2.0 ** 10, delta=d10, nbr=26, I0=1e5, sigma=0.0,
                          recipe="body3d", body_z=0.45 * 40.0)
    if name == "c4":
        return ScanConfig("c4", _geom("cone_helical", 512, 0.9766, 128, 0.625, 888, 1.0239, 32, 1.0964, 2952, 3, 1.0),
                          M=24, n_iter=30, beta=2.0 ** 10, delta=d10, nbr=26, I0=1e5, sigma=0.0,
                          recipe="body3d", body_z=20.0)
    if name == "c5":
        return ScanConfig("c5", _geom("cone_helical", 512, 0.9766, 320, 0.625, 888, 1.0239, 64, 1.0964, 6888, 7, 0.5),
                          M=24, n_iter=20, beta=2.0 ** 10, delta=d10, nbr=26, I0=5e4, sigma=0.0,
                          recipe="body3d", body_z=70.0)
    raise KeyError(name)


CONFIGS = ("c1", "c2", "c3", "c4", "c5")


def scaled(cfg: ScanConfig, name: str, **geom_over) -> ScanConfig:
    """A copy of cfg with geometry fields overridden (small parity cases)."""
    g = dict(cfg.geom)
    g.update(geom_over)
    return ScanConfig(name, g, cfg.M, cfg.n_iter, cfg.beta, cfg.delta, cfg.nbr, cfg.I0, cfg.sigma,
                      cfg.recipe, cfg.body_z, dict(cfg.extra))


def slab_geom(g: dict, z0: int, z1: int) -> dict:
    """The geometry of slices [z0, z1) of g's volume (same scan; voxel centres on g's grid)."""
    s = dict(g)
    s["nz"] = z1 - z0
    s["offz"] = g.get("offz", 0.0) + ((z0 + z1 - 1) / 2.0 - (g["nz"] - 1) / 2.0) * g["dz"]
    return s


def fov_radius(g: dict) -> float:
    """Radius of the circle every fan covers: dso sin(ns ds / (2 dsd))."""
    return g["dso"] * math.sin(g["ns"] * g["ds"] / (2.0 * g["dsd"]))


# ---------------------------------------------------------------------------
# Phantoms: list of (cx, cy, cz, ax, ay, az, angle_rad, delta_mu)
# ---------------------------------------------------------------------------

def _overlaps(e, others, margin=1.0):
    """Conservative overlap test: bounding circles in-plane and z-extents (2D: in-plane only)."""
    for o in others:
        dxy = math.hypot(e[0] - o[0], e[1] - o[1])
        if dxy >= max(e[3], e[4]) + max(o[3], o[4]) + margin:
            continue
        ez, oz = e[5], o[5]
        if ez == 0.0 or math.isinf(ez) or oz == 0.0 or math.isinf(oz):
            return True
        if abs(e[2] - o[2]) < ez + oz + margin:
            return True
    return False


def phantom(cfg: ScanConfig, seed: int | None = None):
    """Seeded list of ellipsoids (2D: ellipses with az = inf)."""
    c = int(cfg.name[1]) if cfg.name[:1] == "c" and cfg.name[1:2].isdigit() else 0
    rng = np.random.Generator(np.random.PCG64(1000 + c if seed is None else seed))
    g = cfg.geom
    inf = float("inf")
    ell = []
    if cfg.recipe == "c1":
        body = (0.0, 0.0, 0.0, 108.8, 89.6, inf, 0.0, 0.015)
        ell.append(body)
        inserts = []
        while len(inserts) < 8:
            a, b = rng.uniform(5, 25, size=2)
            cx, cy = rng.uniform(-0.7, 0.7) * body[3], rng.uniform(-0.7, 0.7) * body[4]
            e = (cx, cy, 0.0, a, b, 0.0, rng.uniform(0, math.pi), rng.uniform(-0.015, 0.005))
            if (cx / body[3]) ** 2 + (cy / body[4]) ** 2 > (1 - max(a, b) / min(body[3], body[4])) ** 2:
                continue
            if _overlaps(e, inserts):
                continue
            inserts.append(e)
        ell += [(e[0], e[1], 0.0, e[3], e[4], inf, e[6], e[7]) for e in inserts]
        return ell
    threed = not cfg.is2d
    Z = g["nz"] * g["dz"] if threed else 0.0
    bz = cfg.body_z if threed else inf
    body = (0.0, 0.0, 0.0, 200.0, 150.0, bz, 0.0, MU_WATER)
    lz = (0.3 / 0.45) * bz if threed else inf
    sz = (0.4 / 0.45) * bz if threed else inf
    fixed = [(-80.0, 20.0, 0.0, 40.0, 60.0, lz, 0.0, -MU_WATER),
             (80.0, 20.0, 0.0, 40.0, 60.0, lz, 0.0, -MU_WATER)]
    if threed:
        fixed.append((0.0, -100.0, 0.0, 15.0, 15.0, sz, 0.0, MU_WATER))
    else:
        fixed.append((0.0, -100.0, 0.0, 15.0, 15.0, inf, 0.0, MU_WATER))
    ell.append(body)
    ell += fixed
    n_ins = 10 if threed else 6
    inserts = []
    tries = 0
    while len(inserts) < n_ins and tries < 100000:
        tries += 1
        a, b = rng.uniform(5, 30, size=2)
        az = min(rng.uniform(5, 30), (0.3 / 0.45) * bz) if threed else 0.0
        cx, cy = rng.uniform(-0.75, 0.75) * 200.0, rng.uniform(-0.75, 0.75) * 150.0
        cz = rng.uniform(-0.5, 0.5) * (bz - az) if threed else 0.0
        e = (cx, cy, cz, a, b, az, rng.uniform(0, math.pi), rng.uniform(-0.004, 0.004))
        r = max(a, b)
        if ((abs(cx) + r) / 200.0) ** 2 + ((abs(cy) + r) / 150.0) ** 2 > 1.0:
            continue
        if _overlaps(e, inserts + fixed):
            continue
        inserts.append(e)
    ell += [e if threed else (e[0], e[1], 0.0, e[3], e[4], inf, e[6], e[7]) for e in inserts]
    return ell


# ---------------------------------------------------------------------------
# Ray geometry of a detector cell centre (O1) — used only to synthesise data
# ---------------------------------------------------------------------------

def cell_rays(g: dict, views, device="cpu", dtype=torch.float64):
    """Source points S[v,3] and unit directions U[v,ns,nt,3] of cell-centre rays."""
    views = torch.as_tensor(views, dtype=dtype, device=device)
    turns = g["orbit_deg"] / 360.0
    beta = g["orbit_start_deg"] * math.pi / 180.0 + 2 * math.pi * turns * views / g["na"]
    sb, cb = torch.sin(beta), torch.cos(beta)
    if g["kind"] == "cone_helical":
        h = g["pitch"] * g["nt"] * g["dt"] * g["dso"] / g["dsd"]
        zs = (views - (g["na"] - 1) / 2.0) * h / (g["na"] / turns)
    else:
        zs = torch.zeros_like(views)
    S = torch.stack([-g["dso"] * sb, g["dso"] * cb, zs], -1)
    c = torch.arange(g["ns"], dtype=dtype, device=device)
    gam = (c - (g["ns"] - 1) / 2.0 - g["offs"]) * g["ds"] / g["dsd"]
    nt = 1 if g["kind"] == "fan2d" else g["nt"]
    r = torch.arange(nt, dtype=dtype, device=device)
    t = (r - (nt - 1) / 2.0 - g["offt"]) * g["dt"] if g["kind"] != "fan2d" else torch.zeros(1, dtype=dtype, device=device)
    ec = torch.stack([sb, -cb], -1)          # [v,2]
    ep = torch.stack([cb, sb], -1)
    dxy = g["dsd"] * (torch.cos(gam)[None, :, None] * ec[:, None, :] + torch.sin(gam)[None, :, None] * ep[:, None, :])
    D = torch.empty((len(views), g["ns"], nt, 3), dtype=dtype, device=device)
    D[..., 0] = dxy[:, :, None, 0].expand(-1, -1, nt)
    D[..., 1] = dxy[:, :, None, 1].expand(-1, -1, nt)
    D[..., 2] = t[None, None, :].expand(len(views), g["ns"], nt)
    n = torch.linalg.vector_norm(D, dim=-1, keepdim=True)
    return S, D / n


def line_integrals(g: dict, ell, views, device="cpu"):
    """Exact line integrals of the ellipsoid phantom along cell-centre rays: [v, ns, nt]."""
    S, U = cell_rays(g, views, device)
    p = torch.zeros(U.shape[:-1], dtype=torch.float64, device=device)
    for (cx, cy, cz, ax, ay, az, ang, mu) in ell:
        ca, sa = math.cos(ang), math.sin(ang)
        # rotate into the ellipsoid frame, scale to the unit sphere
        o = S - torch.tensor([cx, cy, cz], dtype=torch.float64, device=device)
        ox = (ca * o[:, 0] + sa * o[:, 1]) / ax
        oy = (-sa * o[:, 0] + ca * o[:, 1]) / ay
        ux = (ca * U[..., 0] + sa * U[..., 1]) / ax
        uy = (-sa * U[..., 0] + ca * U[..., 1]) / ay
        if math.isinf(az):
            oz = torch.zeros_like(ox); uz = torch.zeros_like(ux)
        else:
            oz = o[:, 2] / az; uz = U[..., 2] / az
        ox, oy, oz = ox[:, None, None], oy[:, None, None], oz[:, None, None]
        A = ux * ux + uy * uy + uz * uz
        B = 2 * (ox * ux + oy * uy + oz * uz)
        C = ox * ox + oy * oy + oz * oz - 1
        disc = B * B - 4 * A * C
        chord = torch.where(disc > 0, torch.sqrt(disc.clamp_min(0)) / A, torch.zeros_like(A))
        p += mu * chord
    return p


def noisy_data(g: dict, ell, I0: float, sigma: float, seed: int, device="cpu", views_per_chunk=64):
    """Transmission data for an ellipsoid list: dict(y, w, p_true) fp32 [na][ns][nt] (O3)."""
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    ys, ws, ps = [], [], []
    for v0 in range(0, g["na"], views_per_chunk):
        views = list(range(v0, min(g["na"], v0 + views_per_chunk)))
        p = line_integrals(g, ell, views, device)
        lam = I0 * torch.exp(-p)
        Y = torch.poisson(lam, generator=gen)
        if sigma > 0:
            Y = Y + sigma * torch.randn(Y.shape, generator=gen, dtype=Y.dtype, device=device)
        Yt = Y.clamp_min(1.0)
        ys.append(torch.log(I0 / Yt).float())
        ws.append((Yt * Yt / (Yt + sigma ** 2)).float())
        ps.append(p.float())
    return dict(y=torch.cat(ys), w=torch.cat(ws), p_true=torch.cat(ps))


def synthesize(cfg: ScanConfig, device="cpu", views_per_chunk=64, seed_noise=None):
    """Return dict(y, w, p_true) fp32 in the ABI sinogram layout [na][ns][nt]."""
    c = int(cfg.name[1]) if cfg.name[:1] == "c" and cfg.name[1:2].isdigit() else 0
    return noisy_data(cfg.geom, phantom(cfg), cfg.I0, cfg.sigma, 2000 + c if seed_noise is None else seed_noise,
                      device, views_per_chunk)


def support_mask(cfg: ScanConfig, device="cpu"):
    """S0 = voxels whose centre has r_xy <= r_FOV - dx (O4), uint8 [ny][nx][nz]."""
    g = cfg.geom
    ix = torch.arange(g["nx"], dtype=torch.float64, device=device)
    iy = torch.arange(g["ny"], dtype=torch.float64, device=device)
    xc = (ix - (g["nx"] - 1) / 2.0) * g["dx"] + g["offx"]
    yc = (iy - (g["ny"] - 1) / 2.0) * g["dy"] + g["offy"]
    r = torch.sqrt(yc[:, None] ** 2 + xc[None, :] ** 2)
    m = (r <= fov_radius(g) - g["dx"]).to(torch.uint8)
    nz = 1 if cfg.is2d else g["nz"]
    return m[:, :, None].expand(-1, -1, nz).contiguous()


def voxelized_phantom(cfg: ScanConfig, ss=4, device="cpu"):
    """Phantom sampled on the grid with ss^3 supersampling, fp32 [ny][nx][nz] (sanity only)."""
    g = cfg.geom
    nz = 1 if cfg.is2d else g["nz"]
    out = torch.zeros((g["ny"], g["nx"], nz), dtype=torch.float64, device=device)
    o = (torch.arange(ss, dtype=torch.float64, device=device) + 0.5) / ss - 0.5
    ell = phantom(cfg)
    for sy in o:
        for sx in o:
            for sz in (o if not cfg.is2d else torch.zeros(1, dtype=torch.float64)):
                xc = (torch.arange(g["nx"], dtype=torch.float64, device=device) - (g["nx"] - 1) / 2.0 + sx) * g["dx"]
                yc = (torch.arange(g["ny"], dtype=torch.float64, device=device) - (g["ny"] - 1) / 2.0 + sy) * g["dy"]
                zc = ((torch.arange(nz, dtype=torch.float64, device=device) - (nz - 1) / 2.0 + sz) * g["dz"]
                      if not cfg.is2d else torch.zeros(1, dtype=torch.float64, device=device))
                Y, X, Zc = torch.meshgrid(yc, xc, zc, indexing="ij")
                for (cx, cy, cz, ax, ay, az, ang, mu) in ell:
                    ca, sa = math.cos(ang), math.sin(ang)
                    u = (ca * (X - cx) + sa * (Y - cy)) / ax
                    w = (-sa * (X - cx) + ca * (Y - cy)) / ay
                    q = u * u + w * w + (0 if math.isinf(az) else ((Zc - cz) / az) ** 2)
                    out += mu * (q <= 1).double()
    n = ss * ss * (1 if cfg.is2d else ss)
    return (out / n).float()


# ---------------------------------------------------------------------------
# Layout permutations ABI <-> oracle (pure data movement)
# ---------------------------------------------------------------------------

def to_oracle_image(x):
    """[ny][nx][nz] -> [nz][ny][nx] numpy fp64."""
    x = np.asarray(x.detach().cpu() if isinstance(x, torch.Tensor) else x)
    return np.ascontiguousarray(np.transpose(x, (2, 0, 1))).astype(np.float64)


def from_oracle_image(x):
    return np.ascontiguousarray(np.transpose(np.asarray(x), (1, 2, 0)))


def to_oracle_sino(p):
    """[v][ns][nt] -> [v][nt][ns] numpy fp64."""
    p = np.asarray(p.detach().cpu() if isinstance(p, torch.Tensor) else p)
    return np.ascontiguousarray(np.transpose(p, (0, 2, 1))).astype(np.float64)


def from_oracle_sino(p):
    return np.ascontiguousarray(np.transpose(np.asarray(p), (0, 2, 1)))
