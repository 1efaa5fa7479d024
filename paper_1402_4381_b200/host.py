"""Host-side helpers of the product path (no device arithmetic).

* ``max_subsets_axial`` / ``max_subsets_helical`` — the paper's subset-count rules,
  PAPER.md P:541-559 (eqs. max_M_axial, max_M_helical; s_axial ~ 40, s_helical ~ 24).
* ``rank_view_block`` — the multi-GPU partition of one subset's views:
  rank p of P owns a contiguous block of the subset's n_m views.
* ``rank_zslab`` — the z-slab decomposition (NEXT-3): rank p owns slices [z0, z1) of the
  volume and works on the slab's own geometry (``inputs.slab_geom``).
* ``rank_slab`` — the multi-GPU partition of the image for the SQS update: rank p owns a
  contiguous block of image rows (iy); buffers are padded to P equal slabs (mirror of
  ``slab_geometry`` in ct_abi.cu).
* ``rank_band`` — the z-band of slices a rank's view block of a subset can see (band-limited
  exchange of helical scans; mirror of ``rank_band`` in ct_abi.cu).
"""
from __future__ import annotations

import math


def max_subsets_axial(n_views: int, s_axial: float = 40) -> int:
    """M_axial <= (number of views) / s_axial."""
    return max(1, int(math.floor(n_views / s_axial)))


def max_subsets_helical(views_per_turn: int, dso: float, dsd: float, pitch: float, s_helical: float = 24) -> int:
    """M_helical <= (views per turn) dso / (p s_helical dsd)."""
    return max(1, int(math.floor(views_per_turn * dso / (pitch * s_helical * dsd))))


def subset_views(na: int, M: int, m: int) -> tuple[int, int, int]:
    """(first, stride, count) of subset m = {v : v mod M = m} (reading G12)."""
    return m, M, (na - m + M - 1) // M


def rank_view_block(count: int, rank: int, nranks: int) -> tuple[int, int]:
    """Contiguous block [k0, k0 + n) of a subset's `count` views owned by `rank` (§8(e))."""
    base, extra = divmod(count, nranks)
    k0 = rank * base + min(rank, extra)
    return k0, base + (1 if rank < extra else 0)


def rank_slab(ny: int, rank: int, nranks: int) -> tuple[int, int, int]:
    """Rows [iy0, iy1) of the image owned by `rank`, and the padded rows per slab R (P*R >= ny)."""
    R = (ny + nranks - 1) // nranks
    return min(ny, rank * R), min(ny, (rank + 1) * R), R


def rank_zslab(nz: int, rank: int, nranks: int) -> tuple[int, int]:
    """Slices [z0, z1) of the volume owned by `rank` in the z-slab decomposition (NEXT-3)."""
    base, extra = divmod(nz, nranks)
    z0 = rank * base + min(rank, extra)
    return z0, z0 + base + (1 if rank < extra else 0)


def helical_zhalf(g: dict) -> float:
    """Bound on |z - z_s| of any voxel a view can see (mm): half the detector height (plus its
    offset) at the smallest magnification, plus one slice (mirror of DevGeom.zhalf)."""
    hx = 0.5 * (g["nx"] - 1) * g["dx"] + abs(g.get("offx", 0.0)) + g["dx"]
    hy = 0.5 * (g["ny"] - 1) * g["dy"] + abs(g.get("offy", 0.0)) + g["dy"]
    rmax = math.hypot(hx, hy)
    return (0.5 * g["nt"] * g["dt"] + 0.5 * abs(g.get("offt", 0.0)) * g["dt"]) * (g["dso"] + rmax) / g["dsd"] + g["dz"]


def zslab_window(g: dict, M: int, m: int, z0: int, z1: int) -> tuple[int, int]:
    """Indices [k0, k1) of subset m's views whose cone can reach slices [z0, z1) of the volume
    (helical z-slab ranks; mirror of zslab_window_of in ct_abi.cu: source heights within the
    cone's z reach of the slab, widened by one slice and one / two views)."""
    count = (g["na"] - m + M - 1) // M
    if g["kind"] != "cone_helical" or count == 0:
        return 0, count
    turns = g["orbit_deg"] / 360.0
    h = g["pitch"] * g["nt"] * g["dt"] * g["dso"] / g["dsd"]
    dzs = h / (g["na"] / turns)
    zs0 = -(g["na"] - 1) / 2.0 * dzs
    zb0 = -(g["nz"] - 1) / 2.0 * g["dz"] + g.get("offz", 0.0) - 0.5 * g["dz"]
    zlo, zhi = zb0 + z0 * g["dz"], zb0 + z1 * g["dz"]
    zh = helical_zhalf(g) + g["dz"]
    vlo, vhi = (zlo - zh - zs0) / dzs, (zhi + zh - zs0) / dzs
    k0 = max(0, math.floor((vlo - m) / M) - 1)
    k1 = min(count, math.ceil((vhi - m) / M) + 2)
    return k0, max(k0, k1)


def zslab_exchange_floats(g: dict, M: int, m: int, rank: int, nranks: int) -> int:
    """Floats rank `rank` receives in the windowed z-slab exchange of subset m: for every other
    rank, the views both windows hold, times the detector cells per view."""
    z0, z1 = rank_zslab(g["nz"], rank, nranks)
    a0, a1 = zslab_window(g, M, m, z0, z1)
    n = 0
    for q in range(nranks):
        if q != rank:
            b0, b1 = zslab_window(g, M, m, *rank_zslab(g["nz"], q, nranks))
            n += max(0, min(a1, b1) - max(a0, b0))
    return n * g["ns"] * g["nt"]


def rank_band(g: dict, M: int, m: int, rank: int, nranks: int) -> tuple[int, int]:
    """Slices [b0, b1) in which `rank`'s partial back-projection of subset m can be non-zero:
    the source heights of its contiguous view block widened by the cone's z reach and one
    slice (helical scans)."""
    count = (g["na"] - m + M - 1) // M
    k0, n = rank_view_block(count, rank, nranks)
    if n <= 0:
        return 0, 0
    turns = g["orbit_deg"] / 360.0
    h = g["pitch"] * g["nt"] * g["dt"] * g["dso"] / g["dsd"]
    dzs = h / (g["na"] / turns)
    zs0 = -(g["na"] - 1) / 2.0 * dzs
    za, zb = zs0 + (m + k0 * M) * dzs, zs0 + (m + (k0 + n - 1) * M) * dzs
    zh = helical_zhalf(g) + g["dz"]
    zb0 = -(g["nz"] - 1) / 2.0 * g["dz"] + g.get("offz", 0.0) - 0.5 * g["dz"]
    b0 = max(0, math.floor((min(za, zb) - zh - zb0) / g["dz"]) - 1)
    b1 = min(g["nz"], math.ceil((max(za, zb) + zh - zb0) / g["dz"]) + 1)
    return b0, max(b0, b1)
