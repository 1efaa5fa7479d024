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
