"""fp64 CPU ORACLE for the OS-LALM CT hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package.  The product
package ``paper_1402_4381_b200`` never imports it, and the two share no code.

This module is a thin ctypes loader around ``oracle.c`` (plain C, fp64,
OpenMP over independent outputs).  Every function there cites the paper
passage (PAPER.md line) or SURVEY §8(c) reading (O1..O7, G1..G21) it follows.

Layouts used by the oracle (its own textbook layout; tests permute to/from the
C-ABI layout):  image ``x[iz][iy][ix]``; sinogram ``p[view][row][channel]``.

Parity status (see DESIGN.md §Oracle pins): every function here is pinned by a
``-m "not gpu"`` test in ``tests/test_oracle_*.py``; none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

KIND = {"fan2d": 0, "cone_axial": 1, "cone_helical": 2}


class _Geom(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int),
        ("nx", ctypes.c_int), ("ny", ctypes.c_int), ("nz", ctypes.c_int),
        ("dx", ctypes.c_double), ("dy", ctypes.c_double), ("dz", ctypes.c_double),
        ("offx", ctypes.c_double), ("offy", ctypes.c_double), ("offz", ctypes.c_double),
        ("ns", ctypes.c_int), ("nt", ctypes.c_int),
        ("ds", ctypes.c_double), ("dt", ctypes.c_double),
        ("offs", ctypes.c_double), ("offt", ctypes.c_double),
        ("dso", ctypes.c_double), ("dsd", ctypes.c_double),
        ("na", ctypes.c_int),
        ("orbit_deg", ctypes.c_double), ("orbit_start_deg", ctypes.c_double),
        ("pitch", ctypes.c_double),
    ]


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc, -O2, IEEE fp64, OpenMP)."""
    with _lock:
        if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
            tmp = _LIB + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                                   "-D_GNU_SOURCE", "-o", tmp, _SRC, "-lm"])
            os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        G = ctypes.POINTER(_Geom)
        dp = ctypes.POINTER(ctypes.c_double)
        u8 = ctypes.POINTER(ctypes.c_uint8)
        ip = ctypes.POINTER(ctypes.c_int)
        i, d = ctypes.c_int, ctypes.c_double
        L.or_view_angle.argtypes = [G, i]; L.or_view_angle.restype = d
        L.or_source_z.argtypes = [G, i]; L.or_source_z.restype = d
        L.or_weight.argtypes = [G, i, i, i, i, i, i]; L.or_weight.restype = d
        L.or_transaxial.argtypes = [G, i, i, i, dp]; L.or_transaxial.restype = None
        L.or_fwd.argtypes = [G, i, i, i, dp, dp]; L.or_fwd.restype = None
        L.or_back.argtypes = [G, i, i, i, dp, dp]; L.or_back.restype = None
        L.or_count_vv.argtypes = [G, i, i, i, u8]; L.or_count_vv.restype = ctypes.c_longlong
        L.or_sqs_denom.argtypes = [G, dp, u8, dp]; L.or_sqs_denom.restype = None
        L.or_reg_value.argtypes = [G, d, d, i, u8, dp]; L.or_reg_value.restype = d
        L.or_reg_grad.argtypes = [G, d, d, i, u8, dp, dp, dp]; L.or_reg_grad.restype = None
        L.or_cost.argtypes = [G, dp, dp, d, d, i, u8, dp]; L.or_cost.restype = d
        L.or_bit_reversal.argtypes = [i, ip]; L.or_bit_reversal.restype = None
        L.or_rho_l.argtypes = [ctypes.c_long, d]; L.or_rho_l.restype = d
        L.or_subset_grad.argtypes = [G, i, i, dp, dp, dp, dp]; L.or_subset_grad.restype = None
        L.or_oslalm_run.argtypes = [G, dp, dp, dp, u8, i, i, d, d, d, d, i, i, i, dp, dp, dp, dp, i, i, i, d, dp]
        L.or_inner_fista.argtypes = [G, d, d, i, u8, dp, d, dp, dp, i, dp]
        L.or_inner_fista.restype = None
        L.or_fbp.argtypes = [G, dp, dp]; L.or_fbp.restype = i
        L.or_oslalm_run.restype = None
        _lib = L
    return _lib


# ----------------------------------------------------------------------------
# Python-facing helpers (fp64 numpy arrays in the oracle's own layout)
# ----------------------------------------------------------------------------

def geom(g: dict) -> _Geom:
    """Build the C geometry struct from a plain dict of scan parameters."""
    s = _Geom()
    s.kind = KIND[g["kind"]]
    for k in ("nx", "ny", "nz", "ns", "nt", "na"):
        setattr(s, k, int(g[k]))
    for k in ("dx", "dy", "dz", "offx", "offy", "offz", "ds", "dt", "offs", "offt",
              "dso", "dsd", "orbit_deg", "orbit_start_deg", "pitch"):
        setattr(s, k, float(g.get(k, 0.0)))
    return s


def _alpha_ptr(a, n):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous and a.size >= n, "alpha_out: float64[n_iter]"
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _d(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _u8(a):
    a = np.ascontiguousarray(a, dtype=np.uint8)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))


def img_shape(g):
    return (1 if g["kind"] == "fan2d" else g["nz"], g["ny"], g["nx"])


def sino_shape(g, count):
    return (count, 1 if g["kind"] == "fan2d" else g["nt"], g["ns"])


def nviews(g, first, stride):
    return (g["na"] - first + stride - 1) // stride


def fwd(g, x, first=0, stride=1, count=None):
    count = nviews(g, first, stride) if count is None else count
    x, xp = _d(np.reshape(x, img_shape(g)))
    p = np.zeros(sino_shape(g, count))
    _, pp = _d(p)
    lib().or_fwd(geom(g), first, stride, count, xp, pp)
    return p


def back(g, p, first=0, stride=1, count=None):
    count = nviews(g, first, stride) if count is None else count
    p, pp = _d(np.reshape(p, sino_shape(g, count)))
    x = np.zeros(img_shape(g))
    _, xp = _d(x)
    lib().or_back(geom(g), first, stride, count, pp, xp)
    return x


def weight(g, v, ix, iy, iz, r, c):
    return lib().or_weight(geom(g), v, ix, iy, iz, r, c)


def transaxial(g, v, ix, iy):
    out = np.zeros(6)
    _, op = _d(out)
    lib().or_transaxial(geom(g), v, ix, iy, op)
    return out


def view_angle(g, v):
    return lib().or_view_angle(geom(g), v)


def source_z(g, v):
    return lib().or_source_z(geom(g), v)


def count_vv(g, mask=None, first=0, stride=1, count=None):
    count = nviews(g, first, stride) if count is None else count
    if mask is None:
        return lib().or_count_vv(geom(g), first, stride, count, None)
    m, mp = _u8(np.reshape(mask, img_shape(g)))
    return lib().or_count_vv(geom(g), first, stride, count, mp)


def sqs_denom(g, w, mask):
    w, wp = _d(np.reshape(w, sino_shape(g, g["na"])))
    m = np.array(np.reshape(mask, img_shape(g)), dtype=np.uint8, copy=True)
    _, mp = _u8(m)
    dl = np.zeros(img_shape(g))
    _, dp = _d(dl)
    lib().or_sqs_denom(geom(g), wp, mp, dp)
    return dl, m


def reg_value(g, beta, delta, nbr, mask, x):
    m, mp = _u8(np.reshape(mask, img_shape(g)))
    x, xp = _d(np.reshape(x, img_shape(g)))
    return lib().or_reg_value(geom(g), beta, delta, nbr, mp, xp)


def reg_grad(g, beta, delta, nbr, mask, x):
    m, mp = _u8(np.reshape(mask, img_shape(g)))
    x, xp = _d(np.reshape(x, img_shape(g)))
    gr = np.zeros(img_shape(g)); cu = np.zeros(img_shape(g))
    _, gp = _d(gr); _, cp = _d(cu)
    lib().or_reg_grad(geom(g), beta, delta, nbr, mp, xp, gp, cp)
    return gr, cu


def cost(g, y, w, beta, delta, nbr, mask, x):
    y, yp = _d(np.reshape(y, sino_shape(g, g["na"])))
    w, wp = _d(np.reshape(w, sino_shape(g, g["na"])))
    m, mp = _u8(np.reshape(mask, img_shape(g)))
    x, xp = _d(np.reshape(x, img_shape(g)))
    return lib().or_cost(geom(g), yp, wp, beta, delta, nbr, mp, xp)


def bit_reversal(M):
    out = (ctypes.c_int * M)()
    lib().or_bit_reversal(M, out)
    return list(out)


def rho_l(l, rho_min=1e-3):
    return lib().or_rho_l(int(l), float(rho_min))


def subset_grad(g, M, m, y, w, x):
    y, yp = _d(np.reshape(y, sino_shape(g, g["na"])))
    w, wp = _d(np.reshape(w, sino_shape(g, g["na"])))
    x, xp = _d(np.reshape(x, img_shape(g)))
    G = np.zeros(img_shape(g))
    _, Gp = _d(G)
    lib().or_subset_grad(geom(g), M, m, yp, wp, xp, Gp)
    return G


def inner_fista(g, beta, delta, nbr, mask, dl, rho, xk, s, n):
    """n warm-started FISTA iterations on the inner denoising problem (NEXT-1)."""
    m, mp = _u8(np.reshape(mask, img_shape(g)))
    dl, dp = _d(np.reshape(dl, img_shape(g)))
    xk, xp = _d(np.reshape(xk, img_shape(g)))
    s, sp = _d(np.reshape(s, img_shape(g)))
    out = np.zeros(img_shape(g))
    _, op = _d(out)
    lib().or_inner_fista(geom(g), beta, delta, nbr, mp, dp, rho, xp, sp, n, op)
    return out


def fbp(g, p):
    """FBP (fan) / FDK (cone, circular orbit) initial image of sinogram p (reading B-FBP), or
    the view-normalised helical FDK (reading B-FBP-H); raises for a partial circular orbit."""
    p, pp = _d(np.reshape(p, sino_shape(g, g["na"])))
    x = np.zeros(img_shape(g))
    _, xp = _d(x)
    if lib().or_fbp(geom(g), pp, xp) != 0:
        raise ValueError("FBP of a circular orbit needs one full turn")
    return x


def oslalm_run(g, y, w, dl, mask, x0, *, M, mode="continuation", rho_fixed=1.0, rho_min=1e-3,
               beta, delta, nbr, n_iter, trailing=False, inner="sqs", n_inner=1, bb=False, alpha_min=1e-6,
               alpha_out=None):
    """Run O7; returns (x, log[n_steps,3] = (rho, xi, restart), g, G).
    inner = "sqs" (one Huber-curvature SQS step, G14) or "fista" (n_inner FISTA iterations, NEXT-1).
    bb = True: Barzilai-Borwein scaling H_k = alpha_k D_L (NEXT-2); alpha_out (float64 array of
    n_iter, optional) receives the alpha used in each outer iteration."""
    y, yp = _d(np.reshape(y, sino_shape(g, g["na"])))
    w, wp = _d(np.reshape(w, sino_shape(g, g["na"])))
    dl, dp = _d(np.reshape(dl, img_shape(g)))
    m, mp = _u8(np.reshape(mask, img_shape(g)))
    x = np.array(np.reshape(x0, img_shape(g)), dtype=np.float64, copy=True)
    _, xp = _d(x)
    log = np.zeros((n_iter * M, 3))
    _, lp = _d(log)
    gs = np.zeros(img_shape(g)); Gs = np.zeros(img_shape(g))
    _, gp = _d(gs); _, Gp = _d(Gs)
    lib().or_oslalm_run(geom(g), yp, wp, dp, mp, M, 0 if mode == "fixed" else 1, rho_fixed, rho_min,
                        beta, delta, nbr, n_iter, 1 if trailing else 0, xp, lp, gp, Gp,
                        0 if inner == "sqs" else 1, int(n_inner), 1 if bb else 0, float(alpha_min),
                        _alpha_ptr(alpha_out, n_iter))
    return x, log, gs, Gs
