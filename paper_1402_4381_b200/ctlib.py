"""Thin Python binding of the C ABI in ``include/ct_oslalm.h`` (ctypes).

Argument marshalling only: every step of the hot path runs in the sm_100a kernels
of ``libct_oslalm.so``.  There is no CPU fallback — if the library is missing or
a call fails, a ``CTError`` is raised.  Tensors must be contiguous CUDA tensors in
the ABI layouts (image ``[ny][nx][nz]`` fp32, sinogram ``[count][ns][nt]`` fp32,
mask uint8) on the geometry's device; work is enqueued on torch's current stream.

Module-level functions carry the ABI names (``ct_fwd_proj`` ...); ``Geometry`` and
``OSLALM`` are convenience wrappers that own the handles and workspaces.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CT_OSLALM_LIB", os.path.join(_HERE, "libct_oslalm.so"))   # override: tuning experiments only

CT_FAN2D, CT_CONE_AXIAL, CT_CONE_HELICAL = 0, 1, 2
KIND = {"fan2d": CT_FAN2D, "cone_axial": CT_CONE_AXIAL, "cone_helical": CT_CONE_HELICAL}
STATUS = {0: "CT_OK", 1: "CT_EINVAL", 2: "CT_EUNSUPPORTED", 3: "CT_ENOMEM", 4: "CT_ECUDA", 5: "CT_ENCCL",
          6: "CT_ESTATE"}

# Symbols declared in include/ct_oslalm.h (checked by tests/test_abi.py)
EXPORTS = ("ct_geom_create", "ct_geom_destroy", "ct_last_error", "ct_fwd_proj", "ct_back_proj",
           "ct_sqs_denom_scratch_bytes", "ct_sqs_denom", "ct_reg_grad", "ct_count_vv", "ct_oslalm_state_bytes",
           "ct_oslalm_state_create", "ct_fbp", "ct_fbp_scratch_bytes", "ct_peak_l2_read", "ct_oslalm_state_destroy", "ct_oslalm_state_get", "ct_oslalm_state_reset",
           "ct_oslalm_set_timing", "ct_oslalm_get_timing", "ct_oslalm_iter",
           "ct_oslalm_run", "ct_comm_init", "ct_comm_init_zslab", "ct_comm_init_virtual", "ct_comm_set_exchange", "ct_comm_get_unique_id", "ct_build_info", "ct_kernel_launches")


class CTError(RuntimeError):
    pass


class ct_geom_desc(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("nx", ctypes.c_int), ("ny", ctypes.c_int), ("nz", ctypes.c_int),
                ("dx", ctypes.c_double), ("dy", ctypes.c_double), ("dz", ctypes.c_double),
                ("offx", ctypes.c_double), ("offy", ctypes.c_double), ("offz", ctypes.c_double),
                ("ns", ctypes.c_int), ("nt", ctypes.c_int), ("ds", ctypes.c_double), ("dt", ctypes.c_double),
                ("offs", ctypes.c_double), ("offt", ctypes.c_double), ("dso", ctypes.c_double),
                ("dsd", ctypes.c_double), ("na", ctypes.c_int), ("orbit_deg", ctypes.c_double),
                ("orbit_start_deg", ctypes.c_double), ("pitch", ctypes.c_double), ("device", ctypes.c_int)]


class ct_views(ctypes.Structure):
    _fields_ = [("first", ctypes.c_int), ("stride", ctypes.c_int), ("count", ctypes.c_int)]


class ct_reg(ctypes.Structure):
    _fields_ = [("beta", ctypes.c_double), ("delta", ctypes.c_double), ("nbr", ctypes.c_int)]


class ct_oslalm_cfg(ctypes.Structure):
    _fields_ = [("M", ctypes.c_int), ("mode", ctypes.c_int), ("rho_fixed", ctypes.c_double),
                ("rho_min", ctypes.c_double), ("n_inner", ctypes.c_int), ("inner", ctypes.c_int), ("reg", ct_reg),
                ("bb", ctypes.c_int), ("alpha_min", ctypes.c_double)]


class ct_oslalm_data(ctypes.Structure):
    _fields_ = [("y", ctypes.c_void_p), ("w", ctypes.c_void_p), ("dl", ctypes.c_void_p), ("mask", ctypes.c_void_p)]


class ct_oslalm_log(ctypes.Structure):
    _fields_ = [("rho", ctypes.POINTER(ctypes.c_double)), ("xi", ctypes.POINTER(ctypes.c_double)),
                ("restart", ctypes.POINTER(ctypes.c_int)), ("capacity", ctypes.c_int), ("count", ctypes.c_int)]


class ct_oslalm_state_view(ctypes.Structure):
    _fields_ = [("g", ctypes.c_void_p), ("G", ctypes.c_void_p), ("rho", ctypes.c_void_p), ("l", ctypes.c_void_p),
                ("step", ctypes.c_void_p), ("initialised", ctypes.c_int), ("alpha", ctypes.c_void_p)]


_lib = None


def load():
    """Load the in-tree library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise CTError(f"{LIB_PATH} not built: run `python -m paper_1402_4381_b200.build` (no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER
    vp, i, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    L.ct_geom_create.argtypes = [P(ct_geom_desc), P(vp)]
    L.ct_geom_destroy.argtypes = [vp]; L.ct_geom_destroy.restype = None
    L.ct_last_error.restype = ctypes.c_char_p
    L.ct_build_info.restype = ctypes.c_char_p
    L.ct_kernel_launches.restype = ctypes.c_ulonglong
    L.ct_fwd_proj.argtypes = [vp, ct_views, vp, vp, vp]
    L.ct_back_proj.argtypes = [vp, ct_views, vp, vp, i, vp]
    L.ct_sqs_denom_scratch_bytes.argtypes = [vp, P(sz)]
    L.ct_sqs_denom.argtypes = [vp, vp, vp, vp, vp, vp]
    L.ct_reg_grad.argtypes = [vp, P(ct_reg), vp, vp, vp, vp, vp]
    L.ct_count_vv.argtypes = [vp, ct_views, vp, vp, P(ctypes.c_longlong), vp]
    L.ct_oslalm_state_bytes.argtypes = [vp, P(ct_oslalm_cfg), P(sz)]
    L.ct_oslalm_state_create.argtypes = [vp, P(ct_oslalm_cfg), vp, sz, P(vp)]
    L.ct_oslalm_state_destroy.argtypes = [vp]; L.ct_oslalm_state_destroy.restype = None
    L.ct_oslalm_state_get.argtypes = [vp, P(ct_oslalm_state_view)]
    L.ct_fbp_scratch_bytes.argtypes = [vp, P(ctypes.c_size_t)]
    L.ct_fbp.argtypes = [vp, vp, vp, vp, vp]
    L.ct_peak_l2_read.argtypes = [i, ctypes.c_size_t, i, P(ctypes.c_double)]
    L.ct_oslalm_state_reset.argtypes = [vp]
    L.ct_oslalm_set_timing.argtypes = [vp, i]
    L.ct_oslalm_get_timing.argtypes = [vp, P(ctypes.c_double), P(ctypes.c_longlong)]
    L.ct_oslalm_iter.argtypes = [vp, P(ct_oslalm_cfg), P(ct_oslalm_data), vp, vp, vp]
    L.ct_oslalm_run.argtypes = [vp, P(ct_oslalm_cfg), P(ct_oslalm_data), vp, vp, i, P(ct_oslalm_log), vp]
    L.ct_comm_init.argtypes = [vp, i, i, vp]
    L.ct_comm_init_zslab.argtypes = [vp, i, i, vp]
    L.ct_comm_init_virtual.argtypes = [P(vp), i, i]
    L.ct_comm_set_exchange.argtypes = [vp, i]
    L.ct_comm_get_unique_id.argtypes = [vp]
    _check_provenance(L)
    _lib = L
    return L


def _check_provenance(L):
    """The library must have been built from the sources next to it (source hash compiled
    into ct_build_info), so a GPU run provably uses the HEAD build.  Tuning variants loaded
    through CT_OSLALM_LIB are exempt."""
    if "CT_OSLALM_LIB" in os.environ:
        return
    from . import build as _b
    info = L.ct_build_info().decode()
    want = _b.source_hash()
    if f"src={want}" not in info:
        raise CTError(f"{LIB_PATH} is stale ({info.split('src=')[-1]} != sources {want}): "
                      f"rebuild with `python -m paper_1402_4381_b200.build`")


def _check(rc):
    if rc != 0:
        msg = _lib.ct_last_error().decode(errors="replace")
        raise CTError(f"{STATUS.get(rc, rc)}: {msg}")


def _stream(stream=None, h=None):
    """The caller's stream (default: the current stream of the geometry's device)."""
    s = (torch.cuda.current_stream(_dev(h)) if h is not None and _dev(h) is not None else torch.cuda.current_stream()) \
        if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t, dtype, name, numel=None):
    """Device pointer of a contiguous CUDA tensor; `numel`: the element count the call reads or
    writes through it (the C ABI takes bare pointers, so sizes are checked here)."""
    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise CTError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise CTError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise CTError(f"{name} must be contiguous")
    if numel is not None and t.numel() < numel:
        raise CTError(f"{name} has {t.numel()} elements, the call needs {numel}")
    return ctypes.c_void_p(t.data_ptr())


# element counts per geometry handle (image, cells per view, views), for the size checks
_SIZES = {}


def _img(h):
    return _SIZES[h.value][0] if h.value in _SIZES else None


def _cells(h, count):
    return _SIZES[h.value][1] * count if h.value in _SIZES else None


def _na(h):
    return _SIZES[h.value][2] if h.value in _SIZES else 0


def _dev(h):
    return _SIZES[h.value][3] if h is not None and h.value in _SIZES else None


def _on_dev(h, *tensors):
    """Every tensor handed to a call on geometry h must live on h's device (the C ABI takes
    bare pointers and launches on the geometry's device)."""
    d = _dev(h)
    if d is None:
        return
    for t in tensors:
        if isinstance(t, torch.Tensor) and t.is_cuda and t.device.index != d:
            raise CTError(f"tensor on cuda:{t.device.index}, geometry on cuda:{d}")

# ---------------------------------------------------------------------------
# ABI-named functions (marshalling only)
# ---------------------------------------------------------------------------

def ct_geom_create(geom: dict, device: int = 0):
    L = load()
    d = ct_geom_desc()
    d.kind = KIND[geom["kind"]]
    for k in ("nx", "ny", "nz", "ns", "nt", "na"):
        setattr(d, k, int(geom[k]))
    for k in ("dx", "dy", "dz", "offx", "offy", "offz", "ds", "dt", "offs", "offt", "dso", "dsd",
              "orbit_deg", "orbit_start_deg", "pitch"):
        setattr(d, k, float(geom.get(k, 0.0)))
    d.device = int(device)
    h = ctypes.c_void_p()
    _check(L.ct_geom_create(ctypes.byref(d), ctypes.byref(h)))
    is2d = geom["kind"] == "fan2d"
    _SIZES[h.value] = (int(geom["nx"]) * int(geom["ny"]) * (1 if is2d else int(geom["nz"])),
                       int(geom["ns"]) * (1 if is2d else int(geom["nt"])), int(geom["na"]), int(device))
    return h


def ct_geom_destroy(h):
    _SIZES.pop(h.value, None)
    load().ct_geom_destroy(h)


def ct_fwd_proj(h, views, x, y, stream=None):
    _on_dev(h, x, y)
    _check(load().ct_fwd_proj(h, ct_views(*views), _ptr(x, torch.float32, "x", _img(h)),
                              _ptr(y, torch.float32, "y", _cells(h, views[2])), _stream(stream, h)))


def ct_peak_l2_read(device=0, mib=48, reps=200):
    """L2-resident read bandwidth (GB/s) of the device (diagnostic)."""
    v = ctypes.c_double()
    _check(load().ct_peak_l2_read(int(device), int(mib) * 1024 * 1024, int(reps), ctypes.byref(v)))
    return v.value


def ct_fbp_scratch_bytes(h):
    n = ctypes.c_size_t()
    _check(load().ct_fbp_scratch_bytes(h, ctypes.byref(n)))
    return n.value


def ct_fbp(h, y, x, scratch, stream=None):
    _on_dev(h, y, x, scratch)
    _check(load().ct_fbp(h, _ptr(y, torch.float32, "y", _cells(h, _na(h))), _ptr(x, torch.float32, "x", _img(h)),
                         _ptr(scratch, torch.uint8, "scratch", ct_fbp_scratch_bytes(h)), _stream(stream, h)))


def ct_back_proj(h, views, y, x, accumulate=False, stream=None):
    _on_dev(h, y, x)
    _check(load().ct_back_proj(h, ct_views(*views), _ptr(y, torch.float32, "y", _cells(h, views[2])),
                               _ptr(x, torch.float32, "x", _img(h)), 1 if accumulate else 0, _stream(stream, h)))


def ct_sqs_denom_scratch_bytes(h):
    n = ctypes.c_size_t()
    _check(load().ct_sqs_denom_scratch_bytes(h, ctypes.byref(n)))
    return n.value


def ct_sqs_denom(h, w, mask, dl, scratch, stream=None):
    _on_dev(h, w, mask, dl, scratch)
    _check(load().ct_sqs_denom(h, _ptr(w, torch.float32, "w", _cells(h, _na(h))), _ptr(mask, torch.uint8, "mask", _img(h)),
                               _ptr(dl, torch.float32, "dl", _img(h)),
                               _ptr(scratch, torch.uint8, "scratch", ct_sqs_denom_scratch_bytes(h)), _stream(stream, h)))


def ct_reg_grad(h, reg, mask, x, grad, curv=None, stream=None):
    _on_dev(h, mask, x, grad, curv)
    r = ct_reg(float(reg[0]), float(reg[1]), int(reg[2]))
    n = _img(h)
    _check(load().ct_reg_grad(h, ctypes.byref(r), _ptr(mask, torch.uint8, "mask", n), _ptr(x, torch.float32, "x", n),
                              _ptr(grad, torch.float32, "grad", n), _ptr(curv, torch.float32, "curv", n),
                              _stream(stream, h)))


def ct_count_vv(h, views, mask, scratch, stream=None):
    _on_dev(h, mask, scratch)
    """Returns (U, nnz, C) of the view list (see the header)."""
    out = (ctypes.c_longlong * 3)()
    _check(load().ct_count_vv(h, ct_views(*views), _ptr(mask, torch.uint8, "mask", _img(h)),
                              _ptr(scratch, torch.uint8, "scratch"), out, _stream(stream, h)))
    return tuple(int(v) for v in out)


def ct_kernel_launches() -> int:
    return int(load().ct_kernel_launches())


def ct_build_info() -> str:
    return load().ct_build_info().decode()


def ct_comm_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load().ct_comm_get_unique_id(buf))
    return buf.raw


def ct_comm_init(h, rank, nranks, uid: bytes, zslab=False):
    buf = ctypes.create_string_buffer(bytes(uid), 128)
    f = load().ct_comm_init_zslab if zslab else load().ct_comm_init
    _check(f(h, int(rank), int(nranks), buf))


EXCHANGE = {"auto": 0, "full": 1, "band": 2}


def ct_comm_set_exchange(h, mode="auto"):
    """Row-slab multi-rank exchange: "full" (reduce-scatter / all-gather), "band" (z-band blocks,
    helical) or "auto" (band for helical scans)."""
    _check(load().ct_comm_set_exchange(h, EXCHANGE[mode]))


def ct_comm_init_virtual(handles, zslab=False):
    """Attach len(handles) geometry handles of one device as virtual ranks 0..P-1 (validation
    of the multi-rank path on one GPU; each rank must then be driven by its own thread)."""
    arr = (ctypes.c_void_p * len(handles))(*[h.value for h in handles])
    _check(load().ct_comm_init_virtual(arr, len(handles), 1 if zslab else 0))


# ---------------------------------------------------------------------------
# Convenience wrappers
# ---------------------------------------------------------------------------

class Geometry:
    """Owns a ct_geom handle; image/sinogram shapes follow the ABI layouts."""

    def __init__(self, geom: dict, device: int = 0):
        self.geom = dict(geom)
        self.device = torch.device("cuda", device)
        self.h = ct_geom_create(geom, device)
        self.is2d = geom["kind"] == "fan2d"
        self.nz = 1 if self.is2d else int(geom["nz"])
        self.nt = 1 if self.is2d else int(geom["nt"])
        self.img_shape = (int(geom["ny"]), int(geom["nx"]), self.nz)
        self.na = int(geom["na"])
        self.rank, self.nranks = 0, 1

    def __del__(self):
        try:
            if getattr(self, "h", None):
                ct_geom_destroy(self.h)
        except Exception:
            pass

    def sino_shape(self, count):
        return (count, int(self.geom["ns"]), self.nt)

    def views(self, first=0, stride=1, count=None):
        if count is None:
            count = (self.na - first + stride - 1) // stride
        return (first, stride, count)

    def fwd(self, x, views=None, out=None):
        v = views or self.views()
        if out is None:
            out = torch.empty(self.sino_shape(v[2]), dtype=torch.float32, device=self.device)
        ct_fwd_proj(self.h, v, x, out)
        return out

    def back(self, y, views=None, out=None, accumulate=False):
        v = views or self.views()
        if out is None:
            out = torch.zeros(self.img_shape, dtype=torch.float32, device=self.device)
        ct_back_proj(self.h, v, y, out, accumulate)
        return out

    def sqs_denom(self, w, mask):
        mask = mask.clone()
        dl = torch.empty(self.img_shape, dtype=torch.float32, device=self.device)
        scratch = torch.empty(ct_sqs_denom_scratch_bytes(self.h), dtype=torch.uint8, device=self.device)
        ct_sqs_denom(self.h, w, mask, dl, scratch)
        return dl, mask

    def fbp(self, y, stream=None):
        """FBP / FDK initial image (NEXT-4) of the ABI-layout sinogram y [na][ns][nt]."""
        L = load()
        n = ctypes.c_size_t()
        _check(L.ct_fbp_scratch_bytes(self.h, ctypes.byref(n)))
        scratch = torch.empty(n.value, dtype=torch.uint8, device=self.device)
        x = torch.empty(self.img_shape, dtype=torch.float32, device=self.device)
        _check(L.ct_fbp(self.h, _ptr(y, torch.float32, "y", _cells(self.h, self.na)), _ptr(x, torch.float32, "x"),
                        ctypes.c_void_p(scratch.data_ptr()), _stream(stream, self.h)))
        return x

    def reg_grad(self, x, mask, beta, delta, nbr, want_curv=True):
        grad = torch.empty_like(x)
        curv = torch.empty_like(x) if want_curv else None
        ct_reg_grad(self.h, (beta, delta, nbr), mask, x, grad, curv)
        return grad, curv

    def count_vv(self, mask, views=None):
        """U (voxel-view pairs with a non-empty footprint) of the view list."""
        return self.counts(mask, views)[0]

    def counts(self, mask, views=None):
        """(U, nnz, C) of the view list."""
        scratch = torch.zeros(32, dtype=torch.uint8, device=self.device)
        return ct_count_vv(self.h, views or self.views(), mask, scratch)

    @staticmethod
    def comm_init_virtual(geos, zslab=False):
        """geos[r] becomes virtual rank r of len(geos) (one device, one host thread per rank)."""
        ct_comm_init_virtual([g.h for g in geos], zslab)
        for r, g in enumerate(geos):
            g.rank, g.nranks = r, len(geos)

    def comm_init(self, rank, nranks, uid, zslab=False):
        """Attach an NCCL communicator.  zslab=True: this geometry is rank `rank`'s z-slab of the
        volume (host.rank_zslab / inputs.slab_geom), partial sinograms are summed (NEXT-3)."""
        ct_comm_init(self.h, rank, nranks, uid, zslab)
        self.rank, self.nranks = rank, nranks


class OSLALM:
    """OS-LALM solver state over a caller-owned (torch) device workspace."""

    def __init__(self, geo: Geometry, M, *, mode="continuation", rho_fixed=1.0, rho_min=1e-3, beta, delta, nbr,
                 n_inner=1, inner="sqs", bb=False, alpha_min=1e-6):
        self.geo = geo
        self.cfg = ct_oslalm_cfg(int(M), 1 if mode == "continuation" else 0, float(rho_fixed), float(rho_min),
                                 int(n_inner), 0 if inner == "sqs" else 1, ct_reg(float(beta), float(delta), int(nbr)),
                                 1 if bb else 0, float(alpha_min))
        L = load()
        n = ctypes.c_size_t()
        _check(L.ct_oslalm_state_bytes(geo.h, ctypes.byref(self.cfg), ctypes.byref(n)))
        self.workspace = torch.empty(n.value + 256, dtype=torch.uint8, device=geo.device)
        base = self.workspace.data_ptr()
        off = (-base) % 256
        self.h = ctypes.c_void_p()
        _check(L.ct_oslalm_state_create(geo.h, ctypes.byref(self.cfg), ctypes.c_void_p(base + off), n.value,
                                        ctypes.byref(self.h)))
        self._data = None

    def __del__(self):
        try:
            if getattr(self, "h", None):
                load().ct_oslalm_state_destroy(self.h)
        except Exception:
            pass

    def set_data(self, y, w, dl, mask):
        _on_dev(self.geo.h, y, w, dl, mask)
        self._keep = (y, w, dl, mask)
        h, na = self.geo.h, self.geo.na
        self._data = ct_oslalm_data(_ptr(y, torch.float32, "y", _cells(h, na)), _ptr(w, torch.float32, "w", _cells(h, na)),
                                    _ptr(dl, torch.float32, "dl", _img(h)), _ptr(mask, torch.uint8, "mask", _img(h)))

    def iterate(self, x, stream=None):
        _on_dev(self.geo.h, x)
        _check(load().ct_oslalm_iter(self.geo.h, ctypes.byref(self.cfg), ctypes.byref(self._data), self.h,
                                     _ptr(x, torch.float32, "x", _img(self.geo.h)), _stream(stream, self.geo.h)))

    def reset(self):
        _check(load().ct_oslalm_state_reset(self.h))

    def set_timing(self, enable=True):
        _check(load().ct_oslalm_set_timing(self.h, 1 if enable else 0))

    def timing(self):
        """{class: (total ms, launches)} for sqs_update, fwd, back, finalize, exchange."""
        ms = (ctypes.c_double * 5)(); n = (ctypes.c_longlong * 5)()
        _check(load().ct_oslalm_get_timing(self.h, ms, n))
        names = ("sqs_update", "fwd_resid", "back_gupd", "xi_finalize", "exchange")
        return {names[i]: (ms[i], n[i]) for i in range(5)}

    def run(self, x, n_iter, log=False, stream=None):
        _on_dev(self.geo.h, x)
        L = load()
        lg = None
        if log:
            cap = n_iter * self.cfg.M
            rho = (ctypes.c_double * cap)(); xi = (ctypes.c_double * cap)(); rs = (ctypes.c_int * cap)()
            lg = ct_oslalm_log(rho, xi, rs, cap, 0)
        _check(L.ct_oslalm_run(self.geo.h, ctypes.byref(self.cfg), ctypes.byref(self._data), self.h,
                               _ptr(x, torch.float32, "x", _img(self.geo.h)), int(n_iter), ctypes.byref(lg) if lg else None,
                               _stream(stream, self.geo.h)))
        if log:
            n = lg.count
            return [(rho[i], xi[i], rs[i]) for i in range(n)]
        return None

    def state(self):
        v = ct_oslalm_state_view()
        _check(load().ct_oslalm_state_get(self.h, ctypes.byref(v)))
        return v

    def _ws_view(self, ptr, n, dtype):
        off = ptr - self.workspace.data_ptr()
        nb = n * torch.empty((), dtype=dtype).element_size()
        return self.workspace[off:off + nb].view(dtype)

    def split_gradient(self):
        """The split gradient g as a tensor view of the workspace ([ny][nx][nz])."""
        n = self.geo.img_shape[0] * self.geo.img_shape[1] * self.geo.img_shape[2]
        return self._ws_view(self.state().g, n, torch.float32).view(self.geo.img_shape)

    def subset_gradient(self):
        n = self.geo.img_shape[0] * self.geo.img_shape[1] * self.geo.img_shape[2]
        return self._ws_view(self.state().G, n, torch.float32).view(self.geo.img_shape)

    def scalars(self):
        """(rho for the next step, continuation counter l, inner steps taken)."""
        v = self.state()
        rho = self._ws_view(v.rho, 1, torch.float64).item()
        l = self._ws_view(v.l, 1, torch.int64).item()
        st = self._ws_view(v.step, 1, torch.int64).item()
        return rho, l, st

    def alpha(self):
        """Barzilai-Borwein scale alpha used by the next outer iteration (1.0 without BB)."""
        return self._ws_view(self.state().alpha, 1, torch.float64).item()
