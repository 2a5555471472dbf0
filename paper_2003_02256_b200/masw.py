"""Thin ctypes binding of libmasw.so (include/masw.h): argument marshalling only.

Every entry point keeps the C name.  Inputs may be numpy arrays (host path: the library
stages them to the device) or torch tensors (CUDA tensors take the device path on the
current torch stream; CPU tensors take the host path).  Outputs are allocated like the
inputs unless given.  There is no CPU fallback: if libmasw.so is missing or CUDA is not
usable the calls raise.
"""
from __future__ import annotations

import ctypes
import os
from typing import NamedTuple, Optional

import numpy as np

from . import build as _build

LIB_PATH = os.environ.get("MASW_LIB", _build.LIB)   # MASW_LIB: variant builds (experiments)

OK, WARN_NO_SIGN_CHANGE = 0, 1
E_ARG, E_MODEL, E_GRID, E_RANGE, E_NONFINITE, E_CUDA, E_NOMEM = -1, -2, -3, -4, -5, -6, -7
IDX_NO_CHANGE, IDX_NONFINITE = -1, -2
ASYNC, TIME_SCAN = 0x1, 0x2
SCHED_CONTIGUOUS, SCHED_MODULAR, TEAM_STATS = 0x4, 0x8, 0x10
SCHED_ROWS, SCHED_MODELS = 0x20, 0x40   # force the row / model-major scan kernel
STABLE = 0x80   # cancellation-free, exponentially scaled element (f3), k h <= 700
PIVOTED = 0x100   # every scan sign by the banded GEPP (validation / A-B)
SCHED_PAIRS = 0x200   # force the pair scan (one model: two wavelengths per warp in lockstep)
DIRECT = 0x400   # no small-c prefix: the direct element everywhere (reading S15''; A/B only)
MAX_LAYERS = 64


class MaswError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        msg = _strerror(code)
        if code == E_CUDA:
            msg += f" ({lib().masw_last_cuda_error().decode()})"
        super().__init__(f"{where}: {msg}")


class _Model(ctypes.Structure):
    _fields_ = [("n_layers", ctypes.c_int32), ("h", ctypes.c_void_p), ("alpha", ctypes.c_void_p),
                ("beta", ctypes.c_void_p), ("rho", ctypes.c_void_p)]


class _Ensemble(ctypes.Structure):
    _fields_ = [("n_models", ctypes.c_int64), ("n_layers", ctypes.c_int32),
                ("h", ctypes.c_void_p), ("alpha", ctypes.c_void_p), ("beta", ctypes.c_void_p),
                ("rho", ctypes.c_void_p)]


class _Exec(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("cuda_stream", ctypes.c_void_p),
                ("team_warps", ctypes.c_int32), ("flags", ctypes.c_uint32)]


_lib = None
_P = ctypes.c_void_p
_I64 = ctypes.c_int64


def lib():
    """Load libmasw.so (built in-tree by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; "
                              "g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
        L = ctypes.CDLL(LIB_PATH)
        L.masw_curve.argtypes = [ctypes.POINTER(_Model), _P, _I64, _P, _I64, _P, _P,
                                 ctypes.POINTER(_Exec)]
        L.masw_curves_ensemble.argtypes = [ctypes.POINTER(_Ensemble), _P, _I64, _P, _I64, _P, _P,
                                           _P, _P, ctypes.POINTER(_Exec)]
        L.masw_misfit.argtypes = [_P, _P, _I64, _P, ctypes.POINTER(_Exec)]
        L.masw_misfit_batch.argtypes = [_P, _P, _I64, _I64, _P, ctypes.POINTER(_Exec)]
        L.masw_argmin.argtypes = [_P, _I64, _P, _P, ctypes.POINTER(_Exec)]
        L.masw_det_grid.argtypes = [ctypes.POINTER(_Model), _P, _I64, _P, _I64, _P, _P, _P,
                                    ctypes.POINTER(_Exec)]
        L.masw_strerror.restype = ctypes.c_char_p
        L.masw_strerror.argtypes = [ctypes.c_int]
        L.masw_last_cuda_error.restype = ctypes.c_char_p
        L.masw_kernel_launches.restype = ctypes.c_int64
        L.masw_last_scan_ms.restype = ctypes.c_double
        L.masw_last_team_dets.restype = ctypes.c_int64
        L.masw_last_team_dets.argtypes = [ctypes.POINTER(ctypes.c_int64), ctypes.c_int64]
        L.masw_recent_scan_ms.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int32]
        L.masw_last_work.argtypes = [ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
        L.masw_last_fallbacks.restype = ctypes.c_int64
        L.masw_last_fallbacks.argtypes = []
        L.masw_last_prefix.argtypes = [ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
        L.masw_probe_fp64_peak.argtypes = [ctypes.c_int32, ctypes.c_double,
                                           ctypes.POINTER(ctypes.c_double),
                                           ctypes.POINTER(ctypes.c_double)]
        _lib = L
    return _lib


def _strerror(code: int) -> str:
    return lib().masw_strerror(int(code)).decode()


# ------------------------------------------------------------------ marshalling helpers

def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


class _Buf:
    """A contiguous fp64/int32/int64 buffer and its raw pointer (keeps a reference alive)."""

    def __init__(self, x, dtype):
        self.obj = x
        if _is_torch(x):
            import torch

            tdt = {np.float64: torch.float64, np.int32: torch.int32, np.int64: torch.int64}[dtype]
            if x.dtype != tdt or not x.is_contiguous():
                x = x.to(tdt).contiguous()
            self.obj = x
            self.ptr = x.data_ptr()
            self.cuda = x.is_cuda
            self.device = x.device.index if x.is_cuda else -1
        else:
            x = np.ascontiguousarray(x, dtype=dtype)
            self.obj = x
            self.ptr = x.ctypes.data
            self.cuda = False
            self.device = -1


def _empty_like_kind(ref: _Buf, shape, dtype, fill=None):
    if ref.cuda:
        import torch

        tdt = {np.float64: torch.float64, np.int32: torch.int32, np.int64: torch.int64}[dtype]
        t = torch.empty(shape, dtype=tdt, device=f"cuda:{ref.device}")
        if fill is not None:
            t.fill_(fill)
        return t
    a = np.empty(shape, dtype=dtype)
    if fill is not None:
        a.fill(fill)
    return a


def _exec(ref: _Buf, team_warps=0, flags=0, stream=None, device=None) -> _Exec:
    if ref.cuda and stream is None:
        import torch

        stream = torch.cuda.current_stream(ref.device).cuda_stream
    dev = ref.device if device is None else device
    return _Exec(int(dev), ctypes.c_void_p(stream or 0), int(team_warps), int(flags))


def _check(code: int, where: str) -> int:
    if code < 0:
        raise MaswError(code, where)
    return code


class Curve(NamedTuple):
    status: int
    ct: object
    idx: object


class EnsembleResult(NamedTuple):
    status: int
    ct: object
    idx: object
    misfit: object


# ------------------------------------------------------------------ entry points

def masw_curve(h, alpha, beta, rho, lam, c, *, team_warps=0, flags=0, stream=None,
               ct_out=None, idx_out=None) -> Curve:
    """C_t of one model (Algorithm 1) → Curve(status, ct[L], idx[L])."""
    bh, ba, bb, br = (_Buf(x, np.float64) for x in (h, alpha, beta, rho))
    bl, bc = _Buf(lam, np.float64), _Buf(c, np.float64)
    L, V = len(bl.obj), len(bc.obj)
    ct = ct_out if ct_out is not None else _empty_like_kind(bl, (L,), np.float64)
    idx = idx_out if idx_out is not None else _empty_like_kind(bl, (L,), np.int32)
    bct, bidx = _Buf(ct, np.float64), _Buf(idx, np.int32)
    mod = _Model(len(bh.obj), bh.ptr, ba.ptr, bb.ptr, br.ptr)
    ex = _exec(bl, team_warps, flags, stream)
    st = lib().masw_curve(ctypes.byref(mod), bl.ptr, L, bc.ptr, V, bct.ptr, bidx.ptr,
                          ctypes.byref(ex))
    return Curve(_check(st, "masw_curve"), bct.obj, bidx.obj)


def masw_curves_ensemble(h, alpha, beta, rho, lam, c, ce=None, *, team_warps=0, flags=0,
                         stream=None, ct_out=None, idx_out=None, misfit_out=None,
                         want_idx=True) -> EnsembleResult:
    """C_t[M][L], idx[M][L] and misfit[M] of M models against C_e."""
    bh, ba, bb, br = (_Buf(x, np.float64) for x in (h, alpha, beta, rho))
    bl, bc = _Buf(lam, np.float64), _Buf(c, np.float64)
    M, N = bh.obj.shape
    L, V = len(bl.obj), len(bc.obj)
    bce = _Buf(ce, np.float64) if ce is not None else None
    ct = ct_out if ct_out is not None else _empty_like_kind(bl, (M, L), np.float64)
    bct = _Buf(ct, np.float64)
    bidx = None
    if want_idx or idx_out is not None:
        idx = idx_out if idx_out is not None else _empty_like_kind(bl, (M, L), np.int32)
        bidx = _Buf(idx, np.int32)
    bmis = None
    if bce is not None:
        mis = misfit_out if misfit_out is not None else _empty_like_kind(bl, (M,), np.float64)
        bmis = _Buf(mis, np.float64)
    ens = _Ensemble(M, N, bh.ptr, ba.ptr, bb.ptr, br.ptr)
    ex = _exec(bl, team_warps, flags, stream)
    st = lib().masw_curves_ensemble(ctypes.byref(ens), bl.ptr, L, bc.ptr, V,
                                    bce.ptr if bce else None, bct.ptr,
                                    bidx.ptr if bidx else None, bmis.ptr if bmis else None,
                                    ctypes.byref(ex))
    return EnsembleResult(_check(st, "masw_curves_ensemble"), bct.obj,
                          bidx.obj if bidx else None, bmis.obj if bmis else None)


def masw_misfit(ct, ce, *, stream=None) -> float:
    """Algorithm 2 of one curve."""
    bct, bce = _Buf(ct, np.float64), _Buf(ce, np.float64)
    out = _empty_like_kind(bct, (1,), np.float64)
    bo = _Buf(out, np.float64)
    ex = _exec(bct, 0, 0, stream)
    _check(lib().masw_misfit(bct.ptr, bce.ptr, len(bct.obj), bo.ptr, ctypes.byref(ex)),
           "masw_misfit")
    return float(bo.obj[0])


def masw_misfit_batch(ct, ce, *, stream=None, misfit_out=None):
    bct, bce = _Buf(ct, np.float64), _Buf(ce, np.float64)
    M, L = bct.obj.shape
    out = misfit_out if misfit_out is not None else _empty_like_kind(bct, (M,), np.float64)
    bo = _Buf(out, np.float64)
    ex = _exec(bct, 0, 0, stream)
    _check(lib().masw_misfit_batch(bct.ptr, bce.ptr, M, L, bo.ptr, ctypes.byref(ex)),
           "masw_misfit_batch")
    return bo.obj


def masw_argmin(misfit, *, stream=None, flags=0):
    """(best index, best misfit), ties → lowest index."""
    bm = _Buf(misfit, np.float64)
    b = _empty_like_kind(bm, (1,), np.int64)
    v = _empty_like_kind(bm, (1,), np.float64)
    bb, bv = _Buf(b, np.int64), _Buf(v, np.float64)
    ex = _exec(bm, 0, flags, stream)
    _check(lib().masw_argmin(bm.ptr, len(bm.obj), bb.ptr, bv.ptr, ctypes.byref(ex)),
           "masw_argmin")
    return bb.obj, bv.obj


def masw_det_grid(h, alpha, beta, rho, lam, c, *, flags=0, stream=None):
    """Full (λ, c) determinant grid (debug/parity) → (mant re [L][V], mant im, exp2 [L][V]).
    flags=STABLE evaluates the cancellation-free, exponentially scaled element (f3)."""
    bh, ba, bb, br = (_Buf(x, np.float64) for x in (h, alpha, beta, rho))
    bl, bc = _Buf(lam, np.float64), _Buf(c, np.float64)
    L, V = len(bl.obj), len(bc.obj)
    re = _Buf(_empty_like_kind(bl, (L, V), np.float64), np.float64)
    im = _Buf(_empty_like_kind(bl, (L, V), np.float64), np.float64)
    ex2 = _Buf(_empty_like_kind(bl, (L, V), np.int32), np.int32)
    mod = _Model(len(bh.obj), bh.ptr, ba.ptr, bb.ptr, br.ptr)
    ex = _exec(bl, 0, flags, stream)
    _check(lib().masw_det_grid(ctypes.byref(mod), bl.ptr, L, bc.ptr, V, re.ptr, im.ptr,
                               ex2.ptr, ctypes.byref(ex)), "masw_det_grid")
    return re.obj, im.obj, ex2.obj


def masw_kernel_launches() -> int:
    return int(lib().masw_kernel_launches())


def masw_last_scan_ms() -> float:
    return float(lib().masw_last_scan_ms())


def masw_recent_scan_ms(n: int):
    """Scan-kernel device times (ms) of the last n MASW_TIME_SCAN launches, oldest first."""
    buf = (ctypes.c_double * max(n, 1))()
    k = lib().masw_recent_scan_ms(buf, n)
    return [buf[i] for i in range(max(k, 0))]


def masw_last_team_dets():
    """Per-team algorithmic det counts of the last MASW_TEAM_STATS call (numpy int64)."""
    n = int(lib().masw_last_team_dets(None, 0))
    if n < 0:
        return None
    out = np.zeros(n, dtype=np.int64)
    lib().masw_last_team_dets(out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), n)
    return out


def masw_last_fallbacks() -> int:
    """Determinants of the last synchronous scan re-evaluated with partial pivoting."""
    return int(lib().masw_last_fallbacks())


def masw_last_prefix():
    """(rows with a small-c prefix, dets evaluated there with the stable element) of the last
    synchronous call (reading S15''); (-1, -1) if none was recorded."""
    r, d = ctypes.c_int64(-1), ctypes.c_int64(-1)
    lib().masw_last_prefix(ctypes.byref(r), ctypes.byref(d))
    return int(r.value), int(d.value)


def masw_last_work():
    a, e = ctypes.c_int64(-1), ctypes.c_int64(-1)
    lib().masw_last_work(ctypes.byref(a), ctypes.byref(e))
    return int(a.value), int(e.value)


def masw_probe_fp64_peak(device: int = -1, target_ms: float = 200.0):
    tf, ms = ctypes.c_double(0), ctypes.c_double(0)
    _check(lib().masw_probe_fp64_peak(device, target_ms, ctypes.byref(tf), ctypes.byref(ms)),
           "masw_probe_fp64_peak")
    return tf.value, ms.value
