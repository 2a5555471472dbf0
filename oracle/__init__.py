"""ctypes binding of the CPU fp64 oracle (oracle/masw_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` leg / ``--impl reference`` arm.  The product package
(``paper_2003_02256_b200``) never imports this module, and this module never imports the
product.  Each function mirrors one oracle step and cites the
passage it follows in the C source.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "masw_oracle.c")
CORE = os.path.join(HERE, "masw_det_core.h")
LIB = os.path.join(HERE, "libmasw_oracle.so")

OK, WARN_NO_SIGN_CHANGE = 0, 1
E_ARG, E_MODEL, E_GRID, E_RANGE, E_NONFINITE = -1, -2, -3, -4, -5
IDX_NO_CHANGE, IDX_NONFINITE = -1, -2

_lock = threading.Lock()
_lib = None

_D = ctypes.POINTER(ctypes.c_double)
_I32 = ctypes.POINTER(ctypes.c_int32)
_I64 = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, no fast-math, no FMA contraction)."""
    if (force or not os.path.exists(LIB) or
            os.path.getmtime(LIB) < max(os.path.getmtime(SRC), os.path.getmtime(CORE))):
        cmd = ["gcc", "-std=gnu11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
               "-shared", "-pthread", "-o", LIB + ".tmp", SRC, "-lquadmath", "-lm"]
        subprocess.check_call(cmd)
        os.replace(LIB + ".tmp", LIB)
    return LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(LIB)
            L.oracle_wavenumber.restype = ctypes.c_double
            L.oracle_wavenumber.argtypes = [ctypes.c_double]
            L.oracle_perturb_velocity.restype = ctypes.c_double
            L.oracle_perturb_velocity.argtypes = [ctypes.c_int32, _D, _D, ctypes.c_double]
            L.oracle_validate_model.argtypes = [ctypes.c_int32, _D, _D, _D, _D]
            L.oracle_layer_element.argtypes = [ctypes.c_double] * 6 + [_D]
            L.oracle_layer_element.restype = None
            L.oracle_halfspace_element.argtypes = [ctypes.c_double] * 5 + [_D]
            L.oracle_halfspace_element.restype = None
            L.oracle_assemble.argtypes = [ctypes.c_int32, _D, _D, _D, _D, ctypes.c_double,
                                          ctypes.c_double, _D]
            L.oracle_assemble.restype = None
            L.oracle_det_dense.argtypes = [ctypes.c_int32, _D, _D, _I32]
            L.oracle_det.argtypes = [ctypes.c_int32, _D, _D, _D, _D, ctypes.c_double,
                                     ctypes.c_double, _D, _I32]
            L.oracle_det_ld.argtypes = L.oracle_det.argtypes
            L.oracle_det_fp64.argtypes = L.oracle_det.argtypes
            L.oracle_det_q.argtypes = L.oracle_det.argtypes
            L.oracle_fp64_error_bound.restype = ctypes.c_double
            L.oracle_fp64_error_bound.argtypes = [ctypes.c_int32, _D, _D, _D, ctypes.c_double,
                                                  ctypes.c_double]
            L.oracle_det_grid_ld.argtypes = [ctypes.c_int32, _D, _D, _D, _D, _D, ctypes.c_int64,
                                             _D, ctypes.c_int64, _D, _D, _I32, _I32,
                                             ctypes.c_int32]
            L.oracle_det_kappa.argtypes = [ctypes.c_int32, _D, _D, _D, _D, ctypes.c_double,
                                           ctypes.c_double, _D]
            L.oracle_det_grid_kappa.argtypes = [ctypes.c_int32, _D, _D, _D, _D, _D,
                                                ctypes.c_int64, _D, ctypes.c_int64, _D, _I32,
                                                ctypes.c_int32]
            L.oracle_curve.argtypes = [ctypes.c_int32, _D, _D, _D, _D, _D, ctypes.c_int64, _D,
                                       ctypes.c_int64, _D, _I32, _I64, ctypes.c_int32]
            L.oracle_misfit.argtypes = [_D, _D, ctypes.c_int64, _D]
            L.oracle_misfit_ld.argtypes = [_D, _D, ctypes.c_int64, _D]
            L.oracle_ensemble.argtypes = [ctypes.c_int64, ctypes.c_int32, _D, _D, _D, _D, _D,
                                          ctypes.c_int64, _D, ctypes.c_int64, _D, _D, _I32, _D,
                                          _I64, _I64, ctypes.c_int32]
            L.oracle_det_grid.argtypes = [ctypes.c_int32, _D, _D, _D, _D, _D, ctypes.c_int64, _D,
                                          ctypes.c_int64, _D, _D, _I32, _I32, ctypes.c_int32]
            _lib = L
    return _lib


def _d(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(_D)


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


# ---------------------------------------------------------------- steps O1..O6

def wavenumber(lam: float) -> float:
    """O1: k = 2π/λ (reading S2)."""
    return lib().oracle_wavenumber(float(lam))


def perturb_velocity(alpha, beta, c: float) -> float:
    """O2: MASWaves near-velocity perturbation (reading S4)."""
    a, pa = _d(alpha)
    b, pb = _d(beta)
    return lib().oracle_perturb_velocity(len(a) - 1, pa, pb, float(c))


def validate_model(h, alpha, beta, rho) -> int:
    """O0 for one model."""
    args = [_d(x) for x in (h, alpha, beta, rho)]
    return lib().oracle_validate_model(len(args[0][0]), *[p for _, p in args])


def layer_element(h, alpha, beta, rho, k, c) -> np.ndarray:
    """O3: complex 4×4 Kausel–Roësset layer element."""
    out = np.zeros(32)
    lib().oracle_layer_element(float(h), float(alpha), float(beta), float(rho), float(k),
                               float(c), out.ctypes.data_as(_D))
    return (out[0::2] + 1j * out[1::2]).reshape(4, 4)


def halfspace_element(alpha, beta, rho, k, c) -> np.ndarray:
    """O4: complex 2×2 half-space element."""
    out = np.zeros(8)
    lib().oracle_halfspace_element(float(alpha), float(beta), float(rho), float(k), float(c),
                                   out.ctypes.data_as(_D))
    return (out[0::2] + 1j * out[1::2]).reshape(2, 2)


def assemble(h, alpha, beta, rho, k, c) -> np.ndarray:
    """Dense global K of order 2(N+1) at the given (already perturbed) c."""
    N = len(h)
    n = 2 * (N + 1)
    out = np.zeros(2 * n * n)
    args = [_d(x) for x in (h, alpha, beta, rho)]
    lib().oracle_assemble(N, *[p for _, p in args], float(k), float(c), out.ctypes.data_as(_D))
    return (out[0::2] + 1j * out[1::2]).reshape(n, n)


def det_dense(A: np.ndarray):
    """O5: dense partial-pivot LU determinant → (complex mantissa, exponent, status)."""
    A = np.ascontiguousarray(A, dtype=np.complex128)
    n = A.shape[0]
    buf = np.empty(2 * n * n)
    buf[0::2] = A.real.ravel()
    buf[1::2] = A.imag.ravel()
    m = np.zeros(2)
    e = ctypes.c_int32(0)
    st = lib().oracle_det_dense(n, buf.ctypes.data_as(_D), m.ctypes.data_as(_D), ctypes.byref(e))
    return complex(m[0], m[1]), int(e.value), st


def det(h, alpha, beta, rho, lam, c, extended: bool = False, precision: str = "auto"):
    """O1–O5 at one (λ, c): returns (complex mantissa, exponent, status).

    precision "auto" is the oracle's own choice (fp64, or binary128 where the fp64 error
    bound exceeds its threshold, reading S15''); "fp64" forces the fp64 instance.
    ``extended=True`` runs the same arithmetic in long double (reading S15' audit)."""
    N = len(h)
    args = [_d(x) for x in (h, alpha, beta, rho)]
    m = np.zeros(2)
    e = ctypes.c_int32(0)
    if extended:
        fn = lib().oracle_det_ld
    else:
        fn = {"auto": lib().oracle_det, "fp64": lib().oracle_det_fp64}[precision]
    st = fn(N, *[p for _, p in args], float(lam), float(c), m.ctypes.data_as(_D), ctypes.byref(e))
    return complex(m[0], m[1]), int(e.value), st


def det_quad(h, alpha, beta, rho, lam, c):
    """O1–O5 in binary128 (reading S15''): (re_hi, re_lo, im_hi, im_lo) of the mantissa,
    exponent, status -- the mantissa to ~34 digits as two doubles per part."""
    N = len(h)
    args = [_d(x) for x in (h, alpha, beta, rho)]
    m = np.zeros(4)
    e = ctypes.c_int32(0)
    st = lib().oracle_det_q(N, *[p for _, p in args], float(lam), float(c),
                            m.ctypes.data_as(_D), ctypes.byref(e))
    return tuple(float(x) for x in m), int(e.value), st


def fp64_error_bound(h, alpha, beta, k, c):
    """Reading S15'': u·max_e[16(β_e/c)⁴ + (α_e β_e/c²)²/(k h_e)⁴], the a-priori relative
    error scale of an fp64 evaluation of det K at (k, c)."""
    N = len(h)
    args = [_d(x) for x in (h, alpha, beta)]
    return float(lib().oracle_fp64_error_bound(N, *[p for _, p in args], float(k), float(c)))


def det_kappa(h, alpha, beta, rho, lam, c):
    """Conditioning of det K w.r.t. 1-ulp errors in the per-layer cosh/sinh/sqrt values
    (reading S15'): relative det change bound, from long-double finite differences."""
    N = len(h)
    args = [_d(x) for x in (h, alpha, beta, rho)]
    out = ctypes.c_double(0.0)
    lib().oracle_det_kappa(N, *[p for _, p in args], float(lam), float(c), ctypes.byref(out))
    return out.value


def det_grid_kappa(h, alpha, beta, rho, lam, c, nthreads: int | None = None):
    """det_kappa on the full (λ, c) grid → kappa[L][V]."""
    N = len(h)
    args = [_d(x) for x in (h, alpha, beta, rho)]
    lam, plam = _d(lam)
    c, pc = _d(c)
    L, V = len(lam), len(c)
    kap = np.zeros((L, V))
    sts = np.zeros((L, V), dtype=np.int32)
    lib().oracle_det_grid_kappa(N, *[p for _, p in args], plam, L, pc, V, kap.ctypes.data_as(_D),
                                sts.ctypes.data_as(_I32), nthreads or default_threads())
    return kap


def classify_change(h, alpha, beta, rho, lam, c_lo, c_hi, iters: int = 40):
    """P10 (reading S21): is the sign change of Re det K in (c_lo, c_hi] a
    ROOT (a dispersion-curve point) or a POLE (an element's D_e -> 0, a clamped-layer
    resonance)?  Bisection on sgn Re det (O6) for `iters` halvings; near a simple root
    |Re det| shrinks ~1 bit per halving, near a simple pole it grows ~1 bit per halving, so
    the change of log2|Re det| at the bracket ends tells them apart.  A diagnostic: reported,
    not gated (the scan's semantics stay "first sign change").

    Returns (kind, c_star, dlog2) with kind in {"root", "pole", "undecided"}."""
    def sgn_log(c):
        m, e, st = det(h, alpha, beta, rho, lam, c)
        if st != 0 or m.real == 0.0:
            return 0.0, -math.inf
        return math.copysign(1.0, m.real), math.log2(abs(m.real)) + e

    s_lo, l_lo = sgn_log(c_lo)
    s_hi, l_hi = sgn_log(c_hi)
    if s_lo == s_hi:
        raise ValueError("no sign change of Re det in the bracket")
    l0 = max(l_lo, l_hi)
    lo, hi = float(c_lo), float(c_hi)
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        s, l = sgn_log(mid)
        if s == s_lo:
            lo, l_lo = mid, l
        else:
            hi, l_hi = mid, l
    d = max(l_lo, l_hi) - l0
    kind = "root" if d < -0.5 * iters else ("pole" if d > 0.5 * iters else "undecided")
    return kind, 0.5 * (lo + hi), d


# ---------------------------------------------------------------- O7..O10

def curve(h, alpha, beta, rho, lam, c, nthreads: int | None = None):
    """O7: Algorithm 1 for one model → (status, C_t[L], idx[L], ndet[L])."""
    N = len(h)
    args = [_d(x) for x in (h, alpha, beta, rho)]
    lam, plam = _d(lam)
    c, pc = _d(c)
    L, V = len(lam), len(c)
    ct = np.full(L, np.nan)
    idx = np.zeros(L, dtype=np.int32)
    nd = np.zeros(L, dtype=np.int64)
    st = lib().oracle_curve(N, *[p for _, p in args], plam, L, pc, V, ct.ctypes.data_as(_D),
                            idx.ctypes.data_as(_I32), nd.ctypes.data_as(_I64),
                            nthreads or default_threads())
    return st, ct, idx, nd


def misfit(ct, ce):
    """O8: Algorithm 2 → (status, m)."""
    ct, pct = _d(ct)
    ce, pce = _d(ce)
    out = ctypes.c_double(0.0)
    st = lib().oracle_misfit(pct, pce, len(ct), ctypes.byref(out))
    return st, out.value


def misfit_ld(ct, ce):
    ct, pct = _d(ct)
    ce, pce = _d(ce)
    out = ctypes.c_double(0.0)
    st = lib().oracle_misfit_ld(pct, pce, len(ct), ctypes.byref(out))
    return st, out.value


def ensemble(models, lam, c, ce=None, nthreads: int | None = None):
    """O9: per-model curves + misfits + argmin → dict."""
    M, N = models.h.shape
    args = [_d(x) for x in (models.h, models.alpha, models.beta, models.rho)]
    lam, plam = _d(lam)
    c, pc = _d(c)
    L, V = len(lam), len(c)
    ct = np.full((M, L), np.nan)
    idx = np.zeros((M, L), dtype=np.int32)
    nd = np.zeros((M, L), dtype=np.int64)
    mis = np.full(M, np.nan)
    best = ctypes.c_int64(-1)
    if ce is not None:
        ce, pce = _d(ce)
    else:
        pce = None
    st = lib().oracle_ensemble(M, N, *[p for _, p in args], plam, L, pc, V, pce,
                               ct.ctypes.data_as(_D), idx.ctypes.data_as(_I32),
                               mis.ctypes.data_as(_D), nd.ctypes.data_as(_I64),
                               ctypes.byref(best), nthreads or default_threads())
    return dict(status=st, ct=ct, idx=idx, misfit=mis, ndet=nd, best=int(best.value))


def det_grid(h, alpha, beta, rho, lam, c, nthreads: int | None = None, extended: bool = False):
    """O10: full (λ, c) det grid → (status, mant[L][V] complex, exp[L][V], status[L][V]).

    ``extended=True``: the same grid carried in long double (reading S15' audit)."""
    N = len(h)
    args = [_d(x) for x in (h, alpha, beta, rho)]
    lam, plam = _d(lam)
    c, pc = _d(c)
    L, V = len(lam), len(c)
    mre = np.zeros((L, V))
    mim = np.zeros((L, V))
    ex = np.zeros((L, V), dtype=np.int32)
    sts = np.zeros((L, V), dtype=np.int32)
    fn = lib().oracle_det_grid_ld if extended else lib().oracle_det_grid
    st = fn(N, *[p for _, p in args], plam, L, pc, V, mre.ctypes.data_as(_D),
                               mim.ctypes.data_as(_D), ex.ctypes.data_as(_I32),
                               sts.ctypes.data_as(_I32), nthreads or default_threads())
    return st, mre + 1j * mim, ex, sts
