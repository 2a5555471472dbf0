"""Parity rules of BASELINE.json's north_star, as DESIGN.md states them (readings S15, S16).

  * det K within 1e-9 relative (complex), inside the det-parity domain:
        c_j >= 0.5 * beta_min  and  |det_o| >= 1e-12 * max_row |det_o|           (S15)
        and kappa <= 1e-10                                                   (S15')
    where kappa (oracle.det_grid_kappa) is the first-order relative change of det K when each
    per-layer cosh/sinh value and square root -- quantities every fp64 evaluation of the
    Kausel-Roesset formulas must round -- is off by one unit roundoff.  Where kappa is large
    (e.g. long lambda at low c: D ~ 1e-6 by cancellation, 1 ulp in one cosh moves det K by
    1e-9) two correct fp64 implementations legitimately differ by more than 1e-9.
  * C_t: the same grid index as the oracle, except where the oracle's |Re det| at the
    straddling points falls below 1e-12 of its scan maximum; there one step is allowed (S16).
  * misfit within 1e-9 relative of oracle_misfit(GPU C_t, C_e)                      (S13)
"""
import math

import numpy as np

DET_RTOL = 1e-9
AUDIT_RTOL = 1e-11
KAPPA_MAX = 1e-10
NEAR_ROOT = 1e-12
MISFIT_RTOL = 1e-9


def det_to_complex_scaled(mant, exp2, ref_exp):
    """(mant * 2^exp2) / 2^ref_exp as complex (exact scaling by powers of two)."""
    return np.ldexp(mant.real, exp2 - ref_exp) + 1j * np.ldexp(mant.imag, exp2 - ref_exp)


def det_grid_rel_err(g_mant, g_exp, o_mant, o_exp):
    """Elementwise |det_g - det_o| / |det_o| computed in the oracle's exponent frame."""
    g = det_to_complex_scaled(g_mant, g_exp, o_exp)
    with np.errstate(divide="ignore", invalid="ignore"):
        return np.abs(g - o_mant) / np.abs(o_mant)


def det_domain(o_mant, o_exp, c, beta_min, kappa=None):
    """Boolean mask of the det-parity domain (S15, and S15' when the oracle's conditioning
    grid kappa is given) on an [L][V] oracle grid."""
    logabs = np.log2(np.abs(o_mant)) + o_exp
    rowmax = np.max(np.where(np.isfinite(logabs), logabs, -np.inf), axis=1, keepdims=True)
    big = logabs >= rowmax + math.log2(NEAR_ROOT)
    dom = big & (c[None, :] >= 0.5 * beta_min)
    if kappa is not None:
        dom &= kappa <= KAPPA_MAX
    return dom


def ct_acceptable(orc, model_args, lam, c, idx_g, idx_o):
    """Row-wise S16 rule.  Returns (ok_mask, n_exact, n_one_step)."""
    idx_g = np.asarray(idx_g)
    idx_o = np.asarray(idx_o)
    ok = idx_g == idx_o
    one = 0
    for i in np.nonzero(~ok)[0]:
        a, b = int(idx_g[i]), int(idx_o[i])
        if a < 1 or b < 1 or abs(a - b) > 1:
            continue
        jlo, jhi = min(a, b), max(a, b)
        vals = []
        for j in range(0, jhi + 1):
            m, e, st = orc.det(*model_args, float(lam[i]), float(c[j]))
            vals.append(abs(m.real) * 2.0 ** e if st == 0 else math.inf)
        M = max(vals)
        near = min(vals[jlo - 1], vals[jlo], vals[jhi])
        if near < NEAR_ROOT * M:
            ok[i] = True
            one += 1
    return ok, int(np.sum(idx_g == idx_o)), one


def misfit_ok(orc, ct_g, ce, mis_g):
    st, m = orc.misfit(ct_g, ce)
    if math.isinf(m) or math.isinf(mis_g):
        return math.isinf(m) and math.isinf(mis_g)
    if m == 0.0:
        return mis_g == 0.0
    return abs(mis_g - m) <= MISFIT_RTOL * abs(m)
