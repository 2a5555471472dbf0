"""The algebra of the stable element (masw_det.cuh "stable element"),
checked in 50-digit arithmetic: the cancellation-free, exponentially scaled expressions
equal the App. A element entries exactly (up to 1e-40 relative), for both-hyperbolic and
mixed (hyperbolic P, trigonometric S) layers.  The GPU test (test_gpu_stable.py) then
checks the fp64 implementation against mpmath; this test pins the identities themselves,
independently of any fp64 code.
"""
import mpmath as mp
import numpy as np
import pytest


def direct_entries(kh, k, c, al, be, rho):
    """App. A, as tests/test_oracle_pins.py::_mp_det spells it (real r, s)."""
    r = mp.sqrt(mp.mpc(1 - c * c / al ** 2))
    s = mp.sqrt(mp.mpc(1 - c * c / be ** 2))
    Cr, Sr, Cs, Ss = mp.cosh(kh * r), mp.sinh(kh * r), mp.cosh(kh * s), mp.sinh(kh * s)
    D = 2 * (1 - Cr * Cs) + (1 / (r * s) + r * s) * Sr * Ss
    f = k * rho * c * c / D
    return {
        "k11": f * (Cr * Ss / s - r * Sr * Cs),
        "k12": f * (Cr * Cs - r * s * Sr * Ss - 1) - k * rho * be * be * (1 + s * s),
        "k13": f * (r * Sr - Ss / s),
        "k14": f * (Cs - Cr),
        "k22": f * (Sr * Cs / r - s * Cr * Ss),
        "k24": f * (s * Ss - Sr / r),
    }


def scaled(x):
    e = mp.exp(-x)
    return mp.cosh(x) * e, mp.sinh(x) * e, e


def stable_hh(kh, k, c, al, be, rho):
    """elem_stable_hh of masw_det.cuh, term by term."""
    a, b = c * c / al ** 2, c * c / be ** 2
    r, s = mp.sqrt(1 - a), mp.sqrt(1 - b)
    rs = r * s
    w = (a + b - a * b) / (1 + rs)
    dl = kh * ((b - a) / (r + s)) / 2
    Rc, Rs, Re = scaled(kh * r)
    Sc, Ss, Se = scaled(kh * s)
    Dc, Ds, De = scaled(dl)
    es2 = Se * Se
    sd2 = Ds * Ds
    sdcd2 = 2 * Ds * Dc
    csig = Sc * Dc + Ss * Ds
    ssig = Ss * Dc + Sc * Ds
    Dh = (w * w) / rs * Rs * Ss - 4 * sd2 * es2
    krho, mu = k * rho, k * rho * be * be
    fh = krho * c * c / Dh
    return {
        "k11": fh / s * (w * Rs * Sc - sdcd2 * es2),
        "k12": fh * (2 * sd2 * es2 + w * Rs * Ss) - mu * (2 - b),
        "k13": fh / s * Se * (2 * csig * Ds - w * Rs),
        "k14": -2 * fh * ssig * Ds * Se,
        "k22": fh / r * (sdcd2 * es2 + w * Rc * Ss),
        "k24": -fh / r * (2 * csig * Ds * Se + w * Ss * Re),
    }


def stable_ht(kh, k, c, al, be, rho):
    """elem_stable_ht: P wave scaled by e^-th_r, S wave trigonometric."""
    r = mp.sqrt(1 - c * c / al ** 2)
    xi = mp.sqrt(c * c / be ** 2 - 1)
    Rc, Rs, er = scaled(kh * r)
    Cr, XSr, SXr = Rc, r * Rs, Rs / r
    th = kh * xi
    Cs, XSs, SXs = mp.cos(th), -xi * mp.sin(th), mp.sin(th) / xi
    qb = 1 - c * c / be ** 2
    Dh = SXr * SXs + XSr * XSs + 2 * (er - Cr * Cs)
    krho, mu = k * rho, k * rho * be * be
    fh = krho * c * c / Dh
    return {
        "k11": fh * (Cr * SXs - XSr * Cs),
        "k12": fh * (Cr * Cs - XSr * XSs - er) - mu * (1 + qb),
        "k13": fh * (XSr - er * SXs),
        "k14": fh * (er * Cs - Cr),
        "k22": fh * (SXr * Cs - Cr * XSs),
        "k24": fh * (er * XSs - SXr),
    }


@pytest.mark.parametrize("seed", range(4))
def test_stable_hh_identities(seed):
    mp.mp.dps = 60
    rng = np.random.default_rng(seed)
    for _ in range(25):
        be = mp.mpf(rng.uniform(50, 400))
        al = be * mp.mpf(rng.uniform(1.5, 6))
        rho = mp.mpf(rng.uniform(1500, 2200))
        k = mp.mpf(rng.uniform(0.05, 12))
        kh = k * mp.mpf(rng.uniform(0.2, 8))
        c = be * mp.mpf(10.0 ** rng.uniform(-2, np.log10(0.99)))      # c < beta
        d, st = direct_entries(kh, k, c, al, be, rho), stable_hh(kh, k, c, al, be, rho)
        for key in d:
            assert abs(d[key] - st[key]) <= mp.mpf(10) ** -40 * (abs(d[key]) + 1), key


@pytest.mark.parametrize("seed", range(3))
def test_stable_ht_identities(seed):
    mp.mp.dps = 60
    rng = np.random.default_rng(100 + seed)
    for _ in range(25):
        be = mp.mpf(rng.uniform(50, 400))
        al = be * mp.mpf(rng.uniform(1.5, 6))
        rho = mp.mpf(rng.uniform(1500, 2200))
        k = mp.mpf(rng.uniform(0.05, 12))
        kh = k * mp.mpf(rng.uniform(0.2, 8))
        c = be + (al - be) * mp.mpf(rng.uniform(0.01, 0.99))            # beta < c < alpha
        d, st = direct_entries(kh, k, c, al, be, rho), stable_ht(kh, k, c, al, be, rho)
        for key in d:
            assert abs(d[key] - st[key]) <= mp.mpf(10) ** -40 * (abs(d[key]) + 1), key


def test_halfspace_gw_identity():
    """halfspace_root: w/(1 - rs) = w (1 + rs)/(a + b - ab) with a = c^2/alpha^2, w = b."""
    mp.mp.dps = 60
    for c in (mp.mpf("0.5"), mp.mpf(30), mp.mpf(150)):
        al, be = mp.mpf(1440), mp.mpf(290)
        a, b = c * c / al ** 2, c * c / be ** 2
        r, s = mp.sqrt(1 - a), mp.sqrt(1 - b)
        assert abs(b / (1 - r * s) - b * (1 + r * s) / (a + b - a * b)) < mp.mpf(10) ** -50
