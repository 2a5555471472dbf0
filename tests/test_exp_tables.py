"""The cosh/sinh tables and polynomials of the scan kernels (csrc/masw_exp_table.h), checked
against 50-digit mpmath on the host (no GPU): every sampled table row correctly rounded, the
polynomials within their stated error bounds, and the kernels' reconstruction
    th = m d + r,  cosh th = A (1 + E) + B O,  sinh th = B (1 + E) + A O
replayed with exactly emulated fp64 fma/add/mul (Fractions, one rounding per operation) --
the coarse table (d = 1/16, any call) and the fine one (d = 1/128, calls with k h <= 50.5) --
within ~1.5 ulp of cosh and sinh.  These are the values every layer element is built from
(App. A's C, S terms; PAPER.md:74 cites the element, reading S1)."""
import os
import random
import re
from fractions import Fraction

import mpmath as mp
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "paper_2003_02256_b200", "csrc", "masw_exp_table.h")
mp.mp.dps = 50


def _parse():
    src = open(HDR).read()
    consts = {}
    for name, val in re.findall(r"constexpr double (\w+) = ([^;]+);", src):
        v = val.strip()
        consts[name] = float.fromhex(v) if v.startswith(("0x", "-0x")) else float(v)
    arrays = {}
    for name, body in re.findall(r"static __constant__ double (\w+)\[\d+\] = \{([^}]*)\};", src):
        arrays[name] = [float.fromhex(x.strip()) for x in body.split(",")]
    tabs = {}
    for name, body in re.findall(r"__device__ const double2 (\w+)\[kExpTabNF?\] = \{(.*?)\n\};", src, re.S):
        rows = re.findall(r"\{([^,]+), ([^}]+)\}", body)
        tabs[name] = [(float.fromhex(a.strip()), float.fromhex(b.strip())) for a, b in rows]
    return consts, arrays, tabs


C, A, T = _parse()


def rnd(x: Fraction) -> float:
    """x rounded to the nearest double (ties to even), via mpmath at 200 bits."""
    with mp.workprec(200):
        return float(mp.mpf(x.numerator) / x.denominator)


def fma(a, b, c):
    return rnd(Fraction(a) * Fraction(b) + Fraction(c))


def mul(a, b):
    return rnd(Fraction(a) * Fraction(b))


def add(a, b):
    return rnd(Fraction(a) + Fraction(b))


SHIFTER = 6755399441055744.0   # 1.5 * 2^52


def cosh_sinh(th, fine):
    """The kernels' cosh_sinh / cosh_sinh_fine (masw_det.cuh), operation by operation."""
    d = C["kExpFD"] if fine else C["kExpD"]
    tab = T["g_cosh_sinh_fine" if fine else "g_cosh_sinh"]
    S = SHIFTER * d
    t = add(th, S)
    md = add(t, -S)
    m = int(round((t - S) / d))
    r = add(th, -md)
    assert Fraction(r) == Fraction(th) - Fraction(md)   # exact reduction
    u = mul(r, r)
    if fine:
        pe = fma(C["kExpFE1_0"], u, A["c_expFE1"][1])
        po = fma(C["kExpFO2_0"], u, A["c_expFO2"][1])
        po = fma(po, u, A["c_expFO2"][2])
    else:
        pe = fma(C["kExpE2_0"], u, A["c_expE2"][1])
        po = fma(C["kExpO3_0"], u, A["c_expO3"][1])
        pe = fma(pe, u, A["c_expE2"][2])
        for i in (2, 3):
            po = fma(po, u, A["c_expO3"][i])
    E, O = mul(pe, u), mul(po, r)
    a, b = tab[min(m, len(tab) - 1)]
    return fma(a, E, fma(b, O, a)), fma(b, E, fma(a, O, b))


def ulp(x):
    return abs(mp.mpf(x)) * mp.mpf(2) ** -52


def test_table_rows_correctly_rounded():
    rng = random.Random(7)
    for name, d, n in (("g_cosh_sinh", mp.mpf(1) / 16, 5680),
                       ("g_cosh_sinh_fine", mp.mpf(1) / 128, 6472)):
        tab = T[name]
        assert len(tab) == n
        for m in [0, 1, 2, n - 1] + rng.sample(range(3, n - 1), 150):
            ch, sh = mp.cosh(m * d), mp.sinh(m * d)
            assert tab[m][0] == float(ch) and tab[m][1] == float(sh), (name, m)


def test_fine_range_constant():
    # the fine table covers th < (6472 - 1/2) / 128; the scans take it only for k h <= 50.5
    assert C["kExpFineKhMax"] == pytest.approx((6472 - 0.5) / 128)
    src = open(os.path.join(ROOT, "paper_2003_02256_b200", "csrc", "masw_det.cuh")).read()
    kh = float(re.search(r"#define MASW_FINE_KH_MAX ([0-9.]+)", src).group(1))
    assert kh < C["kExpFineKhMax"]


@pytest.mark.parametrize("fine", [False, True])
def test_polynomials_within_stated_error(fine):
    d = mp.mpf(1) / (128 if fine else 16)
    umax = (d / 2) ** 2
    if fine:
        pe = [C["kExpFE1_0"], A["c_expFE1"][1]]
        po = [C["kExpFO2_0"]] + A["c_expFO2"][1:]
    else:
        pe = [C["kExpE2_0"]] + A["c_expE2"][1:]
        po = [C["kExpO3_0"]] + A["c_expO3"][1:]
    worst_e = worst_o = mp.mpf(0)
    for i in range(401):
        r = d / 2 * i / 400
        u = r * r
        E = mp.polyval([mp.mpf(c) for c in pe], u) * u
        O = mp.polyval([mp.mpf(c) for c in po], u) * r
        worst_e = max(worst_e, abs(E - (mp.cosh(r) - 1)))
        if r:
            worst_o = max(worst_o, abs(O / mp.sinh(r) - 1))
    assert umax < 1e-2
    assert worst_e < 1e-18      # E's absolute error (what cosh = A (1 + E) + B O sees)
    assert worst_o < 1e-18      # O's relative error


@pytest.mark.parametrize("fine", [False, True])
def test_reconstruction_within_1p5_ulp(fine):
    rng = random.Random(11 + fine)
    hi = 50.5 if fine else 350.0
    pts = [0.0, 1e-300, 1e-9, 0.5 / 128, 0.03125, 1.0, hi] + [rng.uniform(0, hi) for _ in range(150)]
    pts += [rng.uniform(0, 0.1) for _ in range(40)]
    worst = 0.0
    for th in pts:
        ch, sh = cosh_sinh(th, fine)
        ech, esh = mp.cosh(th), mp.sinh(th)
        worst = max(worst, float(abs(ch - ech) / ulp(ech)))
        if th:
            worst = max(worst, float(abs(sh - esh) / ulp(esh)))
        else:
            assert sh == 0.0
    assert worst < 1.5, worst


def test_fine_and_coarse_agree_to_rounding():
    """Both tables evaluate the same function: the scans of a call with k h <= 50.5 (fine) and
    the coarse path differ only by rounding (so C_t can differ only at near-roots, S16)."""
    rng = random.Random(3)
    for _ in range(120):
        th = rng.uniform(0, 50.5)
        a, b = cosh_sinh(th, False), cosh_sinh(th, True)
        assert abs(a[0] - b[0]) <= 2 * float(ulp(a[0])) and abs(a[1] - b[1]) <= 2 * float(ulp(a[1]) or 1e-300)
