"""Pins of the CPU fp64 oracle (SURVEY.md §8(c) P1–P12) against things other than itself:
closed forms, textbook routines, mathematical identities, brute force and the paper's
printed examples.  Each pin is chosen so that a plausible slip in the oracle (a dropped
term, a wrong sign or index, a transposed operand) fails at least one test.

No GPU needed; marked ``not gpu`` implicitly.
"""
import math
import os

import numpy as np
import pytest
from scipy.optimize import brentq

import synth


# ------------------------------------------------------------------ independent textbook pieces

def rayleigh_function(c, alpha, beta):
    """Textbook Rayleigh function R(c) = (2 − c²/β²)² − 4·√(1 − c²/α²)·√(1 − c²/β²), c < β."""
    return (2.0 - c * c / beta ** 2) ** 2 - 4.0 * math.sqrt(1 - c * c / alpha ** 2) * math.sqrt(
        1 - c * c / beta ** 2)


def rayleigh_root(alpha, beta):
    """Rayleigh-wave velocity by bracketing bisection on R(c) in (0.5β, β)."""
    return brentq(lambda c: rayleigh_function(c, alpha, beta), 0.5 * beta, beta * (1 - 1e-15),
                  xtol=1e-14, rtol=1e-15)


def first_grid_above(grid, x):
    j = int(np.searchsorted(grid, x, side="right"))
    return j, grid[j]


# ------------------------------------------------------------------ P1 half-space / Rayleigh

def test_rayleigh_closed_form_poisson_quarter():
    # ν = 1/4 ⇒ α = √3 β ⇒ c_R/β = √(2 − 2/√3) (classical closed form)
    b = 200.0
    cr = rayleigh_root(b * math.sqrt(3.0), b)
    assert abs(cr / b - math.sqrt(2.0 - 2.0 / math.sqrt(3.0))) < 1e-13
    assert abs(cr / b - 0.9194016867619659) < 1e-13


@pytest.mark.parametrize("c", [50.0, 120.0, 183.0, 199.0])
def test_halfspace_det_equals_rayleigh_function(orc, c):
    """det K_hs = −(kρβ²)²·R(c)/(1 − rs): the half-space element's determinant is the
    Rayleigh function up to a non-vanishing factor (App. A; derivation in DESIGN.md)."""
    b, a, rho = 200.0, 200.0 * math.sqrt(3.0), 1900.0
    for lam in (3.0, 10.0, 40.0):
        k = 2 * math.pi / lam
        K = orc.halfspace_element(a, b, rho, k, c)
        det = K[0, 0] * K[1, 1] - K[0, 1] * K[1, 0]
        r = math.sqrt(1 - c * c / a ** 2)
        s = math.sqrt(1 - c * c / b ** 2)
        want = -(k * rho * b * b) ** 2 * rayleigh_function(c, a, b) / (1 - r * s)
        assert abs(det.imag) == 0.0
        assert abs(det.real - want) <= 1e-12 * (k * rho * b * b) ** 2


@pytest.mark.parametrize("lam", [5.0, 10.0, 20.0])
def test_P1_homogeneous_halfspace_rayleigh_index(orc, lam):
    """Homogeneous half-space (thin dummy layer identical to it), ν = 0.25, β = 200:
    C_t is the first grid velocity above 0.9194β."""
    b = 200.0
    a = b * math.sqrt(3.0)
    grid = synth.maswaves_grid()
    j, cj = first_grid_above(grid, rayleigh_root(a, b))
    st, ct, idx, nd = orc.curve([1.0], [a, a], [b, b], [1900.0, 1900.0], [lam], grid)
    assert st == orc.OK
    assert (j, cj) == (367, 184.0)
    assert idx[0] == j and ct[0] == cj and nd[0] == j + 1


# ------------------------------------------------------------------ P2 identical stack

@pytest.mark.parametrize("N", [1, 3, 6])
def test_P2_identical_layers_collapse_to_halfspace(orc, N):
    b = 200.0
    a = b * math.sqrt(3.0)
    grid = synth.maswaves_grid()
    h = [1.0 + 0.5 * e for e in range(N)]
    st, ct, idx, nd = orc.curve(h, [a] * (N + 1), [b] * (N + 1), [1900.0] * (N + 1),
                                [5.0, 10.0, 20.0], grid)
    assert st == orc.OK
    assert list(idx) == [367, 367, 367]


# ------------------------------------------------------------------ P3 h → ∞

@pytest.mark.parametrize("c", [80.0, 150.0, 190.0])
def test_P3_thick_layer_top_block_tends_to_halfspace(orc, c):
    b, a, rho = 200.0, 346.0, 1800.0
    k = 2 * math.pi / 10.0
    Kh = orc.halfspace_element(a, b, rho, k, c)
    sh = math.sqrt(1 - c * c / b ** 2)
    Ke = orc.layer_element(40.0 / (k * sh), a, b, rho, k, c)    # k·s·h = 40 ⇒ e^{-40} terms
    scale = np.abs(Kh).max()
    assert np.abs(Ke[:2, :2] - Kh).max() <= 1e-12 * scale
    # the coupling to the far face decays like e^{−k s h}
    assert np.abs(Ke[:2, 2:]).max() <= 1e-12 * scale


# ------------------------------------------------------------------ P4 condensation

@pytest.mark.parametrize("c", [120.0, 250.0, 400.0, 20.0])
@pytest.mark.parametrize("h1,h2", [(1.0, 2.0), (0.3, 3.7)])
def test_P4_condensation_of_stacked_layers(orc, c, h1, h2):
    """A layer of thickness h1+h2 equals two stacked layers of the same material with the
    interface DOFs statically condensed (Schur complement).  Exercises both real and
    imaginary r, s branches: c < β, β < c < α, c > α."""
    b, a, rho = 200.0, 346.0, 1800.0
    k = 2 * math.pi / 7.0
    K1 = orc.layer_element(h1, a, b, rho, k, c)
    K2 = orc.layer_element(h2, a, b, rho, k, c)
    K12 = orc.layer_element(h1 + h2, a, b, rho, k, c)
    G = np.zeros((6, 6), dtype=complex)
    G[0:4, 0:4] += K1
    G[2:6, 2:6] += K2
    keep = [0, 1, 4, 5]
    mid = [2, 3]
    S = G[np.ix_(keep, keep)] - G[np.ix_(keep, mid)] @ np.linalg.solve(G[np.ix_(mid, mid)],
                                                                        G[np.ix_(mid, keep)])
    scale = np.abs(K12).max()
    assert np.abs(S - K12).max() <= 1e-10 * scale


# ------------------------------------------------------------------ P5 structure

def test_P5_element_identities_and_symmetry(orc):
    rng = np.random.default_rng(5)
    for _ in range(50):
        b = rng.uniform(60, 400)
        a = b * rng.uniform(1.2, 8.0)
        c = rng.uniform(5, 1.5 * a)
        Ke = orc.layer_element(rng.uniform(0.2, 6), a, b, rng.uniform(1500, 2200),
                               2 * math.pi / rng.uniform(0.5, 80), c)
        assert np.array_equal(Ke, Ke.T)
        assert Ke[2, 2] == Ke[0, 0] and Ke[3, 3] == Ke[1, 1]
        assert Ke[2, 3] == -Ke[0, 1] and Ke[1, 2] == -Ke[0, 3]
        # every layer entry is even in r and s ⇒ exactly real for real c, k (reading S3/S5)
        assert np.all(Ke.imag == 0.0)


@pytest.mark.parametrize("N", [1, 2, 5, 10])
def test_P5_assembly_order_band_and_block_tridiagonal(orc, N):
    rng = np.random.default_rng(N)
    beta = rng.uniform(80, 300, N + 1)
    alpha = beta * 2.2
    h = rng.uniform(0.5, 4, N)
    rho = rng.uniform(1700, 2000, N + 1)
    K = orc.assemble(h, alpha, beta, rho, 2 * math.pi / 9.0, 0.8 * beta.min())
    n = 2 * (N + 1)
    assert K.shape == (n, n)                              # PAPER.md:78 order 2(N+1)
    assert np.array_equal(K, K.T)                         # "symmetric banded" PAPER.md:78
    for i in range(n):
        for j in range(n):
            if abs(i - j) > 3:
                assert K[i, j] == 0                       # heptadiagonal
            if i // 2 != j // 2 and abs(i // 2 - j // 2) > 1:
                assert K[i, j] == 0                       # 2×2 block-tridiagonal (reading S10)
    # below β_N and α_N the whole matrix is real (reading S5)
    assert np.all(K.imag == 0.0)
    # above β_N the half-space block is complex, layers stay real
    K2 = orc.assemble(h, alpha, beta, rho, 2 * math.pi / 9.0, beta[N] * 1.1)
    assert np.all(K2[: 2 * N, : 2 * N].imag == 0.0)
    assert np.any(K2[2 * N:, 2 * N:].imag != 0.0)


def test_P5_paper_matrix_size_fact():
    """N=6 → 196 entries × 16 B = 3136 B per matrix; 500×1000 ≈ 1.6 GB."""
    n = 2 * (6 + 1)
    assert n * n == 196 and n * n * 16 == 3136
    assert 500 * 1000 * 3136 == 1_568_000_000


# ------------------------------------------------------------------ P6 config-2 twin

def test_P6_maswaves_twin_same_indices(orc):
    out = []
    for name in ("maswaves", "maswaves_twin"):
        w = synth.workload(name)
        m = w.models
        st, ct, idx, nd = orc.curve(m.h[0], m.alpha[0], m.beta[0], m.rho[0], w.lam, w.c)
        assert st == orc.OK
        out.append(idx)
    assert np.array_equal(out[0], out[1])


# ------------------------------------------------------------------ P7 determinant

def test_P7_dense_det_special_cases(orc):
    m, e, st = orc.det_dense(np.eye(7))
    assert st == 0 and m * 2.0 ** e == 1.0
    m, e, st = orc.det_dense(np.diag([2.0, 3.0, 4.0]).astype(complex))
    assert m * 2.0 ** e == 24.0
    P = np.eye(4)[[1, 0, 2, 3]]                       # one swap ⇒ −1
    m, e, st = orc.det_dense(P)
    assert m * 2.0 ** e == -1.0
    A = np.array([[0, 2], [3, 0]], dtype=complex)     # needs pivoting: det = −6
    m, e, st = orc.det_dense(A)
    assert m * 2.0 ** e == -6.0
    m, e, st = orc.det_dense(np.zeros((3, 3)))
    assert m == 0 and st == 0
    A = np.eye(3, dtype=complex)
    A[1, 1] = np.nan
    assert orc.det_dense(A)[2] == orc.E_NONFINITE


def test_P7_dense_det_matches_lapack_random(orc):
    rng = np.random.default_rng(7)
    for n in (2, 4, 7, 14, 22):
        for _ in range(20):
            A = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
            m, e, st = orc.det_dense(A)
            want = np.linalg.det(A)
            got = m * 2.0 ** e
            assert abs(got - want) <= 1e-12 * abs(want)
            assert 0.5 <= max(abs(m.real), abs(m.imag)) < 1.0


def test_P7_det_of_stiffness_matches_lapack_and_magnitude(orc):
    w = synth.workload("maswaves")
    m = w.models
    for lam in (40.0, 5.0, 1.0):
        for c in (50.0, 149.0, 300.0, 480.0):
            k = orc.wavenumber(lam)
            K = orc.assemble(m.h[0], m.alpha[0], m.beta[0], m.rho[0], k, c)
            mant, e, st = orc.det_dense(K)
            sign, logabs = np.linalg.slogdet(K)
            assert abs(math.log(abs(mant)) + e * math.log(2.0) - logabs) < 1e-10
            assert abs(mant / abs(mant) - sign) < 1e-9


def test_P7_wavenumber_and_perturbation(orc):
    assert orc.wavenumber(1.0) == 6.283185307179586
    assert orc.wavenumber(2.0) == 6.283185307179586 / 2.0
    alpha = [240.0, 400.0, 640.0]
    beta = [120.0, 200.0, 320.0]
    assert orc.perturb_velocity(alpha, beta, 119.0) == 119.0
    assert orc.perturb_velocity(alpha, beta, 120.0) == 120.0 * (1 - 1e-4)
    assert orc.perturb_velocity(alpha, beta, 120.00005) == 120.00005 * (1 - 1e-4)
    assert orc.perturb_velocity(alpha, beta, 640.0) == 640.0 * (1 - 1e-4)
    # a perturbed velocity gives a finite determinant where the raw one is 0/0
    m, e, st = orc.det([2.0, 4.0], alpha, beta, [1800, 1900, 2000], 10.0, 200.0)
    assert st == 0 and math.isfinite(m.real)


# ------------------------------------------------------------------ P8 early exit vs brute force

@pytest.mark.parametrize("name", ["tiny", "maswaves"])
def test_P8_early_exit_equals_full_grid_first_change(orc, name):
    w = synth.workload(name)
    m = w.models
    args = (m.h[0], m.alpha[0], m.beta[0], m.rho[0])
    st, ct, idx, nd = orc.curve(*args, w.lam, w.c)
    st2, mant, ex, sts = orc.det_grid(*args, w.lam, w.c)
    assert st2 == 0 and np.all(sts == 0)
    sgn = np.sign(mant.real)
    for i in range(len(w.lam)):
        ch = np.nonzero(sgn[i, 1:] != sgn[i, :-1])[0]
        j = int(ch[0]) + 1
        assert idx[i] == j and ct[i] == w.c[j] and nd[i] == j + 1
        # monotone soundness: every earlier det has the sign of det(V[0])
        assert np.all(sgn[i, :j] == sgn[i, 0])
    assert nd.sum() == (idx + 1).sum() < len(w.lam) * len(w.c)
    assert nd.sum() == {"tiny": 6011, "maswaves": 10992}[name]


def test_P8_no_sign_change_and_zero_sign(orc):
    # grid entirely below the Rayleigh root: no change ⇒ idx −1, C_t NaN, warn status
    b = 200.0
    a = b * math.sqrt(3.0)
    st, ct, idx, nd = orc.curve([1.0], [a, a], [b, b], [1900, 1900], [5.0],
                                np.linspace(50, 150, 11))
    assert st == orc.WARN_NO_SIGN_CHANGE and idx[0] == -1 and math.isnan(ct[0]) and nd[0] == 11


# ------------------------------------------------------------------ P9 fp64 conditioning (mpmath)

def _mp_det(h, alpha, beta, rho, lam, c, dps=50, k_double=False):
    """60-digit det K from App. A (bounds rounding, not the formula).  ``k_double`` uses the
    fp64 wavenumber fl(2π/λ) exactly, so only arithmetic rounding differs from fp64 codes."""
    import mpmath as mp

    mp.mp.dps = dps
    N = len(h)
    n = 2 * (N + 1)
    k = mp.mpf(6.283185307179586 / lam) if k_double else 2 * mp.pi / mp.mpf(lam)
    c = mp.mpf(c)
    K = mp.matrix(n, n)

    def rs(a, b):
        return mp.sqrt(mp.mpc(1 - c * c / mp.mpf(a) ** 2)), mp.sqrt(mp.mpc(1 - c * c / mp.mpf(b) ** 2))

    for e in range(N):
        r, s = rs(alpha[e], beta[e])
        he, rh, bt = mp.mpf(h[e]), mp.mpf(rho[e]), mp.mpf(beta[e])
        Cr, Sr, Cs, Ss = mp.cosh(k * r * he), mp.sinh(k * r * he), mp.cosh(k * s * he), mp.sinh(k * s * he)
        D = 2 * (1 - Cr * Cs) + (1 / (r * s) + r * s) * Sr * Ss
        f = k * rh * c * c / D
        k11 = f * (Cr * Ss / s - r * Sr * Cs)
        k12 = f * (Cr * Cs - r * s * Sr * Ss - 1) - k * rh * bt * bt * (1 + s * s)
        k13 = f * (r * Sr - Ss / s)
        k14 = f * (Cs - Cr)
        k22 = f * (Sr * Cs / r - s * Cr * Ss)
        k24 = f * (s * Ss - Sr / r)
        Ke = [[k11, k12, k13, k14], [k12, k22, -k14, k24], [k13, -k14, k11, -k12], [k14, k24, -k12, k22]]
        for a_ in range(4):
            for b_ in range(4):
                K[2 * e + a_, 2 * e + b_] += Ke[a_][b_]
    r, s = rs(alpha[N], beta[N])
    mu = k * mp.mpf(rho[N]) * mp.mpf(beta[N]) ** 2
    q = (1 - s * s) / (1 - r * s)
    K[2 * N, 2 * N] += mu * r * q
    K[2 * N, 2 * N + 1] += mu * q - 2 * mu
    K[2 * N + 1, 2 * N] += mu * q - 2 * mu
    K[2 * N + 1, 2 * N + 1] += mu * s * q
    return mp.det(K)


@pytest.mark.parametrize("lam", [0.5, 5.0, 100.0])
def test_P9_conditioning_envelope(orc, lam):
    """Within the det-parity domain (c ≥ 0.5 β_min, reading S15) the fp64 oracle det is
    within 1e-9 relative of a 50-digit evaluation (bounds rounding, not the formula)."""
    import mpmath as mp

    m = synth.maswaves_model()
    args = (m.h[0], m.alpha[0], m.beta[0], m.rho[0])
    for c in (40.0, 100.0, 200.0, 285.0, 320.0):
        mant, e, st = orc.det(*args, lam, c)
        got = mp.mpc(mant.real, mant.imag) * mp.mpf(2) ** e
        want = _mp_det(*args, lam, c)
        rel = abs(got - want) / abs(want)
        assert rel < 1e-9, (lam, c, float(rel))


def test_P9_extended_audit_is_accurate(orc):
    """The long-double instance of the oracle's det path (reading S15') reproduces a
    50-digit evaluation at the same fp64 inputs to 1e-11, including points where the fp64
    oracle itself is off by ~1e-9 (so it can serve as the fp64 rounding-error audit)."""
    w = synth.workload("ensemble", M=400)
    mods = w.models
    pts = [(313, 0, 30.554), (230, 17, 232.810), (286, 39, 23.157), (146, 7, 32.414),
           (54, 16, 354.939), (121, 32, 244.121)]
    worst_fp64 = 0.0
    for mi, i, c in pts:
        a = (mods.h[mi], mods.alpha[mi], mods.beta[mi], mods.rho[mi])
        cp = orc.perturb_velocity(a[1], a[2], c)
        ex = complex(_mp_det(*a, w.lam[i], cp, k_double=True))
        ml, el, st = orc.det(*a, w.lam[i], c, extended=True)
        assert st == 0 and abs(ml * 2.0 ** el - ex) <= 1e-11 * abs(ex)
        m, e, st = orc.det(*a, w.lam[i], c)
        worst_fp64 = max(worst_fp64, abs(m * 2.0 ** e - ex) / abs(ex))
    assert worst_fp64 > 1e-10      # the audit matters: fp64 alone is not 1e-10-accurate here


def _mp_det_pert(h, alpha, beta, rho, lam, c, pe, pw, eps, dps=40):
    """50-digit det K with one intermediate value of element pe scaled by (1 + eps):
    pw 0..3 = cosh/sinh of the P and S waves (Cr, Sr, Cs, Ss), 4/5 = r/s (pe == N: half-space)."""
    import mpmath as mp

    mp.mp.dps = dps
    N = len(h)
    n = 2 * (N + 1)
    k = mp.mpf(6.283185307179586 / lam)
    c = mp.mpf(c)
    K = mp.matrix(n, n)
    for e in range(N + 1):
        al, be, rh = mp.mpf(alpha[e]), mp.mpf(beta[e]), mp.mpf(rho[e])
        r = mp.sqrt(mp.mpc(1 - c * c / al ** 2))
        s = mp.sqrt(mp.mpc(1 - c * c / be ** 2))
        if e == pe and pw == 4:
            r *= 1 + eps
        if e == pe and pw == 5:
            s *= 1 + eps
        if e == N:
            mu = k * rh * be * be
            q = (1 - s * s) / (1 - r * s)
            K[2 * N, 2 * N] += mu * r * q
            K[2 * N, 2 * N + 1] += mu * q - 2 * mu
            K[2 * N + 1, 2 * N] += mu * q - 2 * mu
            K[2 * N + 1, 2 * N + 1] += mu * s * q
            continue
        he = mp.mpf(h[e])
        v = [mp.cosh(k * r * he), mp.sinh(k * r * he), mp.cosh(k * s * he), mp.sinh(k * s * he)]
        if e == pe and pw < 4:
            v[pw] *= 1 + eps
        Cr, Sr, Cs, Ss = v
        D = 2 * (1 - Cr * Cs) + (1 / (r * s) + r * s) * Sr * Ss
        f = k * rh * c * c / D
        k11 = f * (Cr * Ss / s - r * Sr * Cs)
        k12 = f * (Cr * Cs - r * s * Sr * Ss - 1) - k * rh * be * be * (1 + s * s)
        k13 = f * (r * Sr - Ss / s)
        k14 = f * (Cs - Cr)
        k22 = f * (Sr * Cs / r - s * Cr * Ss)
        k24 = f * (s * Ss - Sr / r)
        Ke = [[k11, k12, k13, k14], [k12, k22, -k14, k24], [k13, -k14, k11, -k12], [k14, k24, -k12, k22]]
        for a_ in range(4):
            for b_ in range(4):
                K[2 * e + a_, 2 * e + b_] += Ke[a_][b_]
    return mp.det(K)


def test_P9_kappa_matches_mpmath_sensitivity(orc):
    """kappa (reading S15') = 2^-53 * sum |d ln det / d ln v| over the per-layer cosh/sinh
    values and square roots, checked against the same sum from 40-digit finite differences,
    at an ill-conditioned point (long lambda, low c: D ~ 1e-6 by cancellation) and a benign one."""
    import mpmath as mp

    w = synth.workload("ensemble", M=400)
    m = w.models
    for mi, lam, c in [(374, 36.38995596158663, 27.531635247710145), (3, 5.0, 150.0)]:
        a = (m.h[mi], m.alpha[mi], m.beta[mi], m.rho[mi])
        cp = orc.perturb_velocity(a[1], a[2], c)
        N = len(a[0])
        eps = mp.mpf(2) ** -60
        d0 = _mp_det_pert(*a, lam, cp, -1, -1, eps)
        tot = 0
        for pe in range(N + 1):
            for pw in (range(4, 6) if pe == N else range(6)):
                d1 = _mp_det_pert(*a, lam, cp, pe, pw, eps)
                tot += abs(d1 / d0 - 1) / eps
        want = float(tot) * 2.0 ** -53
        got = orc.det_kappa(*a, lam, c)
        assert abs(got - want) <= 0.02 * want, (mi, got, want)
    assert orc.det_kappa(*(m.h[374], m.alpha[374], m.beta[374], m.rho[374]),
                         36.38995596158663, 27.531635247710145) > 1e-9


def test_P9_extended_grid_matches_pointwise(orc):
    w = synth.workload("tiny")
    m = w.models
    a = (m.h[0], m.alpha[0], m.beta[0], m.rho[0])
    st, mant, ex, sts = orc.det_grid(*a, w.lam[:3], w.c[::50], extended=True)
    for i in range(3):
        for j, c in enumerate(w.c[::50]):
            mm, ee, s = orc.det(*a, w.lam[i], c, extended=True)
            assert mm == mant[i, j] and ee == ex[i, j]


# ------------------------------------------------------------------ reading S15'' (small c)
# The oracle's precision ladder: fp64 where the a-priori error scale
#   P(c, k) = u max_e [16 (beta_e/c)^4 + (alpha_e beta_e / c^2)^2 / (k h_e)^4]
# is <= 1e-6, else the same formulas in long double / binary128.  Pinned against 60-digit
# mpmath (bounds rounding, not the formula), never against the oracle itself.

LID = dict(seed=101, N=1, m=28)          # thin stiff lid (beta 491 m/s, 0.77 m) on a soft half-space


def _lid_model():
    mods = synth.random_models(160, LID["N"], LID["seed"])
    return tuple(x[LID["m"]] for x in (mods.h, mods.alpha, mods.beta, mods.rho))


def _mp_sign(a, lam, c):
    return int(np.sign(float(_mp_det(*a, lam, c, dps=60, k_double=True).real)))


def test_S15pp_quad_instance_matches_mpmath(orc):
    """The binary128 instance reproduces 60-digit mpmath within its own error scale
    (40 P 2^-60, u = 2^-113 instead of 2^-53; <= 1e-15 here) at the ill-conditioned low-c
    points, where the fp64 instance is off by tens of percent or more, and at a benign point;
    the automatic choice has mpmath's sign there."""
    import mpmath as mp

    a = _lid_model()
    worst_fp64 = 0.0
    for lam, c in [(60.0, 0.5), (55.0, 1.0), (57.0, 1.5), (5.0, 0.5), (60.0, 150.0)]:
        cp = orc.perturb_velocity(a[1], a[2], c)
        P = orc.fp64_error_bound(a[0], a[1], a[2], 6.283185307179586 / lam, cp)
        ex = _mp_det(*a, lam, cp, dps=60, k_double=True)
        (rh, rl, ih, il), e, st = orc.det_quad(*a, lam, c)
        got = mp.mpc(mp.mpf(rh) + mp.mpf(rl), mp.mpf(ih) + mp.mpf(il)) * mp.mpf(2) ** e
        err = float(abs(got - ex) / abs(ex))
        assert st == 0 and err <= 40.0 * P * 2.0 ** -60 + 1e-30 and err < 1e-15, (lam, c, err, P)
        m, e2, _ = orc.det(*a, lam, c, precision="fp64")
        worst_fp64 = max(worst_fp64, float(abs(mp.mpc(m.real, m.imag) * mp.mpf(2) ** e2 - ex) / abs(ex)))
        ma, ea, _ = orc.det(*a, lam, c)
        assert np.sign(ma.real) == np.sign(float(ex.real))
    assert worst_fp64 > 0.1        # the ladder matters here: fp64 alone is not sign-safe


def test_S15pp_bound_dominates_fp64_error(orc):
    """P is an error SCALE for the fp64 instance: on random layered models at low c the
    measured fp64 error never exceeds 40 P (and P rises as c falls), while every automatic
    (laddered) oracle determinant is within 1e-5 of mpmath."""
    import mpmath as mp

    worst_ratio, worst_auto = 0.0, 0.0
    for N, seed, mi in [(2, 102, 32), (3, 103, 4), (5, 105, 22), (8, 108, 38), (8, 108, 8)]:
        mods = synth.random_models(40, N, seed)
        a = tuple(x[mi] for x in (mods.h, mods.alpha, mods.beta, mods.rho))
        for lam in (60.0, 5.0):
            Ps = []
            for c in (0.5, 2.0, 8.0):
                k = 6.283185307179586 / lam
                cp = orc.perturb_velocity(a[1], a[2], c)
                P = orc.fp64_error_bound(a[0], a[1], a[2], k, cp)
                Ps.append(P)
                ex = _mp_det(*a, lam, cp, dps=60, k_double=True)
                m, e, _ = orc.det(*a, lam, c, precision="fp64")
                err = float(abs(mp.mpc(m.real, m.imag) * mp.mpf(2) ** e - ex) / abs(ex))
                worst_ratio = max(worst_ratio, err / P)
                ma, ea, _ = orc.det(*a, lam, c)
                worst_auto = max(worst_auto, float(abs(mp.mpc(ma.real, ma.imag) * mp.mpf(2) ** ea - ex) / abs(ex)))
            assert Ps[0] > Ps[1] > Ps[2]
    assert worst_ratio < 40.0, worst_ratio
    assert worst_auto < 1e-5, worst_auto


def test_S15pp_lid_first_change_by_brute_force(orc):
    """Algorithm 1 on the lid model from c = 0.5 m/s: the oracle's first
    change (idx 161) is the first change of the EXACT signs -- every mpmath sign from c_0 to
    c_160 equals sgn Re det(c_0), and c_161 differs -- while the fp64 instance alone flips at
    the first points (its sign at c = 0.5 disagrees with mpmath's on some wavelength)."""
    a = _lid_model()
    c = 0.5 * (np.arange(1000, dtype=np.float64) + 1.0)
    lam = 60.0
    st, ct, idx, nd = orc.curve(*a, [lam], c)
    assert st == 0 and int(idx[0]) == 161 and ct[0] == c[161]
    s0 = _mp_sign(a, lam, orc.perturb_velocity(a[1], a[2], c[0]))
    for j in list(range(0, 161, 8)) + [159, 160]:
        assert _mp_sign(a, lam, orc.perturb_velocity(a[1], a[2], c[j])) == s0, j
    assert _mp_sign(a, lam, orc.perturb_velocity(a[1], a[2], c[161])) != s0
    flips = 0
    for l in synth.geom(60.0, 0.8, 24)[:6]:
        m, e, _ = orc.det(*a, l, c[0], precision="fp64")
        flips += int(np.sign(m.real) != _mp_sign(a, l, c[0]))
    assert flips >= 1


# ------------------------------------------------------------------ P11 curve asymptotes

# P10 / reading S21: root or pole.  A soft layer (beta 100 m/s, 10 m) under a scan that starts
# above its shear velocity: its clamped-layer resonances (D -> 0, element entries -> inf) come
# first, interlaced with the system's roots.
SOFT_POLE = dict(h=[10.0], alpha=[200.0, 700.0], beta=[100.0, 350.0], rho=[1800.0, 2000.0])


def soft_pole_grid():
    return 100.5 + 0.25 * np.arange(400, dtype=np.float64)


@pytest.mark.parametrize("lam", [2.0, 10.0, 40.0])
def test_P10_fundamental_mode_changes_are_roots(orc, lam):
    """On the C2 model the first sign change is the fundamental mode: a root, |det| -> 0."""
    w = synth.workload("maswaves")
    m = w.models
    a = (m.h[0], m.alpha[0], m.beta[0], m.rho[0])
    st, ct, idx, _ = orc.curve(*a, np.array([lam]), w.c)
    j = int(idx[0])
    kind, cs, d = orc.classify_change(*a, lam, w.c[j - 1], w.c[j])
    assert kind == "root" and w.c[j - 1] < cs <= w.c[j] and d < -30


def test_P10_pole_first_is_an_element_singularity(orc):
    """The first change of the soft-layer model is a POLE, and there the layer element blows
    up (D_0 -> 0) while at the next change -- a root -- it stays moderate."""
    a = (SOFT_POLE["h"], SOFT_POLE["alpha"], SOFT_POLE["beta"], SOFT_POLE["rho"])
    c, lam = soft_pole_grid(), 1.0
    st, m, e, _ = orc.det_grid(*a, np.array([lam]), c)
    s = np.sign(m[0].real)
    ch = np.nonzero(s[1:] != s[:-1])[0] + 1
    st, ct, idx, _ = orc.curve(*a, np.array([lam]), c)
    assert idx[0] == ch[0]                                            # O7 on this grid
    k = 2.0 * math.pi / lam
    kinds, mags = [], []
    for j in ch[:4]:
        kind, cs, d = orc.classify_change(*a, lam, c[j - 1], c[j])
        kinds.append(kind)
        el = orc.layer_element(a[0][0], a[1][0], a[2][0], a[3][0], k, cs)
        mags.append(np.abs(el).max())
    assert kinds[0] == "pole" and "root" in kinds[1:]
    r = kinds.index("root")
    assert mags[0] > 1e9 * mags[r]


def test_P11_short_wavelength_tends_to_top_layer_rayleigh(orc):
    m = synth.maswaves_model()
    grid = synth.maswaves_grid()
    cr = rayleigh_root(1440.0, 75.0)
    j, cj = first_grid_above(grid, cr)
    st, ct, idx, nd = orc.curve(m.h[0], m.alpha[0], m.beta[0], m.rho[0], [0.1, 0.25, 0.5], grid)
    assert st == orc.OK
    assert list(idx) == [j] * 3 and cj == 72.0    # the paper's 72 m/s tier


def test_P11_long_wavelength_below_halfspace_rayleigh(orc):
    m = synth.maswaves_model()
    grid = synth.maswaves_grid()
    cr = rayleigh_root(1440.0, 290.0)
    st, ct, idx, nd = orc.curve(m.h[0], m.alpha[0], m.beta[0], m.rho[0], [100.0, 200.0, 600.0],
                                grid)
    assert st == orc.OK
    assert np.all(np.diff(ct) >= 0) and ct[-1] <= first_grid_above(grid, cr)[1]
    assert ct[-1] >= cr - 5.0


# ------------------------------------------------------------------ paper tiers (golden)

def test_paper_uniform_tiers_reproduced_by_maswaves_model(orc):
    """uniform curves whose wavelengths "match test velocities of 72, 238,
    and 256" — the C2 model reproduces each tier at the wavelengths in the fixture."""
    rows = [l.split() for l in open(f"{synth.GOLDEN_DIR}/paper_tiers.txt")
            if l.strip() and not l.startswith("#")]
    lam = [float(r[0]) for r in rows]
    want = [float(r[1]) for r in rows]
    m = synth.maswaves_model()
    st, ct, idx, nd = orc.curve(m.h[0], m.alpha[0], m.beta[0], m.rho[0], lam,
                                synth.maswaves_grid())
    assert list(ct) == want


# ------------------------------------------------------------------ P12 misfit (Algorithm 2)

def test_P12_misfit_examples(orc):
    assert orc.misfit([110.0], [100.0]) == (0, pytest.approx(0.10, abs=1e-15))
    assert orc.misfit([110.0, 90.0], [100.0, 100.0])[1] == pytest.approx(0.10, abs=1e-15)  # :231
    ce = synth.load_golden("c2_ct_oracle.txt")
    assert orc.misfit(ce, ce) == (0, 0.0)
    assert orc.misfit([np.nan, 1.0], [1.0, 1.0]) == (0, math.inf)
    assert orc.misfit([1.0], [0.0])[0] == orc.E_ARG
    assert orc.misfit([1.0], [np.inf])[0] == orc.E_NONFINITE


def test_P12_misfit_invariances(orc):
    rng = np.random.default_rng(12)
    for _ in range(100):
        L = int(rng.integers(1, 60))
        ct = rng.uniform(50, 300, L)
        ce = rng.uniform(50, 300, L)
        m0 = orc.misfit(ct, ce)[1]
        s = rng.uniform(0.1, 10)
        p = rng.permutation(L)
        assert abs(orc.misfit(s * ct, s * ce)[1] - m0) <= 1e-12 * m0
        assert abs(orc.misfit(ct[p], ce[p])[1] - m0) <= 1e-12 * m0
        assert abs(orc.misfit_ld(ct, ce)[1] - m0) <= 1e-13 * m0
        want = float(np.mean(np.abs(ct - ce) / ce))
        assert abs(m0 - want) <= 1e-13 * want


# ------------------------------------------------------------------ O0 validation, O9 ensemble

def test_validation_codes(orc):
    assert orc.validate_model([1.0], [300, 300], [100, 100], [1, 1]) == 0
    assert orc.validate_model([0.0], [300, 300], [100, 100], [1, 1]) == orc.E_MODEL
    assert orc.validate_model([1.0], [100, 300], [100, 100], [1, 1]) == orc.E_MODEL   # α = β
    assert orc.validate_model([1.0], [300, 300], [100, 100], [1, -1]) == orc.E_MODEL
    assert orc.validate_model([1.0], [300, 300], [np.nan, 100], [1, 1]) == orc.E_NONFINITE
    g = synth.maswaves_grid()
    m = synth.maswaves_model()
    a = (m.h[0], m.alpha[0], m.beta[0], m.rho[0])
    assert orc.curve(*a, [1.0], g[::-1])[0] == orc.E_GRID           # not increasing
    assert orc.curve(*a, [1.0], g[:1])[0] == orc.E_ARG              # V < 2
    assert orc.curve(*a, [-1.0], g)[0] == orc.E_GRID                # λ ≤ 0
    assert orc.curve(*a, [0.01], g)[0] == orc.E_RANGE               # k h > 350 (S9)
    assert orc.curve(*a, [1.0], np.r_[0.0, g])[0] == orc.E_GRID     # c0 ≤ 0


def test_ensemble_matches_per_model_curves_and_argmin(orc):
    w = synth.workload("ensemble", M=12)
    mods = w.models.take(list(range(11)) + [3])       # duplicate of model 3 ⇒ tie
    mods.h[5] = synth.maswaves_model().h[0].tolist() + [5.0]
    mods.alpha[5] = 1440.0
    mods.beta[5] = [75.0, 90.0, 150.0, 180.0, 240.0, 290.0, 290.0]   # the C2 twin ⇒ misfit 0
    mods.rho[5] = 1850.0
    out = orc.ensemble(mods, w.lam, w.c, w.ce)
    for m in range(12):
        st, ct, idx, nd = orc.curve(mods.h[m], mods.alpha[m], mods.beta[m], mods.rho[m], w.lam, w.c)
        assert np.array_equal(idx, out["idx"][m]) and np.array_equal(nd, out["ndet"][m])
        assert out["misfit"][m] == orc.misfit(ct, w.ce)[1]
    assert out["misfit"][5] == 0.0 and out["best"] == 5
    assert out["misfit"][11] == out["misfit"][3]
    empty = orc.ensemble(mods.slice(0, 0), w.lam, w.c, w.ce)
    assert empty["status"] == 0 and empty["best"] == -1


@pytest.mark.parametrize("seed", [0, 1])
def test_kappa_mask_golden_is_the_oracles(orc, seed):
    """tests/golden/kappa_mask_seed*.npz (the cached reading-S15' mask of the random det-parity
    sample, scripts/make_golden.py kappa) equals oracle.det_kappa <= 1e-10 at 48 random points
    and covers the sample the GPU test draws."""
    import synth

    g = np.load(os.path.join(synth.GOLDEN_DIR, f"kappa_mask_seed{seed}.npz"))
    shape = tuple(int(x) for x in g["shape"])
    mask = np.unpackbits(g["mask"])[: int(np.prod(shape))].reshape(shape) != 0
    assert shape == (20, 40, 256) and 0.9 < mask.mean() < 1.0
    w = synth.workload("ensemble", M=400)
    rng = np.random.default_rng(1000 + seed)
    for _ in range(48):
        t, i, j = (int(rng.integers(n)) for n in shape)
        mi = int(g["models"][t])
        a = tuple(x[mi] for x in (w.models.h, w.models.alpha, w.models.beta, w.models.rho))
        assert (orc.det_kappa(*a, float(w.lam[i]), float(g["c"][t][j])) <= 1e-10) == mask[t, i, j]
