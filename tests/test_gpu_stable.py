"""the stable element (MASW_STABLE) against 50-digit mpmath.

The direct App. A formulas lose accuracy as c -> 0 (reading S15: the entries are O(c^4) /
O(c^2) differences of O(cosh^2) terms) and overflow for k h > ~350 (reading S9).  The
stable element rewrites every bracket in cancellation-free form and scales the hyperbolic
functions by e^-th.  The reference is mpmath at 50 digits
evaluating App. A on the same fp64 inputs (fp64 wavenumber fl(2 pi / lambda)), so only the
arithmetic differs -- the naive fp64 oracle is not accurate enough to judge this path.
"""
import numpy as np
import pytest

import synth
from test_oracle_pins import _mp_det

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def masw():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2003_02256_b200 as m

    m.lib()
    return m


def _grid_det(masw, a, lam, c, flags):
    re, im, ex = masw.masw_det_grid(*a, np.array([lam]), np.asarray(c, dtype=np.float64),
                                    flags=flags)
    return (re[0] + 1j * im[0]) * np.ldexp(1.0, ex[0])


def _rel_errors(masw, a, lam, cs, flags):
    import mpmath as mp

    got = _grid_det(masw, a, lam, cs, flags)
    out = []
    for g, c in zip(got, cs):
        want = _mp_det(*a, lam, float(c), k_double=True)
        g = mp.mpc(float(np.real(g)), float(np.imag(g)))
        out.append(float(abs(g - want) / abs(want)))
    return np.array(out)


FRACS = np.array([0.02, 0.05, 0.1, 0.2, 0.3, 0.5, 0.8])


@pytest.mark.parametrize("lam", [0.5, 5.0, 40.0, 100.0])
def test_stable_element_small_c_vs_mpmath(masw, lam):
    """c = 0.02 .. 0.8 beta_min on the C2 model: the stable element stays within 1e-11 of
    50-digit arithmetic where the direct formulas lose up to ~1e-3 (reading S15)."""
    m = synth.maswaves_model()
    a = (m.h[0], m.alpha[0], m.beta[0], m.rho[0])
    cs = FRACS * float(m.beta[0].min()) * (1.0 + 1e-7)     # off the S4 tolerance band
    err_s = _rel_errors(masw, a, lam, cs, masw.STABLE)
    assert err_s.max() < 1e-11, (lam, err_s)


def test_stable_element_fixes_what_the_direct_formulas_lose(masw):
    """The comparison is meaningful: at long wavelength and small c the default (direct)
    element is far from 50-digit arithmetic, the stable one is not."""
    m = synth.maswaves_model()
    a = (m.h[0], m.alpha[0], m.beta[0], m.rho[0])
    cs = np.array([0.02, 0.05, 0.1]) * float(m.beta[0].min()) * (1.0 + 1e-7)
    err_d = _rel_errors(masw, a, 100.0, cs, 0)
    err_s = _rel_errors(masw, a, 100.0, cs, masw.STABLE)
    assert err_d.max() > 1e-6 and err_s.max() < 1e-11, (err_d, err_s)


@pytest.mark.parametrize("seed", [0, 1])
def test_stable_element_random_models_vs_mpmath(masw, seed):
    """Random C5 models, random wavelengths, c from 0.02 beta_min to above alpha-ish values
    (all three wave cases) -- within 1e-10 of 50-digit arithmetic wherever the determinant is
    not at a root (|det| >= 1e-6 of its neighbours' scale)."""
    rng = np.random.default_rng(seed)
    w = synth.workload("ensemble", M=50)
    worst = 0.0
    for _ in range(6):
        mi = int(rng.integers(50))
        a = (w.models.h[mi], w.models.alpha[mi], w.models.beta[mi], w.models.rho[mi])
        lam = float(rng.choice(w.lam))
        bmin = float(a[2].min())
        cs = np.sort(np.r_[rng.uniform(0.02, 0.95, 4) * bmin, rng.uniform(1.05, 2.5, 2) * bmin])
        err = _rel_errors(masw, a, lam, cs, masw.STABLE)
        worst = max(worst, float(err.max()))
    assert worst < 1e-10, worst


def test_stable_element_thick_layers_beyond_the_direct_range(masw):
    """k h up to 700 (a 50 m layer at lambda = 0.5 m: k h = 628): the direct element is
    rejected (MASW_E_RANGE, cosh would overflow), the scaled one matches 50-digit arithmetic;
    beyond 700 both are rejected."""
    h = np.array([2.0, 50.0])
    beta = np.array([150.0, 220.0, 400.0])
    alpha = np.full(3, 1440.0)
    rho = np.array([1800.0, 1900.0, 2000.0])
    a = (h, alpha, beta, rho)
    cs = np.array([60.0, 120.0, 170.0, 260.0, 500.0])
    with pytest.raises(masw.MaswError) as e:
        masw.masw_det_grid(*a, np.array([0.5]), cs)
    assert e.value.code == masw.E_RANGE
    err = _rel_errors(masw, a, 0.5, cs, masw.STABLE)
    assert err.max() < 1e-10, err
    with pytest.raises(masw.MaswError) as e:
        masw.masw_det_grid(np.array([2.0, 60.0]), alpha, beta, rho, np.array([0.5]), cs,
                           flags=masw.STABLE)
    assert e.value.code == masw.E_RANGE


@pytest.mark.parametrize("name", ["tiny", "maswaves"])
def test_stable_scan_same_curves(masw, orc, name):
    """The scan with the stable element gives C_t within the parity rule of the oracle (the
    sign changes sit at c ~ 0.9 beta, where both elements are accurate)."""
    import masw_parity as parity

    w = synth.workload(name)
    a = (w.models.h[0], w.models.alpha[0], w.models.beta[0], w.models.rho[0])
    st, ct, idx = masw.masw_curve(*a, w.lam, w.c, flags=masw.STABLE)
    ost, oct_, oidx, ond = orc.curve(*a, w.lam, w.c)
    assert st == ost
    ok, exact, one = parity.ct_acceptable(orc, a, w.lam, w.c, idx, oidx)
    assert ok.all()


def test_stable_ensemble_matches_default_and_oracle(masw, orc):
    import masw_parity as parity

    w = synth.workload("ensemble", M=60)
    mods = w.models
    r = masw.masw_curves_ensemble(mods.h, mods.alpha, mods.beta, mods.rho, w.lam, w.c, w.ce,
                                  flags=masw.STABLE)
    o = orc.ensemble(mods, w.lam, w.c, w.ce)
    assert r.status == o["status"]
    for m in range(mods.n_models):
        a = (mods.h[m], mods.alpha[m], mods.beta[m], mods.rho[m])
        ok, exact, one = parity.ct_acceptable(orc, a, w.lam, w.c, r.idx[m], o["idx"][m])
        assert ok.all()


def test_small_c_false_change(masw, orc):
    """Reading S15'' at its extreme: a thin stiff lid (beta 491 m/s, 0.77 m) on a soft
    half-space (beta 81 m/s) scanned from c = 0.5 m/s (c / beta_lid = 0.001, k h = 0.08).
    50-digit mpmath puts Re det K at +1.04e32 at c = 0.5, 1.0 and 1.5 m/s (no sign change
    there); the direct App. A formulas' fp64 error scale there is P ~ 30, so their signs are
    noise (MASW_DIRECT, the round-1 default, reports a false change at index 1).  The DEFAULT
    path evaluates the small-c prefix with the stable element and returns the true first
    change 161 -- in every scan -- as do MASW_STABLE and the oracle (binary128 there)."""
    import mpmath  # noqa: F401

    mods = synth.random_models(160, 1, 101)
    a = tuple(x[28] for x in (mods.h, mods.alpha, mods.beta, mods.rho))
    lam = synth.geom(60.0, 0.8, 24)[:2]
    c = 0.5 * (np.arange(1000, dtype=np.float64) + 1.0)
    for cj in c[:3]:
        for l in lam:
            assert float(_mp_det(*a, float(l), float(cj), k_double=True).real) > 1e31
    ost, oct_, oidx, _ = orc.curve(*a, lam, c)
    assert ost == 0 and list(oidx) == [161, 161]
    for fl in (0, masw.SCHED_ROWS, masw.SCHED_PAIRS, masw.STABLE):
        st, ct, idx = masw.masw_curve(*a, lam, c, flags=fl)
        assert st == 0 and list(idx) == [161, 161], fl
    # the same model inside an ensemble (model-major scan, forced)
    M = np.repeat
    ens = [np.ascontiguousarray(M(x[None], 8, axis=0)) for x in a]
    r = masw.masw_curves_ensemble(*ens, lam, c, None, flags=masw.SCHED_MODELS)
    assert r.status == 0 and np.all(np.asarray(r.idx) == 161)
    rows, dets = masw.masw_last_prefix()
    assert rows == 16 and dets > 0
    # the direct element alone gets it wrong (the defect the prefix removes)
    st, ct, idx = masw.masw_curve(*a, lam, c, flags=masw.DIRECT)
    assert list(idx) != [161, 161]


def test_prefix_holds_the_whole_curve(masw, orc):
    """A 1 cm lid with a large P-wave velocity: Q_r reaches c* ~ 430 / 285 / 142 m/s at
    lambda = 60 / 40 / 20 m, so for the first two every grid point up to the first change
    (143.5 m/s) lies in the small-c prefix and the prefix kernel finds the change itself; for
    the third the scan finds it right after the prefix.  A short grid entirely inside
    the prefix without a change gives idx -1 (status WARN)."""
    a = ([0.01], [3000.0, 1000.0], [200.0, 150.0], [1900.0, 2000.0])
    lam = np.array([60.0, 40.0, 20.0])
    c = 1.0 + 0.5 * np.arange(400, dtype=np.float64)
    ost, oct_, oidx, _ = orc.curve(*a, lam, c)
    for fl in (0, masw.SCHED_ROWS, masw.SCHED_PAIRS, masw.STABLE):
        st, ct, idx = masw.masw_curve(*a, lam, c, flags=fl)
        assert st == ost and np.array_equal(np.asarray(idx), oidx), fl
    st, ct, idx = masw.masw_curve(*a, lam, c)
    rows, dets = masw.masw_last_prefix()
    assert rows == 3 and dets >= 2 * int(oidx[0] + 1)   # lambda = 60, 40: inside the prefix
    short = c[:60]
    ost, _, oidx2, _ = orc.curve(*a, lam, short)
    st, ct, idx = masw.masw_curve(*a, lam, short)
    assert st == ost == masw.WARN_NO_SIGN_CHANGE and list(idx) == list(oidx2) == [-1, -1, -1]


def _dev(x):
    return torch.as_tensor(np.ascontiguousarray(x), device="cuda")


def test_stable_all_scans_bitwise(masw):
    """MASW_STABLE through the row, model-major and pair scans: the same f-free stable
    elements in the same order -- identical idx and C_t (ensemble: rows vs model-major; one
    long curve: rows vs pairs)."""
    w = synth.workload("ensemble", M=300)
    m = w.models
    args = [_dev(x) for x in (m.h, m.alpha, m.beta, m.rho)] + [_dev(w.lam), _dev(w.c), _dev(w.ce)]
    rr = masw.masw_curves_ensemble(*args, flags=masw.STABLE | masw.SCHED_ROWS)
    rm = masw.masw_curves_ensemble(*args, flags=masw.STABLE | masw.SCHED_MODELS)
    assert rr.status == rm.status
    assert torch.equal(rr.idx, rm.idx) and torch.equal(rr.misfit, rm.misfit)
    r = synth.workload("realistic")
    a = [_dev(x[0]) for x in (r.models.h, r.models.alpha, r.models.beta, r.models.rho)]
    s1 = masw.masw_curve(*a, _dev(r.lam), _dev(r.c), flags=masw.STABLE | masw.SCHED_ROWS)
    s2 = masw.masw_curve(*a, _dev(r.lam), _dev(r.c), flags=masw.STABLE | masw.SCHED_PAIRS)
    assert s1.status == s2.status and torch.equal(s1.idx, s2.idx) and torch.equal(s1.ct, s2.ct)
    # and the default scan agrees on these configs (sign changes at c ~ 0.9 beta)
    d = masw.masw_curve(*a, _dev(r.lam), _dev(r.c))
    assert int((d.idx != s2.idx).sum()) <= 2
