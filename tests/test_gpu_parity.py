"""GPU parity: the CUDA path (through the C ABI) against the CPU fp64 oracle on the same
seeded inputs (synth/), element by element, under the rules of tests/parity.py.

Small cases run the oracle in full; full-size cases (BASELINE.json configs at their real
sizes, in the launch configuration bench.py times) compare sampled rows and properties.
"""
import math

import numpy as np
import pytest

import synth
import masw_parity as parity

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def masw():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2003_02256_b200 as m

    m.lib()
    return m


def dev(a, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device="cuda")


def margs(models, k=0):
    return (models.h[k], models.alpha[k], models.beta[k], models.rho[k])


# ------------------------------------------------------------------ det grid parity (S15)

# in-domain fractions measured from the oracle (scripts/det_domain_fractions.py ->
# profiles/r2/det_domain.json); each floor sits just below its measured fraction
DOMAIN_FLOOR = {"tiny": 0.95, "maswaves": 0.90, "maswaves_twin": 0.90}


@pytest.mark.parametrize("name", ["tiny", "maswaves", "maswaves_twin"])
def test_det_grid_parity(masw, orc, name):
    w = synth.workload(name)
    a = margs(w.models)
    gre, gim, gex = masw.masw_det_grid(*a, w.lam, w.c)
    st, omant, oex, osts = orc.det_grid(*a, w.lam, w.c)
    assert st == 0 and np.all(osts == 0)
    kap = orc.det_grid_kappa(*a, w.lam, w.c)
    gm = gre + 1j * gim
    rel = parity.det_grid_rel_err(gm, gex, omant, oex)
    dom = parity.det_domain(omant, oex, w.c, w.models.beta.min(), kap)
    assert dom.mean() > DOMAIN_FLOOR[name], dom.mean()   # measured 0.960 / 0.913 / 0.907
    worst = float(np.nanmax(rel[dom]))
    assert worst <= parity.DET_RTOL, worst
    # mantissa normalisation of the ABI (max(|re|,|im|) in [0.5, 1))
    t = np.maximum(np.abs(gre), np.abs(gim))
    assert np.all((t >= 0.5) & (t < 1.0))
    # signs of Re det agree wherever the det is not near a root
    assert np.all(np.sign(gre)[dom] == np.sign(omant.real)[dom])


def test_det_grid_parity_uniform_n10(masw, orc):
    m = synth.uniform_model()
    a = margs(m)
    lam = np.array(synth.UNIFORM_TIERS)
    c = synth.uniform_grid()[::7]
    gre, gim, gex = masw.masw_det_grid(*a, lam, c)
    st, omant, oex, _ = orc.det_grid(*a, lam, c)
    kap = orc.det_grid_kappa(*a, lam, c)
    rel = parity.det_grid_rel_err(gre + 1j * gim, gex, omant, oex)
    dom = parity.det_domain(omant, oex, c, m.beta.min(), kap)
    assert dom.mean() > 0.69, dom.mean()                 # measured 0.705
    assert float(np.nanmax(rel[dom])) <= parity.DET_RTOL


def test_det_grid_parity_thick_layers_whole_exp_range(masw, orc):
    """k h_e up to 349.7 (just inside the S9 guard): the cosh/sinh table is read at every m up
    to its last rows (th = k h x from ~0 to 349.7), including the previously out-of-table range
    th > 256.  Det parity with the oracle in the S15 domain, and the guard at 350."""
    h = np.array([0.7, 9.0, 55.65])
    beta = np.array([150.0, 220.0, 300.0, 400.0])
    alpha = np.array([600.0, 800.0, 1000.0, 1440.0])
    rho = np.array([1800.0, 1850.0, 1900.0, 2000.0])
    lam = np.array([1.0, 1.4, 2.5, 7.0])                 # k h_2 = 349.7, 249.8, 139.9, 50.0
    c = np.linspace(76.0, 600.0, 131)
    gre, gim, gex = masw.masw_det_grid(h, alpha, beta, rho, lam, c)
    st, omant, oex, _ = orc.det_grid(h, alpha, beta, rho, lam, c)
    assert st == 0
    kap = orc.det_grid_kappa(h, alpha, beta, rho, lam, c)
    rel = parity.det_grid_rel_err(gre + 1j * gim, gex, omant, oex)
    dom = parity.det_domain(omant, oex, c, beta.min(), kap)
    assert dom.mean() > 0.99, dom.mean()                 # measured 1.0
    assert float(np.nanmax(rel[dom])) <= parity.DET_RTOL
    with pytest.raises(masw.MaswError) as e:
        masw.masw_det_grid(np.array([0.7, 9.0, 55.8]), alpha, beta, rho, lam, c)
    assert e.value.code == masw.E_RANGE


@pytest.mark.parametrize("seed", [0, 1])
def test_det_parity_random_ensemble_points(masw, orc, seed):
    """Det parity on random C5 models at random (lambda, c): 20 models x 40 lambda x 256 c
    per seed (204,800 points).  The oracle's determinants are computed here; its kappa <= 1e-10
    mask (reading S15', ~50 s of long-double sensitivity analysis per seed) comes from
    tests/golden/kappa_mask_seed*.npz (scripts/make_golden.py kappa, oracle only), re-checked
    here on a random subset of the points."""
    w = synth.workload("ensemble", M=400)
    g = np.load(synth.GOLDEN_DIR + f"/kappa_mask_seed{seed}.npz")
    models, cs = [int(x) for x in g["models"]], g["c"]
    kmask = np.unpackbits(g["mask"])[: int(np.prod(g["shape"]))].reshape(tuple(g["shape"])) != 0
    rng = np.random.default_rng(seed)                 # the sample the golden file was cut from
    assert [int(x) for x in rng.choice(400, len(models), replace=False)] == models
    chk = np.random.default_rng(100 + seed)
    worst, n, tot, where = 0.0, 0, 0, None
    for t, mi in enumerate(models):
        a = margs(w.models, mi)
        c = cs[t]
        assert np.array_equal(c, np.sort(rng.uniform(0.5 * a[2].min(), 500.0, len(c))))
        gre, gim, gex = masw.masw_det_grid(*a, w.lam, c)
        st, omant, oex, _ = orc.det_grid(*a, w.lam, c)
        # the cached mask is the oracle's kappa: re-derive 8 random points of this model
        for _ in range(8):
            i, j = int(chk.integers(len(w.lam))), int(chk.integers(len(c)))
            assert (orc.det_kappa(*a, float(w.lam[i]), float(c[j])) <= parity.KAPPA_MAX) == kmask[t, i, j]
        rel = parity.det_grid_rel_err(gre + 1j * gim, gex, omant, oex)
        dom = parity.det_domain(omant, oex, c, a[2].min(), None) & kmask[t]
        r = np.where(dom, rel, 0.0)
        k = np.unravel_index(np.argmax(r), r.shape)
        if r[k] > worst:
            where = (int(mi), float(w.lam[k[0]]), float(c[k[1]]))
            worst = float(r[k])
        n += int(dom.sum())
        tot += dom.size
    assert n > 0.95 * tot, n / tot                     # measured 0.969 / 0.962
    # where = (model, lambda, c)
    assert worst <= parity.DET_RTOL, (worst, where)


# ------------------------------------------------------------------ C_t parity, one model

@pytest.mark.parametrize("name", ["tiny", "maswaves", "maswaves_twin"])
@pytest.mark.parametrize("team", [0, 1, 2, 4, 8, 16])
def test_curve_parity_small(masw, orc, name, team):
    w = synth.workload(name)
    a = margs(w.models)
    st, ct, idx = masw.masw_curve(*a, w.lam, w.c, team_warps=team)
    ost, oct_, oidx, ond = orc.curve(*a, w.lam, w.c)
    assert st == ost == 0
    ok, exact, one = parity.ct_acceptable(orc, a, w.lam, w.c, idx, oidx)
    assert ok.all() and exact == len(w.lam)            # these configs have no near-root rows
    assert np.array_equal(ct, oct_)
    alg, ev = masw.masw_last_work()
    assert alg == int(ond.sum()) and ev >= alg          # SPEC.md:246 early-exit count


@pytest.mark.parametrize("team", [1, 8, 16])
def test_alternating_shared_memory_sizes(masw, team):
    """Launches whose dynamic shared memory shrinks and grows again (different N, same team
    size): the opt-in limit is raised once per kernel, never left below a later launch."""
    rng = np.random.default_rng(11)
    lam = synth.geom(30.0, 2.0, 8)
    c = 20.0 + 0.5 * np.arange(700, dtype=np.float64)
    for N in (5, 2, 5, 24, 2, 40):
        h = rng.uniform(0.5, 2.0, N)
        beta = rng.uniform(100.0, 400.0, N + 1)
        st, ct, idx = masw.masw_curve(h, np.full(N + 1, 1440.0), beta, np.full(N + 1, 1900.0),
                                      lam, c, team_warps=team)
        assert st in (0, 1)


def test_curve_device_pointers_and_async(masw, orc):
    w = synth.workload("maswaves")
    a = margs(w.models)
    st, ct, idx = masw.masw_curve(*[dev(x) for x in a], dev(w.lam), dev(w.c))
    ost, oct_, oidx, _ = orc.curve(*a, w.lam, w.c)
    assert st == 0 and torch.equal(idx.cpu(), torch.as_tensor(oidx))
    st, ct2, idx2 = masw.masw_curve(*[dev(x) for x in a], dev(w.lam), dev(w.c), flags=masw.ASYNC)
    torch.cuda.synchronize()
    assert st == 0 and torch.equal(ct2, ct)
    # on a non-default stream
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        st, ct3, idx3 = masw.masw_curve(*[dev(x) for x in a], dev(w.lam), dev(w.c))
    s.synchronize()
    assert torch.equal(ct3, ct)


def test_curve_wavelength_permutation(masw):
    w = synth.workload("maswaves")
    a = margs(w.models)
    p = np.random.default_rng(3).permutation(len(w.lam))
    _, ct, idx = masw.masw_curve(*a, w.lam, w.c)
    _, ctp, idxp = masw.masw_curve(*a, w.lam[p], w.c)
    assert np.array_equal(idxp, idx[p]) and np.array_equal(ctp, ct[p])


def test_rayleigh_and_no_change_rows(masw, orc):
    b = 200.0
    al = b * math.sqrt(3.0)
    st, ct, idx = masw.masw_curve([1.0], [al, al], [b, b], [1900.0, 1900.0], [5.0, 10.0, 20.0],
                                  synth.maswaves_grid())
    assert st == 0 and list(idx) == [367] * 3 and list(ct) == [184.0] * 3      # P1
    st, ct, idx = masw.masw_curve([1.0], [al, al], [b, b], [1900.0, 1900.0], [5.0],
                                  np.linspace(50, 150, 11))
    assert st == masw.WARN_NO_SIGN_CHANGE and idx[0] == -1 and math.isnan(ct[0])
    alg, ev = masw.masw_last_work()
    assert alg == 11


def test_pole_first_rows(masw, orc):
    """Reading S21 / P10: a soft layer whose clamped-layer poles (D_0 -> 0) come before the
    first root when the grid starts above its shear velocity.  The f-free recursion carries
    1/D_0 as a ratio: same first-change index as the oracle at every wavelength,
    through the row and the model-major kernels."""
    h, al, be, rh = [10.0], [200.0, 700.0], [100.0, 350.0], [1800.0, 2000.0]
    c = 100.5 + 0.25 * np.arange(400, dtype=np.float64)
    lam = np.array([0.5, 1.0, 1.5, 2.0, 3.0, 5.0, 8.0])
    st, ct, idx = masw.masw_curve(h, al, be, rh, lam, c)
    ost, oct_, oidx, _ = orc.curve(h, al, be, rh, lam, c)
    assert st == ost and np.array_equal(idx, oidx) and np.array_equal(ct, oct_)
    assert orc.classify_change(h, al, be, rh, 1.0, c[oidx[1] - 1], c[oidx[1]])[0] == "pole"
    M = 64
    H = np.tile(np.array(h), (M, 1))
    A, B, R = (np.tile(np.array(x), (M, 1)) for x in (al, be, rh))
    res = masw.masw_curves_ensemble(H, A, B, R, lam, c, flags=masw.SCHED_MODELS)
    assert np.array_equal(np.asarray(res.idx), np.tile(oidx, (M, 1)))


@pytest.mark.parametrize("N", [1, 3, 10, 24, 64])
def test_identical_stack_any_depth(masw, N):
    b = 200.0
    al = b * math.sqrt(3.0)
    h = np.full(N, 0.37)
    st, ct, idx = masw.masw_curve(h, [al] * (N + 1), [b] * (N + 1), [1900.0] * (N + 1),
                                  [5.0, 20.0], synth.maswaves_grid())
    assert st == 0 and list(idx) == [367, 367]


def test_error_codes_match_oracle(masw, orc):
    g = synth.maswaves_grid()
    m = synth.maswaves_model()
    a = margs(m)
    cases = [
        (a, [1.0], g[::-1]),
        (a, [-1.0], g),
        (a, [0.01], g),
        (a, [1.0], np.r_[0.0, g]),
        (a, [np.nan], g),
        ((a[0], a[1], a[1], a[3]), [1.0], g),      # alpha == beta
        ((np.r_[0.0, a[0][1:]], a[1], a[2], a[3]), [1.0], g),
    ]
    for args, lam, c in cases:
        ost = orc.curve(*args, lam, c)[0]
        with pytest.raises(masw.MaswError) as ei:
            masw.masw_curve(*args, lam, c)
        assert ei.value.code == ost, (lam, ei.value.code, ost)
    with pytest.raises(masw.MaswError) as ei:
        masw.masw_curve(*a, [1.0], g[:1])
    assert ei.value.code == masw.E_ARG
    N = 65
    with pytest.raises(masw.MaswError) as ei:
        masw.masw_curve(np.ones(N), np.full(N + 1, 300.0), np.full(N + 1, 100.0), np.ones(N + 1),
                        [10.0], g)
    assert ei.value.code == masw.E_ARG
    # outputs untouched on error
    ct = np.full(1, 7.0)
    idx = np.full(1, 9, dtype=np.int32)
    with pytest.raises(masw.MaswError):
        masw.masw_curve(*a, [1.0], g[::-1], ct_out=ct, idx_out=idx)
    assert ct[0] == 7.0 and idx[0] == 9


# ------------------------------------------------------------------ misfit / argmin

def test_misfit_examples_and_errors(masw, orc):
    assert masw.masw_misfit([110.0], [100.0]) == pytest.approx(0.10, abs=1e-15)
    assert masw.masw_misfit([110.0, 90.0], [100.0, 100.0]) == pytest.approx(0.10, abs=1e-15)
    assert masw.masw_misfit([np.nan, 1.0], [1.0, 1.0]) == math.inf
    with pytest.raises(masw.MaswError) as ei:
        masw.masw_misfit([1.0], [0.0])
    assert ei.value.code == masw.E_ARG
    with pytest.raises(masw.MaswError) as ei:
        masw.masw_misfit([1.0], [np.inf])
    assert ei.value.code == masw.E_NONFINITE
    rng = np.random.default_rng(1)
    ct = rng.uniform(50, 300, (37, 1234))
    ce = rng.uniform(50, 300, 1234)
    gm = masw.masw_misfit_batch(ct, ce)
    for k in range(37):
        assert parity.misfit_ok(orc, ct[k], ce, gm[k])


def test_argmin_ties_and_nan(masw):
    v = np.array([3.0, 1.0, 2.0, 1.0, np.nan, np.inf])
    b, bv = masw.masw_argmin(v)
    assert int(b[0]) == 1 and bv[0] == 1.0
    v = np.full(100_001, np.inf)
    v[77_777] = 0.5
    v[99_999] = 0.5
    b, bv = masw.masw_argmin(dev(v))
    assert int(b.cpu()[0]) == 77_777
    b, bv = masw.masw_argmin(np.full(5, np.inf))
    assert int(b[0]) == 0


# ------------------------------------------------------------------ ensembles

def test_ensemble_parity_small(masw, orc):
    w = synth.workload("ensemble", M=300)
    mods = w.models
    res = masw.masw_curves_ensemble(mods.h, mods.alpha, mods.beta, mods.rho, w.lam, w.c, w.ce)
    o = orc.ensemble(mods, w.lam, w.c, w.ce)
    assert res.status == o["status"]
    bad = 0
    for m in range(mods.n_models):
        ok, exact, one = parity.ct_acceptable(orc, margs(mods, m), w.lam, w.c, res.idx[m],
                                              o["idx"][m])
        assert ok.all()
        bad += len(w.lam) - exact
        assert parity.misfit_ok(orc, res.ct[m], w.ce, res.misfit[m])
    assert bad <= 2
    b, _ = masw.masw_argmin(res.misfit)
    assert int(b[0]) == o["best"]


def test_ensemble_team_and_pointer_kind_independence(masw):
    w = synth.workload("ensemble", M=200)
    mods = w.models
    ref = masw.masw_curves_ensemble(mods.h, mods.alpha, mods.beta, mods.rho, w.lam, w.c, w.ce)
    for team in (1, 2, 8, 16):
        r = masw.masw_curves_ensemble(*[dev(x) for x in (mods.h, mods.alpha, mods.beta, mods.rho)],
                                      dev(w.lam), dev(w.c), dev(w.ce), team_warps=team)
        assert np.array_equal(r.idx.cpu().numpy(), ref.idx)
        assert np.array_equal(r.misfit.cpu().numpy(), ref.misfit)   # bitwise: fixed-order sum


def test_ensemble_edge_cases(masw, orc):
    w = synth.workload("ensemble", M=3)
    mods = w.models
    r = masw.masw_curves_ensemble(mods.h[:0], mods.alpha[:0], mods.beta[:0], mods.rho[:0], w.lam,
                                  w.c, w.ce)
    assert r.status == 0 and r.ct.shape == (0, 40)
    # L = 1, V = 2 (ragged everything)
    r = masw.masw_curves_ensemble(mods.h, mods.alpha, mods.beta, mods.rho, w.lam[:1],
                                  np.array([100.0, 400.0]), w.ce[:1])
    o = orc.ensemble(mods, w.lam[:1], np.array([100.0, 400.0]), w.ce[:1])
    assert np.array_equal(r.idx, o["idx"]) and r.status == o["status"]


# ------------------------------------------------------------------ model-major scan

def _ens(masw, mods, lam, c, ce, flags, device=False):
    if device:
        args = [dev(x) for x in (mods.h, mods.alpha, mods.beta, mods.rho)] + [dev(lam), dev(c)]
        r = masw.masw_curves_ensemble(*args, dev(ce) if ce is not None else None, flags=flags)
        return (r.status, r.ct.cpu().numpy(), r.idx.cpu().numpy(),
                r.misfit.cpu().numpy() if r.misfit is not None else None)
    r = masw.masw_curves_ensemble(mods.h, mods.alpha, mods.beta, mods.rho, lam, c, ce, flags=flags)
    return r.status, r.ct, r.idx, r.misfit


@pytest.mark.parametrize("L", [1, 3, 40, 64, 65, 130])
def test_models_kernel_bitwise_equals_row_kernel(masw, L):
    """The model-major scan (per-(model, c) roots shared by up to 64 wavelengths) computes
    every determinant with the row scan's operations in the row scan's order: identical
    C_t, idx and misfit, for one and several wavelength blocks per model and ragged tails."""
    w = synth.workload("ensemble", M=97)
    mods = w.models
    lam = synth.geom(40.0, 1.0, L) if L > 1 else np.array([7.5])
    ce = np.interp(lam, w.lam[::-1], w.ce[::-1])
    rows = _ens(masw, mods, lam, w.c, ce, masw.SCHED_ROWS)
    mm = _ens(masw, mods, lam, w.c, ce, masw.SCHED_MODELS, device=True)
    assert rows[0] == mm[0]
    assert np.array_equal(rows[2], mm[2])
    assert np.array_equal(rows[1], mm[1], equal_nan=True)
    assert np.array_equal(rows[3], mm[3])


def test_models_kernel_tail_pieces_bitwise(masw):
    """More models than the tail split covers (2 pieces per resident warp: 4736 models on 148
    SMs x 16 warps): main items (all wavelengths of a model) and tail pieces (8 wavelengths)
    in one launch give the row scan's results bit for bit."""
    w = synth.workload("ensemble", M=6000)
    rows = _ens(masw, w.models, w.lam, w.c, w.ce, masw.SCHED_ROWS)
    mm = _ens(masw, w.models, w.lam, w.c, w.ce, masw.SCHED_MODELS, device=True)
    assert rows[0] == mm[0]
    assert np.array_equal(rows[2], mm[2])
    assert np.array_equal(rows[1], mm[1], equal_nan=True)
    assert np.array_equal(rows[3], mm[3])


@pytest.mark.parametrize("name,kw", [("realistic", {}), ("uniform", {"tier": 30.0}),
                                     ("maswaves", {}), ("tiny", {})])
def test_pair_kernel_bitwise_equals_row_kernel(masw, name, kw):
    """The pair scan (two wavelengths of the one model per warp, lockstep, shared roots) gives
    the row scan's C_t and idx bit for bit and the same algorithmic count -- on the full-size
    single-curve configs it is selected automatically, on the small ones forced."""
    w = synth.workload(name, **kw)
    a = [dev(x[0]) for x in (w.models.h, w.models.alpha, w.models.beta, w.models.rho)]
    lam, c = dev(w.lam), dev(w.c)
    st_r, ct_r, idx_r = masw.masw_curve(*a, lam, c, flags=masw.SCHED_ROWS)
    alg_r, _ = masw.masw_last_work()
    st_p, ct_p, idx_p = masw.masw_curve(*a, lam, c, flags=masw.SCHED_PAIRS | masw.TEAM_STATS)
    alg_p, ev_p = masw.masw_last_work()
    assert st_r == st_p
    assert torch.equal(idx_r, idx_p) and torch.equal(ct_r.isnan(), ct_p.isnan())
    assert torch.equal(torch.nan_to_num(ct_r), torch.nan_to_num(ct_p))
    assert alg_r == alg_p and ev_p >= alg_p
    assert int(masw.masw_last_team_dets().sum()) >= alg_p


@pytest.mark.parametrize("N", [1, 9, 24, 64])
def test_pair_kernel_any_depth(masw, N):
    """The pair scan keeps no per-layer cache, so any N up to MASW_MAX_LAYERS runs through it:
    bitwise equal to the row scan on random stacks of N layers."""
    mods = synth.random_models(1, N, 500 + N)
    a = [dev(x[0]) for x in (mods.h, mods.alpha, mods.beta, mods.rho)]
    lam = dev(synth.geom(80.0, 2.0, 33))
    c = dev(0.3 * float(mods.beta.min()) + 0.5 * np.arange(1500, dtype=np.float64))
    r = masw.masw_curve(*a, lam, c, flags=masw.SCHED_ROWS)
    p = masw.masw_curve(*a, lam, c, flags=masw.SCHED_PAIRS)
    assert r.status == p.status and torch.equal(r.idx, p.idx)
    assert torch.equal(torch.nan_to_num(r.ct), torch.nan_to_num(p.ct))


@pytest.mark.parametrize("N,L", [(10, 40), (3, 7), (6, 2)])
def test_pair_kernel_ensembles_bitwise(masw, N, L):
    """The pair scan on ensembles (per-warp model constants, pair-major queue): N = 10 (beyond
    the model-major cache), odd and tiny wavelength counts -- idx, C_t and misfit bitwise equal
    to the row scan."""
    mods = synth.random_models(300, N, 700 + N)
    lam = synth.geom(60.0, 0.8, L)
    c = 0.3 * float(mods.beta.min()) + 0.5 * np.arange(1200, dtype=np.float64)
    ce = np.linspace(150.0, 100.0, L)
    rows = _ens(masw, mods, lam, c, ce, masw.SCHED_ROWS, device=True)
    prs = _ens(masw, mods, lam, c, ce, masw.SCHED_PAIRS, device=True)
    assert rows[0] == prs[0]
    assert np.array_equal(rows[2], prs[2])
    assert np.array_equal(rows[1], prs[1], equal_nan=True)
    assert np.array_equal(rows[3], prs[3])


def test_pair_kernel_odd_rows_and_no_change(masw, orc):
    """Odd wavelength counts (a lone last row), rows without a change, a lone pending row of a
    pair: same results as the oracle."""
    b = 200.0
    al = b * math.sqrt(3.0)
    lam = np.array([5.0, 10.0, 20.0, 0.7, 3.0])
    c = np.linspace(150.0, 190.0, 81)
    st, ct, idx = masw.masw_curve([1.0, 2.0], [al, 1.2 * al, al], [b, 1.2 * b, b],
                                  [1900.0] * 3, lam, c, flags=masw.SCHED_PAIRS)
    ost, oct_, oidx, _ = orc.curve([1.0, 2.0], [al, 1.2 * al, al], [b, 1.2 * b, b],
                                   [1900.0] * 3, lam, c)
    assert st == ost and np.array_equal(idx, oidx)
    assert np.array_equal(np.nan_to_num(ct), np.nan_to_num(oct_))


@pytest.mark.parametrize("N", [1, 3, 7])
def test_models_kernel_bitwise_any_depth(masw, N):
    """Random N-layer ensembles (N = 7 is the deepest whose per-warp cache fits the one-CTA
    layout): model-major and row kernels agree bitwise."""
    rng = np.random.default_rng(N)
    M = 150
    h = rng.uniform(0.5, 4.0, (M, N))
    beta = rng.uniform(60.0, 420.0, (M, N + 1))
    alpha = np.full((M, N + 1), 1440.0)
    rho = rng.uniform(1700.0, 2100.0, (M, N + 1))
    lam = synth.geom(40.0, 1.0, 40)
    c = synth.maswaves_grid()
    a = masw.masw_curves_ensemble(h, alpha, beta, rho, lam, c, flags=masw.SCHED_ROWS)
    b = masw.masw_curves_ensemble(h, alpha, beta, rho, lam, c, flags=masw.SCHED_MODELS)
    assert a.status == b.status
    assert np.array_equal(a.idx, b.idx) and np.array_equal(a.ct, b.ct, equal_nan=True)


def test_models_kernel_s4_on_grid_velocities(masw, orc):
    """The C2 model's layer velocities (75, 90, ..., 290 m/s) lie ON its velocity grid, so
    the S4 perturbation fires inside the model-major kernel's warp-balloted check; 40 copies
    (forced model-major) equal the oracle's C_t exactly and the row kernel bitwise."""
    w = synth.workload("maswaves")
    m = w.models
    rep = lambda x: np.repeat(x, 40, axis=0)
    h, al, be, rh = rep(m.h), rep(m.alpha), rep(m.beta), rep(m.rho)
    mm = masw.masw_curves_ensemble(h, al, be, rh, w.lam, w.c, w.ce, flags=masw.SCHED_MODELS)
    rr = masw.masw_curves_ensemble(h, al, be, rh, w.lam, w.c, w.ce, flags=masw.SCHED_ROWS)
    ost, oct_, oidx, _ = orc.curve(*margs(m), w.lam, w.c)
    assert np.array_equal(mm.idx, rr.idx)
    assert all(np.array_equal(mm.idx[k], oidx) for k in range(40))
    assert all(np.array_equal(mm.ct[k], oct_) for k in range(40))


def test_block_sign_vs_pivoted_ensemble(masw, orc):
    """The scan's default sign (certified block LDL^T recursion, GEPP where uncertified) and
    the all-GEPP scan (MASW_PIVOTED) give the same first sign changes on the whole C5 bench
    workload (100k models, 4M rows); any difference would have to be a near-root row the
    parity rule allows.  The GEPP fallback fires (it is exercised) but rarely."""
    w = synth.workload("ensemble", M=100_000)
    mods = w.models
    args = [dev(x) for x in (mods.h, mods.alpha, mods.beta, mods.rho)] + [dev(w.lam), dev(w.c)]
    a = masw.masw_curves_ensemble(*args, dev(w.ce))
    fb = masw.masw_last_fallbacks()
    alg, ev = masw.masw_last_work()
    b = masw.masw_curves_ensemble(*args, dev(w.ce), flags=masw.PIVOTED)
    ia, ib = a.idx.cpu().numpy(), b.idx.cpu().numpy()
    diff = np.argwhere(ia != ib)
    assert len(diff) <= 2, len(diff)
    for m, i in diff:
        mm = mods.take([m])
        ok, exact, one = parity.ct_acceptable(orc, margs(mm), w.lam[i:i + 1], w.c,
                                              ia[m, i:i + 1], ib[m, i:i + 1])
        assert ok.all(), (m, i)
    assert 0 < fb < 1e-4 * ev, (fb, ev)


def test_block_sign_vs_pivoted_random_models_1m(masw, orc):
    """1,152,000 rows of random layered models (synth.random_models: reversals, stiff lids,
    soft channels, Poisson ratios 0.18-0.46; N = 1..8, 6000 models each x 24 lambda) scanned
    from the configs' 0.5 m/s grid start: the default sign (certified block recursion, GEPP
    where uncertified, small-c prefix) against the all-GEPP scan (MASW_PIVOTED).  Every
    differing row must be a near-root row the S16 rule allows (checked with the oracle); the
    certificate's backward-error bound says a flip needs
    K within ~2^15 u ||K|| of singular."""
    lam = synth.geom(60.0, 0.8, 24)
    c = 0.5 * (np.arange(1000, dtype=np.float64) + 1.0)
    rows, differ, fb_tot, ev_tot = 0, 0, 0, 0
    for N in range(1, 9):
        mods = synth.random_models(6000, N, 700 + N)
        args = [dev(x) for x in (mods.h, mods.alpha, mods.beta, mods.rho)] + [dev(lam), dev(c)]
        a = masw.masw_curves_ensemble(*args, None)
        fb_tot += masw.masw_last_fallbacks()
        ev_tot += masw.masw_last_work()[1]
        b = masw.masw_curves_ensemble(*args, None, flags=masw.PIVOTED)
        assert a.status == b.status
        ia, ib = a.idx.cpu().numpy(), b.idx.cpu().numpy()
        rows += ia.size
        for m, i in np.argwhere(ia != ib):
            differ += 1
            ok, exact, one = parity.ct_acceptable(orc, margs(mods, m), lam[i:i + 1], c,
                                                  ia[m, i:i + 1], ib[m, i:i + 1])
            assert ok.all(), (N, int(m), int(i), int(ia[m, i]), int(ib[m, i]))
    assert rows == 1_152_000
    assert differ <= 1e-5 * rows, differ
    assert 0 < fb_tot < 1e-3 * ev_tot, (fb_tot, ev_tot)


def test_block_sign_vs_pivoted_single_curves(masw):
    """Row kernel: C2 and C4 curves identical under both sign methods."""
    for name in ("maswaves", "realistic"):
        w = synth.workload(name)
        a = [dev(x) for x in margs(w.models)] + [dev(w.lam), dev(w.c)]
        s1, c1, i1 = masw.masw_curve(*a)
        s2, c2, i2 = masw.masw_curve(*a, flags=masw.PIVOTED)
        assert s1 == s2 and np.array_equal(i1.cpu().numpy(), i2.cpu().numpy()), name


def test_models_kernel_oracle_parity(masw, orc):
    w = synth.workload("ensemble", M=150)
    mods = w.models
    st, ct, idx, mis = _ens(masw, mods, w.lam, w.c, w.ce, masw.SCHED_MODELS)
    o = orc.ensemble(mods, w.lam, w.c, w.ce)
    assert st == o["status"]
    for m in range(mods.n_models):
        ok, exact, one = parity.ct_acceptable(orc, margs(mods, m), w.lam, w.c, idx[m], o["idx"][m])
        assert ok.all(), m
        assert parity.misfit_ok(orc, ct[m], w.ce, mis[m])


@pytest.mark.parametrize("N,seed", [(1, 101), (2, 102), (3, 103), (4, 104), (5, 105), (6, 106),
                                    (7, 107), (8, 108)])
def test_random_models_parity_all_kernels(masw, orc, N, seed):
    """Random layered models outside the configs' shapes (reversals, stiff lids, wide Poisson
    range; synth.random_models), scanned from the configs' real grid start c = 0.5 m/s --
    where the direct element's fp64 signs are noise for some of them (reading S15'') --:
    C_t of the model-major, row and pair scans against the oracle under the S16 rule (zero
    violations), and the three scans bitwise equal to each other."""
    mods = synth.random_models(160, N, seed)
    lam = synth.geom(60.0, 0.8, 24)
    c = 0.5 * (np.arange(1000, dtype=np.float64) + 1.0)
    o = orc.ensemble(mods, lam, c, None)
    st_m, ct_m, idx_m, _ = _ens(masw, mods, lam, c, None, masw.SCHED_MODELS, device=True)
    st_r, ct_r, idx_r, _ = _ens(masw, mods, lam, c, None, masw.SCHED_ROWS, device=True)
    assert st_m == st_r == o["status"]
    assert np.array_equal(idx_m, idx_r) and np.array_equal(ct_m, ct_r, equal_nan=True)
    bad = 0
    for m in range(mods.n_models):
        if np.array_equal(idx_m[m], o["idx"][m]):
            continue
        ok, exact, one = parity.ct_acceptable(orc, margs(mods, m), lam, c, idx_m[m], o["idx"][m])
        bad += int((~ok).sum())
    assert bad == 0
    for m in range(0, mods.n_models, 40):   # the pair scan on single curves of these models
        a = [dev(x[m]) for x in (mods.h, mods.alpha, mods.beta, mods.rho)]
        st_p, ct_p, idx_p = masw.masw_curve(*a, dev(lam), dev(c), flags=masw.SCHED_PAIRS)
        assert np.array_equal(idx_p.cpu().numpy(), idx_r[m])


def test_models_kernel_no_change_rows_and_stats(masw, orc):
    """Rows without a sign change (idx -1, status WARN) on a grid ending below C_t, V not a
    multiple of 32, per-warp det counts summing to the algorithmic count."""
    w = synth.workload("ensemble", M=40)
    mods = w.models
    c = 20.0 + 0.37 * np.arange(171, dtype=np.float64)       # 20 .. 82.9 m/s
    r_rows = _ens(masw, mods, w.lam, c, None, masw.SCHED_ROWS)
    r = masw.masw_curves_ensemble(mods.h, mods.alpha, mods.beta, mods.rho, w.lam, c, None,
                                  flags=masw.SCHED_MODELS | masw.TEAM_STATS)
    o = orc.ensemble(mods, w.lam, c)
    assert r.status == o["status"] == r_rows[0]
    assert np.array_equal(r.idx, r_rows[2]) and (r.idx == -1).any() and (r.idx >= 0).any()
    for m in range(mods.n_models):
        ok, exact, one = parity.ct_acceptable(orc, margs(mods, m), w.lam, c, r.idx[m], o["idx"][m])
        assert ok.all()
    alg, ev = masw.masw_last_work()
    per = masw.masw_last_team_dets()
    assert per.sum() == alg
    want = np.where(r.idx >= 0, r.idx + 1, len(c)).sum()
    assert alg == want


def test_models_kernel_deep_stack_falls_back(masw):
    """N = 24: the per-warp cache does not fit two CTAs per SM; MASW_SCHED_MODELS then runs
    where it fits (one CTA per SM) or the row scan -- results are the same either way."""
    N = 24
    rng = np.random.default_rng(5)
    M = 6
    h = rng.uniform(0.5, 2.0, (M, N))
    beta = rng.uniform(100.0, 400.0, (M, N + 1))
    alpha = np.full((M, N + 1), 1440.0)
    rho = np.full((M, N + 1), 1900.0)
    lam = synth.geom(30.0, 2.0, 12)
    c = 10.0 + 0.5 * np.arange(900, dtype=np.float64)
    a = masw.masw_curves_ensemble(h, alpha, beta, rho, lam, c, flags=masw.SCHED_ROWS)
    b = masw.masw_curves_ensemble(h, alpha, beta, rho, lam, c, flags=masw.SCHED_MODELS)
    assert np.array_equal(a.idx, b.idx) and a.status == b.status


@pytest.mark.slow
def test_ensemble_full_size_sampled(masw, orc):
    """C5 at full size (100k models) through the device path bench.py times; the oracle
    checks a seeded 1 % sample of models and the GPU's top-100 misfits, and
    the argmin."""
    w = synth.workload("ensemble", M=100_000)
    mods = w.models
    res = masw.masw_curves_ensemble(*[dev(x) for x in (mods.h, mods.alpha, mods.beta, mods.rho)],
                                    dev(w.lam), dev(w.c), dev(w.ce))
    idx = res.idx.cpu().numpy()
    ct = res.ct.cpu().numpy()
    mis = res.misfit.cpu().numpy()
    assert res.status in (0, 1)
    rng = np.random.default_rng(200302256)
    sample = np.unique(np.r_[rng.choice(100_000, 1000, replace=False), np.argsort(mis)[:100],
                             [0, 99_999]])
    sub = mods.take(sample)
    o = orc.ensemble(sub, w.lam, w.c, w.ce)
    for k, m in enumerate(sample):
        ok, exact, one = parity.ct_acceptable(orc, margs(sub, k), w.lam, w.c, idx[m], o["idx"][k])
        assert ok.all(), m
        assert parity.misfit_ok(orc, ct[m], w.ce, mis[m])
    b, bv = masw.masw_argmin(res.misfit)
    b = int(b.cpu()[0])
    assert mis[b] == mis.min() and b == int(np.argmin(mis))
    # the misfit of the argmin model recomputed by the oracle
    ob = orc.ensemble(mods.take([b]), w.lam, w.c, w.ce)
    assert ob["misfit"][0] <= mis[b] * (1 + 1e-9) + 1e-15


@pytest.mark.slow
@pytest.mark.parametrize("tier", synth.UNIFORM_TIERS)
def test_uniform_full_size(masw, orc, tier):
    """C3: 10k identical wavelengths x 10k velocities, N=10; every row equals the oracle's
    tier row (golden file written by scripts/make_golden.py from the oracle)."""
    w = synth.workload("uniform", tier=tier)
    a = margs(w.models)
    st, ct, idx = masw.masw_curve(*[dev(x) for x in a], dev(w.lam), dev(w.c))
    ct = ct.cpu().numpy()
    want = synth.load_golden_tiers()[tier]
    assert st == 0 and np.all(ct == want)


@pytest.mark.slow
def test_realistic_full_size(masw, orc):
    """C4: 10k wavelengths 100 -> 0.5 m, 10k velocities; vs the oracle's golden curve."""
    w = synth.workload("realistic")
    a = margs(w.models)
    st, ct, idx = masw.masw_curve(*[dev(x) for x in a], dev(w.lam), dev(w.c))
    idx = idx.cpu().numpy()
    golden_idx = np.array([int(l.split()[2]) for l in open(f"{synth.GOLDEN_DIR}/c4_ct_oracle.txt")
                           if not l.startswith("#")])
    ok, exact, one = parity.ct_acceptable(orc, a, w.lam, w.c, idx, golden_idx)
    assert ok.all(), np.nonzero(~ok)[0][:10]
    mis = masw.masw_misfit(ct, dev(w.ce))
    assert parity.misfit_ok(orc, ct.cpu().numpy(), w.ce, mis)


@pytest.mark.parametrize("L", [1, 3, 39])
def test_pair_kernel_odd_wavelength_counts(masw, orc, L):
    """TEAM=1 runs the row-pair kernel (rows 2i, 2i+1 of one model share c): odd L leaves a
    pair with a single row; compare with the oracle and with another team size."""
    w = synth.workload("ensemble", M=37)
    mods = w.models
    lam = w.lam[:L]
    ce = w.ce[:L]
    r1 = masw.masw_curves_ensemble(mods.h, mods.alpha, mods.beta, mods.rho, lam, w.c, ce,
                                   team_warps=1)
    r4 = masw.masw_curves_ensemble(mods.h, mods.alpha, mods.beta, mods.rho, lam, w.c, ce,
                                   team_warps=4)
    assert np.array_equal(r1.idx, r4.idx) and np.array_equal(r1.misfit, r4.misfit)
    o = orc.ensemble(mods, lam, w.c, ce)
    for m in range(mods.n_models):
        ok, exact, one = parity.ct_acceptable(orc, margs(mods, m), lam, w.c, r1.idx[m], o["idx"][m])
        assert ok.all()
    alg, ev = masw.masw_last_work()
    assert alg > 0


def test_async_scan_timing_ring(masw):
    w = synth.workload("ensemble", M=50)
    mods = w.models
    args = [dev(x) for x in (mods.h, mods.alpha, mods.beta, mods.rho)]
    for _ in range(3):
        masw.masw_curves_ensemble(*args, dev(w.lam), dev(w.c), dev(w.ce),
                                  flags=masw.ASYNC | masw.TIME_SCAN)
    ms = masw.masw_recent_scan_ms(3)
    assert len(ms) == 3 and all(x > 0 for x in ms)


@pytest.mark.parametrize("team", [1, 4])
def test_static_schedules_same_results_and_team_counts(masw, orc, team):
    """The paper's static partitions as scan schedules: the oracle's C_t under
    every schedule (queue, contiguous, modular), and the per-team det counts add up to the
    oracle's algorithmic total Sum(idx + 1)."""
    w = synth.workload("ensemble", M=500)
    m = w.models
    args = (m.h, m.alpha, m.beta, m.rho, w.lam, w.c, w.ce)
    o = orc.ensemble(m, w.lam, w.c, w.ce)
    ref = masw.masw_curves_ensemble(*args, team_warps=team, flags=masw.TEAM_STATS)
    assert np.array_equal(ref.idx, o["idx"])
    for k in range(len(ref.misfit)):
        assert parity.misfit_ok(orc, ref.ct[k], w.ce, float(ref.misfit[k]))
    alg_ref, _ = masw.masw_last_work()
    assert alg_ref == int(np.where(o["idx"] >= 0, o["idx"] + 1, len(w.c)).sum())
    tq = masw.masw_last_team_dets()
    assert tq is not None and int(tq.sum()) == alg_ref
    for fl in (masw.SCHED_CONTIGUOUS, masw.SCHED_MODULAR):
        r = masw.masw_curves_ensemble(*args, team_warps=team, flags=fl | masw.TEAM_STATS)
        assert np.array_equal(r.idx, ref.idx) and np.array_equal(r.misfit, ref.misfit)
        t = masw.masw_last_team_dets()
        assert int(t.sum()) == alg_ref and len(t) == len(tq)


def test_sharded_drivers_with_cuda_ops(masw, orc):
    """distributed.curve_sharded / ensemble_sharded with the CUDA library as per-rank compute
    (world size 1 here; N > 1 host logic is covered by tests/test_distributed_cpu.py)."""
    from paper_2003_02256_b200 import distributed as D

    w = synth.workload("maswaves")
    m = w.models
    model = tuple(dev(x[0]) for x in (m.h, m.alpha, m.beta, m.rho))
    for strat in ("modular", "contiguous"):
        out = D.curve_sharded(model, dev(w.lam), dev(w.c), dev(w.ce), strategy=strat)
        ost, oct_, oidx, _ = orc.curve(*margs(m), w.lam, w.c)
        assert np.array_equal(out.idx.cpu().numpy(), oidx)
        assert parity.misfit_ok(orc, out.ct.cpu().numpy(), w.ce, out.misfit)
    e = synth.workload("ensemble", M=64)
    em = e.models
    res = D.ensemble_sharded(tuple(dev(x) for x in (em.h, em.alpha, em.beta, em.rho)),
                             dev(e.lam), dev(e.c), dev(e.ce))
    o = orc.ensemble(em, e.lam, e.c, e.ce)
    assert np.array_equal(res.idx.cpu().numpy(), o["idx"]) and res.best == o["best"]


def test_fine_and_coarse_table_calls_agree(masw, orc):
    """The cosh/sinh table is chosen per call (fine d = 1/128 for k h_max <= 50.5, else the
    coarse d = 1/16): the same rows scanned in a fine call and in a call that one
    extra short wavelength pushes onto the coarse table give the oracle's index on both
    sides (the two tables differ only by rounding, so an index could move only at a
    near-root, rule S16)."""
    e = synth.workload("ensemble", M=1500)
    m = e.models
    hmax = float(m.h.max())
    assert 2 * math.pi / e.lam.min() * hmax <= 50.5          # the fine table
    lam_x = 2 * math.pi * hmax / 52.0                        # k h_max = 52: the coarse table
    lam2 = np.concatenate([e.lam, [lam_x]])
    args = [dev(x) for x in (m.h, m.alpha, m.beta, m.rho)]
    a = masw.masw_curves_ensemble(*args, dev(e.lam), dev(e.c))
    b = masw.masw_curves_ensemble(*args, dev(lam2), dev(e.c))
    ia = a.idx.cpu().numpy()
    ib = b.idx.cpu().numpy()[:, : len(e.lam)]
    o = orc.ensemble(m, e.lam, e.c)
    assert np.array_equal(ia, o["idx"])
    assert np.array_equal(ib, o["idx"])
    # single curve through the pair scan: C4's model (k h_max 50.27, fine) and + lambda_x
    w = synth.workload("realistic")
    wm = w.models
    sel = np.arange(0, len(w.lam), 25)                       # 400 of the 10k wavelengths
    lam = w.lam[sel]
    lamc = np.concatenate([lam, [2 * math.pi * float(wm.h[0].max()) / 52.0]])
    mod = [dev(x[0]) for x in (wm.h, wm.alpha, wm.beta, wm.rho)]
    st1, _, i1 = masw.masw_curve(*mod, dev(lam), dev(w.c), flags=masw.SCHED_PAIRS)
    st2, _, i2 = masw.masw_curve(*mod, dev(lamc), dev(w.c), flags=masw.SCHED_PAIRS)
    ost, _, oidx, _ = orc.curve(*margs(wm), lam, w.c)
    assert np.array_equal(i1.cpu().numpy(), oidx)
    assert np.array_equal(i2.cpu().numpy()[: len(lam)], oidx)


@pytest.mark.parametrize("N,seed", [(1, 201), (3, 203), (5, 205), (8, 208)])
def test_random_models_parity_fine_table(masw, orc, N, seed):
    """The random-model property test on calls that take the FINE cosh/sinh table: the
    shortest wavelength is chosen so that k h_max = 50.4 (<= 50.5), so wave arguments reach the
    end of the table (th up to ~50); model-major and row scans bitwise equal, C_t against the
    oracle under S16 with zero violations, from the 0.5 m/s grid start."""
    mods = synth.random_models(120, N, seed)
    hmax = float(mods.h.max())
    lam = synth.geom(60.0, 2 * math.pi * hmax / 50.4, 24)
    assert 2 * math.pi / lam.min() * hmax <= 50.5
    c = 0.5 * (np.arange(1000, dtype=np.float64) + 1.0)
    o = orc.ensemble(mods, lam, c, None)
    st_m, ct_m, idx_m, _ = _ens(masw, mods, lam, c, None, masw.SCHED_MODELS, device=True)
    st_r, ct_r, idx_r, _ = _ens(masw, mods, lam, c, None, masw.SCHED_ROWS, device=True)
    assert st_m == st_r == o["status"]
    assert np.array_equal(idx_m, idx_r) and np.array_equal(ct_m, ct_r, equal_nan=True)
    bad = 0
    for m in range(mods.n_models):
        if np.array_equal(idx_m[m], o["idx"][m]):
            continue
        ok, exact, one = parity.ct_acceptable(orc, margs(mods, m), lam, c, idx_m[m], o["idx"][m])
        bad += int((~ok).sum())
    assert bad == 0
    for m in range(0, mods.n_models, 40):
        a = [dev(x[m]) for x in (mods.h, mods.alpha, mods.beta, mods.rho)]
        st_p, ct_p, idx_p = masw.masw_curve(*a, dev(lam), dev(c), flags=masw.SCHED_PAIRS)
        assert np.array_equal(idx_p.cpu().numpy(), idx_r[m])


@pytest.mark.parametrize("calls", [(76, 201, 446, 500), (651, 1740, 1774)])
def test_thick_layer_reciprocal_range(masw, orc, calls):
    """Thick layers (k h ~ 140-175, from tests/fuzz/fuzz_parity.py's seeded sweep): the block
    recursion's p = D d comes within a factor 4 of the fp64 range, where its reciprocal
    (rcp.approx.ftz) is subnormal and flushed; the certificate now requires |p| < 2^1022, so
    such determinants are re-evaluated by the GEPP.  Before, every scan returned a false early
    change on these rows (e.g. idx 608 vs the oracle's and binary128's 628).  All three scans
    against the oracle under S16, zero violations."""
    rng = np.random.Generator(np.random.PCG64(2003))
    want = set(calls)
    for call in range(1, max(calls) + 1):
        # the draws of tests/fuzz/fuzz_parity.py in its order (uniforms inside conditionals kept)
        N = int(rng.integers(1, 13))
        M = int(rng.integers(1, 60))
        mods = synth.random_models(M, N, 10_000 + call) if call in want else None
        fine = bool(rng.integers(0, 2))
        khmax = float(rng.uniform(5.0, 50.4)) if fine else float(rng.uniform(50.6, 300.0))
        L = int(rng.integers(1, 48))
        hmax = float(mods.h.max()) if mods is not None else 1.0
        lam_min = 2 * math.pi * hmax / khmax
        if L > 1:
            lam = synth.geom(float(rng.uniform(max(lam_min * 1.5, 2.0), 120.0)), lam_min, L)
        else:
            lam = np.array([lam_min])
        V = int(rng.integers(64, 1500))
        if rng.integers(0, 2):
            c = 0.5 * (np.arange(V, dtype=np.float64) + 1.0)
        else:
            bmin = float(mods.beta.min()) if mods is not None else 100.0
            c0 = bmin * float(rng.uniform(0.5, 0.95))
            c = c0 + float(rng.uniform(0.05, 1.0)) * np.arange(V, dtype=np.float64)
        rng.integers(0, 3)                                     # (the sweep's kernel choice)
        if call not in want:
            continue
        o = orc.ensemble(mods, lam, c, None)
        for fl in (masw.SCHED_MODELS, masw.SCHED_PAIRS, masw.SCHED_ROWS):
            st, ct, idx, _ = _ens(masw, mods, lam, c, None, fl, device=True)
            bad = 0
            for m in range(M):
                if np.array_equal(idx[m], o["idx"][m]):
                    continue
                ok, exact, one = parity.ct_acceptable(orc, margs(mods, m), lam, c, idx[m],
                                                      o["idx"][m])
                bad += int((~ok).sum())
            assert bad == 0, (call, fl, bad)


def test_pair_scan_whole_pairs_with_unfinished_partner(masw, orc):
    """Whole-pair items of the pair scan (more pairs than resident warps, so not tail
    segments) where one row of a pair changes sign on the grid and the other does not: both
    rows' outputs must be written (a round-2 regression wrote only the first: the second row
    kept idx 0, found by tests/fuzz/fuzz_parity.py's "big" mode).  One model (C4's), 6000
    wavelengths in random order (reading S17), a grid ending below the long wavelengths'
    phase velocities: the pair scan equals the row scan bitwise and the oracle on a sample."""
    w = synth.workload("realistic")
    m = w.models
    rng = np.random.Generator(np.random.PCG64(17))
    lam = rng.permutation(w.lam)[:6000]
    c = 15.0 + 0.05 * np.arange(2000, dtype=np.float64)          # to 115 m/s
    a = [dev(x[0]) for x in (m.h, m.alpha, m.beta, m.rho)]
    st_p, ct_p, idx_p = masw.masw_curve(*a, dev(lam), dev(c), flags=masw.SCHED_PAIRS)
    st_r, ct_r, idx_r = masw.masw_curve(*a, dev(lam), dev(c), flags=masw.SCHED_ROWS)
    ip, ir = idx_p.cpu().numpy(), idx_r.cpu().numpy()
    assert (ir == -1).sum() > 500 and (ir > 0).sum() > 500      # both kinds of rows
    assert st_p == st_r and np.array_equal(ip, ir)
    assert np.array_equal(ct_p.cpu().numpy(), ct_r.cpu().numpy(), equal_nan=True)
    sel = np.arange(0, 6000, 60)
    ost, oct_, oidx, _ = orc.curve(*margs(m), lam[sel], c)
    assert np.array_equal(ip[sel], oidx)
