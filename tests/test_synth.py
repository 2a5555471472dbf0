"""The seeded input generators (synth/) produce the shapes and value ranges of SURVEY.md §8(d)
and are deterministic (the oracle and the CUDA path read the same bytes)."""
import numpy as np
import pytest

import oracle
import synth


def test_geom_endpoints_and_monotone():
    g = synth.geom(40.0, 1.0, 40)
    assert g[0] == 40.0 and abs(g[-1] - 1.0) < 1e-14 and len(g) == 40
    assert np.all(np.diff(g) < 0)                      # decreasing "variable" curve


@pytest.mark.parametrize("name", ["tiny", "maswaves", "maswaves_twin", "uniform", "realistic"])
def test_single_model_workloads_valid(name):
    w = synth.workload(name)
    m = w.models
    assert m.n_models == 1
    assert oracle.validate_model(m.h[0], m.alpha[0], m.beta[0], m.rho[0]) == 0
    assert np.all(np.diff(w.c) > 0) and w.c[0] > 0
    assert np.all(w.lam > 0)
    if w.ce is not None:
        assert w.ce.shape == w.lam.shape and np.all(w.ce > 0)


def test_config_sizes():
    assert synth.workload("tiny").lam.shape == (20,) and synth.tiny_grid().shape == (1000,)
    assert synth.variable_lambdas().shape == (40,)     # PAPER.md:216 "40 entries"
    assert synth.uniform_grid().shape == (10_000,) and synth.realistic_grid().shape == (10_000,)
    assert synth.workload("uniform").lam.shape == (10_000,)
    assert synth.maswaves_model().n_layers == 5 and synth.maswaves_model(twin=True).n_layers == 6
    assert synth.uniform_model().n_layers == 10


def test_ensemble_deterministic_prefix_and_ranges():
    a = synth.ensemble_models(2000)
    b = synth.ensemble_models(2000)
    assert all(np.array_equal(x, y) for x, y in zip((a.h, a.alpha, a.beta, a.rho),
                                                    (b.h, b.alpha, b.beta, b.rho)))
    big = synth.ensemble_models(5000)
    assert np.array_equal(big.h[:2000], a.h) and np.array_equal(big.beta[:2000], a.beta)
    beta_ref = np.array([75.0, 90.0, 150.0, 180.0, 240.0, 290.0, 290.0])
    h_ref = np.array([1.0, 1.0, 2.0, 2.0, 4.0, 5.0])
    r = big.beta / beta_ref
    assert r.min() >= 0.6 and r.max() < 1.4
    rh = big.h / h_ref
    assert rh.min() >= 0.5 and rh.max() < 1.5
    assert big.rho.min() >= 1700 and big.rho.max() < 2000
    assert np.all(big.alpha > big.beta)
    assert big.h.flags["C_CONTIGUOUS"] and big.beta.flags["C_CONTIGUOUS"]


def test_golden_curves_match_their_configs():
    assert synth.load_golden("c1_ct_oracle.txt").shape == (20,)
    assert synth.load_golden("c2_ct_oracle.txt").shape == (40,)
    assert synth.load_golden("c4_ct_oracle.txt").shape == (10_000,)
    tiers = synth.load_golden_tiers()
    assert set(tiers) == set(synth.UNIFORM_TIERS)
    # the uniform tiers' C_t are the SURVEY §8(d) values (92.8 / 214.96 / 307.24 m/s)
    assert tiers[1.0] == 92.8 and tiers[30.0] == 214.96 and tiers[200.0] == 307.24


def test_perturbed_ce_is_nontrivial():
    ce = synth.load_golden("c2_ct_oracle.txt")
    p = synth.perturbed_ce(ce)
    assert p.shape == ce.shape and np.all(p > 0) and not np.array_equal(p, ce)
    assert np.max(np.abs(p / ce - 1)) <= 0.02 + 1e-15


def test_bench_flop_convention():
    import bench

    # 35N+30 elimination + 40N assembly + N divisions + 4N exp-class + 3
    assert bench.flops_per_det(6) == 513
    assert abs(bench.fp64_peak_tflops() - 37.22496) < 1e-9
