"""In-domain fractions of the det-parity tests (readings S15 + S15': c >= 0.5 beta_min,
|det| >= 1e-12 of its row maximum, kappa <= 1e-10), computed from the ORACLE only on exactly
the inputs tests/test_gpu_parity.py uses, so the tests' floors can sit just below the measured
fractions.  Writes profiles/r2/det_domain.json.

    python scripts/det_domain_fractions.py
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import masw_parity as parity  # noqa: E402
import oracle  # noqa: E402
import synth  # noqa: E402

# the random det-parity sample of test_det_parity_random_ensemble_points
RAND_MODELS, RAND_C = 20, 256


def frac(a, lam, c):
    st, om, oe, _ = oracle.det_grid(*a, lam, c)
    kap = oracle.det_grid_kappa(*a, lam, c)
    dom = parity.det_domain(om, oe, c, a[2].min(), kap)
    dom_s15 = parity.det_domain(om, oe, c, a[2].min(), None)
    return int(dom.sum()), int(dom.size), int(dom_s15.sum())


def main():
    out = {}
    t0 = time.time()
    for name in ("tiny", "maswaves", "maswaves_twin"):
        w = synth.workload(name)
        m = w.models
        a = (m.h[0], m.alpha[0], m.beta[0], m.rho[0])
        n, tot, n15 = frac(a, w.lam, w.c)
        out[name] = {"in_domain": n, "points": tot, "fraction": n / tot,
                     "fraction_S15_only": n15 / tot}
    m = synth.uniform_model()
    a = (m.h[0], m.alpha[0], m.beta[0], m.rho[0])
    n, tot, n15 = frac(a, np.array(synth.UNIFORM_TIERS), synth.uniform_grid()[::7])
    out["uniform_sample"] = {"in_domain": n, "points": tot, "fraction": n / tot,
                             "fraction_S15_only": n15 / tot}
    h = np.array([0.7, 9.0, 55.65])
    beta = np.array([150.0, 220.0, 300.0, 400.0])
    alpha = np.array([600.0, 800.0, 1000.0, 1440.0])
    rho = np.array([1800.0, 1850.0, 1900.0, 2000.0])
    n, tot, n15 = frac((h, alpha, beta, rho), np.array([1.0, 1.4, 2.5, 7.0]),
                       np.linspace(76.0, 600.0, 131))
    out["thick_layers"] = {"in_domain": n, "points": tot, "fraction": n / tot,
                           "fraction_S15_only": n15 / tot}
    w = synth.workload("ensemble", M=400)
    for seed in (0, 1):
        rng = np.random.default_rng(seed)
        n_all, tot_all, n15_all = 0, 0, 0
        for mi in rng.choice(400, RAND_MODELS, replace=False):
            a = tuple(x[mi] for x in (w.models.h, w.models.alpha, w.models.beta, w.models.rho))
            c = np.sort(rng.uniform(0.5 * a[2].min(), 500.0, RAND_C))
            n, tot, n15 = frac(a, w.lam, c)
            n_all += n
            tot_all += tot
            n15_all += n15
        out[f"random_ensemble_seed{seed}"] = {"in_domain": n_all, "points": tot_all,
                                              "fraction": n_all / tot_all,
                                              "fraction_S15_only": n15_all / tot_all,
                                              "sample": f"{RAND_MODELS} models x 40 lambda x "
                                                        f"{RAND_C} c"}
    out["seconds"] = time.time() - t0
    os.makedirs(os.path.join(ROOT, "profiles", "r2"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", "r2", "det_domain.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
