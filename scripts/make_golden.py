"""Write the oracle-derived golden files under tests/golden/.

Calls ONLY oracle/ (never the CUDA path): every stored value is the CPU fp64 oracle's
C_t on a synth/ workload.  Re-run after any change to the oracle's arithmetic and cite
the passage that justifies the change in the commit message.

    python scripts/make_golden.py            # all files
    python scripts/make_golden.py c2         # one file
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402

OUT = synth.GOLDEN_DIR


def write_curve(fname, title, lam, idx, ct):
    with open(os.path.join(OUT, fname), "w") as fh:
        fh.write(f"# {title}\n")
        fh.write("# written by scripts/make_golden.py from oracle/ (CPU fp64, dense complex LU)\n")
        fh.write("# columns: i lambda_m idx ct_m_per_s\n")
        for i, (l, j, c) in enumerate(zip(lam, idx, ct)):
            fh.write(f"{i} {float(l)!r} {int(j)} {float(c)!r}\n")


def one_model_curve(w):
    m = w.models
    st, ct, idx, nd = oracle.curve(m.h[0], m.alpha[0], m.beta[0], m.rho[0], w.lam, w.c)
    assert st == oracle.OK, st
    return ct, idx, nd


def main(which):
    if "c1" in which:
        w = synth.workload("tiny")
        ct, idx, nd = one_model_curve(w)
        write_curve("c1_ct_oracle.txt", f"C1 tiny: oracle C_t, {int(nd.sum())} dets", w.lam, idx, ct)
    if "c2" in which:
        w = synth.workload("maswaves")
        ct, idx, nd = one_model_curve(w)
        write_curve("c2_ct_oracle.txt", f"C2 MASWaves-style N=5: oracle C_t, {int(nd.sum())} dets",
                    w.lam, idx, ct)
    if "c3" in which:
        m = synth.uniform_model()
        c = synth.uniform_grid()
        lam = np.array(synth.UNIFORM_TIERS)
        st, ct, idx, nd = oracle.curve(m.h[0], m.alpha[0], m.beta[0], m.rho[0], lam, c)
        assert st == oracle.OK
        with open(os.path.join(OUT, "c3_ct_oracle.txt"), "w") as fh:
            fh.write("# C3 uniform N=10 tiers: oracle C_t per distinct lambda (identical inputs give\n")
            fh.write("# identical outputs, so each of the 10k identical rows equals its tier's row)\n")
            fh.write("# columns: lambda_m idx ct_m_per_s\n")
            for l, j, v in zip(lam, idx, ct):
                fh.write(f"{float(l)!r} {int(j)} {float(v)!r}\n")
    if "c4" in which:
        w = synth.workload("realistic")
        t = time.time()
        ct, idx, nd = one_model_curve(w)
        print(f"c4: {time.time() - t:.1f}s, {int(nd.sum())} dets")
        write_curve("c4_ct_oracle.txt", f"C4 realistic N=5: oracle C_t, {int(nd.sum())} dets",
                    w.lam, idx, ct)
    if "kappa" in which:
        # reading S15': the kappa <= 1e-10 mask of the random det-parity sample of
        # tests/test_gpu_parity.py::test_det_parity_random_ensemble_points (the long-double
        # sensitivity analysis costs ~50 s per seed on 16 threads; the test recomputes the
        # oracle's determinants live and re-checks a random subset of this mask)
        w = synth.workload("ensemble", M=KAPPA_POOL)
        for seed in (0, 1):
            models, cs, masks = kappa_sample(w, seed)
            kap = []
            for mi, c in zip(models, cs):
                a = tuple(x[mi] for x in (w.models.h, w.models.alpha, w.models.beta, w.models.rho))
                kap.append(oracle.det_grid_kappa(*a, w.lam, c) <= KAPPA_MAX)
            np.savez_compressed(os.path.join(OUT, f"kappa_mask_seed{seed}.npz"),
                                models=np.asarray(models), c=np.asarray(cs),
                                mask=np.packbits(np.asarray(kap)),
                                shape=np.asarray(np.asarray(kap).shape),
                                note=np.asarray("kappa <= 1e-10 (reading S15'), oracle.det_grid_kappa; "
                                                "written by scripts/make_golden.py kappa"))


# the random det-parity sample (tests/test_gpu_parity.py): KAPPA_MODELS of the first
# KAPPA_POOL C5 models x C5's 40 lambda x KAPPA_C random c in [0.5 beta_min, 500]
KAPPA_POOL, KAPPA_MODELS, KAPPA_C, KAPPA_MAX = 400, 20, 256, 1e-10


def kappa_sample(w, seed):
    rng = np.random.default_rng(seed)
    models = [int(x) for x in rng.choice(KAPPA_POOL, KAPPA_MODELS, replace=False)]
    cs = []
    for mi in models:
        cs.append(np.sort(rng.uniform(0.5 * w.models.beta[mi].min(), 500.0, KAPPA_C)))
    return models, cs, None


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c3", "c4", "kappa"])
