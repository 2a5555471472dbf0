"""Full C5 parity, once ("10 min full run, reported once"): every one of the
4,000,000 (model, lambda) rows of the 100k-model ensemble through the GPU scan bench.py times
and through the CPU oracle on all host cores; idx compared row by row, mismatches judged by
the S16 near-root rule, misfits within 1e-9.  Writes gpurun_out/c5_full_parity.json
(kept as profiles/r1/c5_full_parity.json)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import masw_parity as parity  # noqa: E402
import oracle  # noqa: E402
import paper_2003_02256_b200 as masw  # noqa: E402
import synth  # noqa: E402


def main():
    oracle.build()
    w = synth.workload("ensemble", M=100_000)
    m = w.models
    d = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda")
    r = masw.masw_curves_ensemble(*[d(x) for x in (m.h, m.alpha, m.beta, m.rho)], d(w.lam),
                                  d(w.c), d(w.ce))
    gidx, gmis = r.idx.cpu().numpy(), r.misfit.cpu().numpy()
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    o = oracle.ensemble(m, w.lam, w.c, w.ce, nthreads=cores)
    secs = time.perf_counter() - t0
    oidx, omis = o["idx"], o["misfit"]
    diff = gidx != oidx
    rows_bad = np.argwhere(diff)
    accepted = 0
    for mi, i in rows_bad:
        a = (m.h[mi], m.alpha[mi], m.beta[mi], m.rho[mi])
        ok, _, _ = parity.ct_acceptable(oracle, a, w.lam[i:i + 1], w.c, gidx[mi, i:i + 1],
                                        oidx[mi, i:i + 1])
        accepted += int(ok.all())
    same = gidx == oidx
    both_fin = np.isfinite(gmis) & np.isfinite(omis)
    rel = np.abs(gmis[both_fin] - omis[both_fin]) / np.maximum(np.abs(omis[both_fin]), 1e-300)
    models_exact = np.all(same, axis=1)
    out = {
        "rows": int(gidx.size), "rows_equal": int(same.sum()),
        "rows_different": int(diff.sum()), "different_accepted_by_S16": accepted,
        "misfit_models_compared": int(both_fin.sum()),
        "misfit_max_rel_err_on_exact_models": float(np.max(rel[models_exact[both_fin]])) if rel.size else 0.0,
        "misfit_inf_agree": bool(np.array_equal(np.isinf(gmis), np.isinf(omis))),
        "algorithmic_dets": int(o["ndet"].sum()), "oracle_seconds": secs, "oracle_threads": cores,
        "oracle_dets_per_s": float(o["ndet"].sum() / secs),
    }
    print(json.dumps(out, indent=1))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)   # copied to profiles/r1/
    with open(os.path.join(ROOT, "gpurun_out", "c5_full_parity.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
