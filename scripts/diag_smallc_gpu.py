"""Reading S15'' diagnostic (GPU side): first-change indices of random layered models scanned
from the configs' 0.5 m/s grid start, default element vs the stable element (MASW_STABLE) vs
all-GEPP signs, for N = 1..8.  Writes gpurun_out/smallc_diag.npz; compared against the oracle
and mpmath on the CPU."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2003_02256_b200 as masw  # noqa: E402
import synth  # noqa: E402

out = {}
lam = synth.geom(60.0, 0.8, 24)
c = 0.5 * (np.arange(1000, dtype=np.float64) + 1.0)
for N, seed in [(1, 101), (2, 102), (3, 103), (4, 104), (5, 105), (6, 106), (7, 107), (8, 108)]:
    mods = synth.random_models(160, N, seed)
    for name, fl in [("models", masw.SCHED_MODELS), ("rows", masw.SCHED_ROWS),
                     ("stable", masw.STABLE | masw.SCHED_ROWS), ("pivoted", masw.PIVOTED | masw.SCHED_ROWS)]:
        r = masw.masw_curves_ensemble(mods.h, mods.alpha, mods.beta, mods.rho, lam, c, None, flags=fl)
        out[f"{name}_{N}"] = np.asarray(r.idx)
    w = synth.workload("ensemble", M=20000)
    m = w.models
    for name, fl in [("c5_models", masw.SCHED_MODELS), ("c5_stable", masw.STABLE | masw.SCHED_MODELS)]:
        r = masw.masw_curves_ensemble(m.h, m.alpha, m.beta, m.rho, w.lam, w.c, None, flags=fl)
        out[name] = np.asarray(r.idx)
np.savez(os.path.join(ROOT, "gpurun_out", "smallc_diag.npz"), **out)
print("ok", {k: int((v < 0).sum()) for k, v in out.items()})
