"""Block-sign certificate threshold sweep (development aid; DESIGN.md "sign by block
recursion").  Run once per library variant built with -DMASW_BLOCK_MULT_EXP=E:

    MASW_LIB=build_variants/libmasw_m8.so python scripts/cert_sweep.py

Prints, for C5 and C4 and random layered models from the configs' 0.5 m/s grid start: scan
time (MASW_TIME_SCAN), GEPP re-evaluations (masw_last_fallbacks) and C_t indices compared
with the all-GEPP scan (MASW_PIVOTED) of the same library."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_02256_b200 as masw  # noqa: E402
import synth  # noqa: E402


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda")


def run(args, lam, c, fl, reps=3):
    ts, r = [], None
    for _ in range(reps):
        r = masw.masw_curves_ensemble(*args, lam, c, None, flags=masw.TIME_SCAN | fl)
        torch.cuda.synchronize()
        ts.append(masw.masw_last_scan_ms())
    return statistics.median(ts), masw.masw_last_fallbacks(), masw.masw_last_work(), r.idx


def main():
    out = {"lib": os.path.basename(masw.masw.LIB_PATH)}
    cases = []
    w = synth.workload("ensemble", M=100_000)
    cases.append(("C5", [dev(x) for x in (w.models.h, w.models.alpha, w.models.beta, w.models.rho)],
                  dev(w.lam), dev(w.c)))
    w4 = synth.workload("realistic")
    m4 = w4.models
    cases.append(("C4", [dev(x[:1]) for x in (m4.h, m4.alpha, m4.beta, m4.rho)], dev(w4.lam),
                  dev(w4.c)))
    lam = dev(synth.geom(60.0, 0.8, 24))
    c = dev(0.5 * (np.arange(1000, dtype=np.float64) + 1.0))
    for N in range(1, 9):
        mods = synth.random_models(4000, N, 500 + N)
        cases.append((f"random_N{N}", [dev(x) for x in (mods.h, mods.alpha, mods.beta, mods.rho)],
                      lam, c))
    for name, args, lm, cc in cases:
        t, fb, (alg, ev), idx = run(args, lm, cc, 0)
        tp, _, _, idxp = run(args, lm, cc, masw.PIVOTED, reps=1)
        diff = (idx != idxp)
        out[name] = {"scan_ms": t, "fallbacks": fb, "evaluated": ev, "alg": alg,
                     "fallback_rate": fb / max(ev, 1), "rows": int(idx.numel()),
                     "idx_differs_from_pivoted": int(diff.sum().item()),
                     "pivoted_scan_ms": tp}
        print(name, json.dumps(out[name]), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
