"""Mid-size ensembles: row vs pair vs model-major scans (development aid; MS=2000,8000)."""
import os, sys, statistics
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2003_02256_b200 as masw, synth
d = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda")
cases = [(f"C5-like M={M} N=6", synth.workload("ensemble", M=M).models)
         for M in [int(x) for x in os.environ.get("MS", "2000,8000").split(",")]]
if not os.environ.get("MS"):
    cases.append(("random M=3000 N=10", synth.random_models(3000, 10, 9)))
for name, mods in cases:
    w = synth.workload("ensemble", M=10)
    lam, c = d(w.lam), d(0.5 * (np.arange(1000) + 1.0) + 0.3 * float(mods.beta.min()))
    args = [d(x) for x in (mods.h, mods.alpha, mods.beta, mods.rho)]
    for fl, lab in ((masw.SCHED_ROWS, "rows"), (masw.SCHED_PAIRS, "pairs"), (masw.SCHED_MODELS, "models")):
        for _ in range(2): masw.masw_curves_ensemble(*args, lam, c, flags=fl | masw.TIME_SCAN)
        ts = []
        for _ in range(5):
            masw.masw_curves_ensemble(*args, lam, c, flags=fl | masw.TIME_SCAN); ts.append(masw.masw_last_scan_ms())
        alg, _ = masw.masw_last_work()
        t = statistics.median(ts)
        print(f"{name:22s} {lab:7s} {t:8.3f} ms {alg / t / 1e6:7.2f} Gdet/s", flush=True)
