"""Per-rank shard times of the single-curve configs (C3 uniform, C4 realistic) at the
modular wavelength partition of G = 1, 2, 4, 8 ranks, timed on one GPU for the automatic
kernel choice and forced pair / row scans (development aid; MASW_LIB selects a variant build).

    python scripts/shard_small_probe.py
"""
import sys, os, statistics
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2003_02256_b200 as masw, synth
from paper_2003_02256_b200 import distributed as D
dev = torch.device("cuda:0")
t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=dev)
for name, kw in (("uniform", {"tier": 200.0}), ("realistic", {})):
    w = synth.workload(name, **kw)
    m = w.models
    mod = [t(x[0]) for x in (m.h, m.alpha, m.beta, m.rho)]
    c = t(w.c)
    for G in (1, 2, 4, 8):
        parts = D.partition_wavelengths(len(w.lam), G, "modular")
        lam = t(w.lam[parts[0]])
        for label, fl in ((("auto", 0), ("pairs", masw.SCHED_PAIRS), ("rows", masw.SCHED_ROWS)) if not os.environ.get("AUTO_ONLY") else (("auto", 0),)):
            ts = []
            for k in range(6):
                masw.masw_curve(*mod, lam, c, flags=fl | masw.TIME_SCAN)
                torch.cuda.synchronize()
                if k: ts.append(masw.masw_last_scan_ms())
            print(f"{name:10s} G={G} rows={len(parts[0]):5d} {label:6s} {statistics.median(ts):7.3f} ms", flush=True)
