"""load balance of the wavelength scan.

Within one GPU: kernel time and per-team det counts of the work-stealing queue vs the
paper's static contiguous / modular partitions (over the kernel's teams), on C4 (one
decreasing 10k-wavelength curve) and C5 (ensemble).

Across G workers (GPUs / MPI ranks, G = 1..8): the paper's experiment on the variable-40
curve (C2) and on C4: wavelengths partitioned contiguously or modularly over G workers; each
worker's algorithmic det count (sum of idx+1 over its wavelengths) and its measured device
time (masw_curve on its wavelength subset, median of reps) on this GPU; the simulated
parallel time is the max over workers and the speedup is relative to G = 1.  (One GPU is
available to this build, so the G-worker times are measured per worker, not concurrently.)

    python scripts/load_balance.py [out.json]
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_02256_b200 as masw  # noqa: E402
from paper_2003_02256_b200 import distributed as D  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=dev)


def time_ms(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def within_gpu(name, w, team):
    m = w.models
    args = [t(x) for x in (m.h, m.alpha, m.beta, m.rho)]
    lam, c = t(w.lam), t(w.c)
    out = {}
    for label, fl in (("queue", 0), ("contiguous", masw.SCHED_CONTIGUOUS),
                      ("modular", masw.SCHED_MODULAR)):
        call = lambda: masw.masw_curves_ensemble(*args, lam, c, team_warps=team,
                                                 flags=fl | masw.TIME_SCAN)
        time_ms(call, reps=1)
        scans = []
        for _ in range(3):
            call()
            scans.append(masw.masw_last_scan_ms())
        masw.masw_curves_ensemble(*args, lam, c, team_warps=team, flags=fl | masw.TEAM_STATS)
        td = masw.masw_last_team_dets().astype(np.float64)
        out[label] = {"scan_ms": statistics.median(scans), "teams": int(len(td)),
                      "team_dets_max_over_mean": float(td.max() / td.mean()),
                      "team_dets_cv": float(td.std() / td.mean())}
    return out


def across_workers(name, w, reps):
    m = w.models
    args = [t(x[0]) for x in (m.h, m.alpha, m.beta, m.rho)]
    c = t(w.c)
    st, ct, idx = masw.masw_curve(*args, t(w.lam), c)
    work = np.where(idx.cpu().numpy() >= 0, idx.cpu().numpy() + 1, len(w.c)).astype(np.int64)
    W = len(w.lam)
    res = {}
    t1 = None
    for strat in ("contiguous", "modular"):
        res[strat] = {}
        for G in range(1, 9):
            parts = D.partition_wavelengths(W, G, strat)
            dets = [int(work[p].sum()) for p in parts]
            times = []
            for p in parts:
                lam_p = t(w.lam[p])
                times.append(time_ms(lambda: masw.masw_curve(*args, lam_p, c), reps=reps))
            if G == 1 and t1 is None:
                t1 = times[0]
                d1 = dets[0]
            res[strat][G] = {"worker_dets": dets, "worker_ms": [round(x, 4) for x in times],
                             "det_speedup": d1 / max(dets), "time_speedup": t1 / max(times)}
    return res


def across_workers_ensemble(w, reps):
    """The same partitions at throughput scale: every worker scans ALL models of the C5
    ensemble on its share of the 40 wavelengths (masw_curves_ensemble on device-resident
    inputs), so a worker's device time follows its det count instead of launch latency."""
    m = w.models
    args = [t(x) for x in (m.h, m.alpha, m.beta, m.rho)]
    c = t(w.c)
    st, ct, idx, _ = masw.masw_curves_ensemble(*args, t(w.lam), c)
    ix = idx.cpu().numpy()
    work = np.where(ix >= 0, ix + 1, len(w.c)).astype(np.int64).sum(axis=0)   # per wavelength
    W = len(w.lam)
    res = {}
    t1 = d1 = None
    for strat in ("contiguous", "modular"):
        res[strat] = {}
        for G in range(1, 9):
            parts = D.partition_wavelengths(W, G, strat)
            dets = [int(work[p].sum()) for p in parts]
            times = []
            for p in parts:
                lam_p = t(w.lam[p])
                times.append(time_ms(lambda: masw.masw_curves_ensemble(*args, lam_p, c),
                                     reps=reps))
            if t1 is None:
                t1, d1 = times[0], dets[0]
            res[strat][G] = {"worker_dets": dets, "worker_ms": [round(x, 4) for x in times],
                             "det_speedup": d1 / max(dets), "time_speedup": t1 / max(times)}
    return res


def main():
    out = {"within_gpu": {
        "C4_realistic_team1": within_gpu("realistic", synth.workload("realistic"), 1),
        "C5_ensemble_team1": within_gpu("ensemble", synth.workload("ensemble", M=100_000), 1)},
        "across_workers": {
        "C2_variable40": across_workers("maswaves", synth.workload("maswaves"), 20),
        "C4_realistic": across_workers("realistic", synth.workload("realistic"), 3),
        "C5_ensemble_variable40": across_workers_ensemble(
            synth.workload("ensemble", M=100_000), 3)}}
    path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/load_balance.json"
    json.dump(out, open(path, "w"), indent=1)
    for k, v in out["within_gpu"].items():
        for s, r in v.items():
            print(f"{k:22s} {s:10s} scan {r['scan_ms']:8.3f} ms  teams {r['teams']:5d}  "
                  f"max/mean {r['team_dets_max_over_mean']:.3f}  cv {r['team_dets_cv']:.3f}")
    for k, v in out["across_workers"].items():
        for s, byg in v.items():
            print(k, s, " ".join(f"G{g}:{r['det_speedup']:.2f}/{r['time_speedup']:.2f}"
                                  for g, r in byg.items()))


if __name__ == "__main__":
    main()
