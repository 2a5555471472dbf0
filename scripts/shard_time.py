"""Scan time of the C5 ensemble shard one rank gets at G = 1, 2, 4, 8 (100k / G models) --
the per-rank compute of bench.py's strong-scaling run, measured on one GPU (development aid)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_02256_b200 as masw  # noqa: E402
import synth  # noqa: E402


def main():
    w = synth.workload("ensemble", M=100_000)
    m = w.models
    d = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda")
    lam, c, ce = d(w.lam), d(w.c), d(w.ce)
    base = None
    for G in (1, 2, 4, 8):
        Mr = 100_000 // G
        args = [d(x[:Mr]) for x in (m.h, m.alpha, m.beta, m.rho)]
        for _ in range(2):
            masw.masw_curves_ensemble(*args, lam, c, ce, flags=masw.TIME_SCAN)
        ts = []
        for _ in range(5):
            masw.masw_curves_ensemble(*args, lam, c, ce, flags=masw.TIME_SCAN)
            ts.append(masw.masw_last_scan_ms())
        alg, ev = masw.masw_last_work()
        t = statistics.median(ts)
        rate = alg / (t * 1e-3)
        base = base or rate
        print(f"G={G} models/rank={Mr:6d} scan {t:8.3f} ms  {rate / 1e9:7.3f} Gdet/s/GPU  "
              f"per-GPU efficiency vs G=1 {rate / base:6.3f}", flush=True)


if __name__ == "__main__":
    main()
