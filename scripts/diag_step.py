"""Fine-grained timing of one bench step (development aid)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_02256_b200 as masw  # noqa: E402
import synth  # noqa: E402

M = 100_000
w = synth.workload("ensemble", M=M)
m = w.models
d = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda")
args = [d(x) for x in (m.h, m.alpha, m.beta, m.rho)]
lam, c, ce = d(w.lam), d(w.c), d(w.ce)
ct = torch.empty((M, 40), dtype=torch.float64, device="cuda")
idx = torch.empty((M, 40), dtype=torch.int32, device="cuda")
mis = torch.empty((M,), dtype=torch.float64, device="cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for _ in range(3):
    masw.masw_curves_ensemble(*args, lam, c, ce, ct_out=ct, idx_out=idx, misfit_out=mis)
torch.cuda.synchronize()
mode = os.environ.get("MODE", "async")
for it in range(12):
    flush.zero_()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    h = [time.perf_counter()]
    ev[0].record()
    h.append(time.perf_counter())
    fl = masw.ASYNC | masw.TIME_SCAN if mode == "async" else masw.TIME_SCAN
    masw.masw_curves_ensemble(*args, lam, c, ce, ct_out=ct, idx_out=idx, misfit_out=mis, flags=fl)
    h.append(time.perf_counter())
    ev[1].record()
    b, v = masw.masw_argmin(mis, flags=fl & masw.ASYNC)
    h.append(time.perf_counter())
    ev[2].record()
    ev[2].synchronize()
    h.append(time.perf_counter())
    scan = masw.masw_last_scan_ms()
    print(f"step {it:2d} ev: call {ev[0].elapsed_time(ev[1]):8.3f} argmin {ev[1].elapsed_time(ev[2]):7.3f} "
          f"total {ev[0].elapsed_time(ev[2]):8.3f} scan {scan:8.3f} | host: rec {1e3*(h[1]-h[0]):6.3f} "
          f"call {1e3*(h[2]-h[1]):7.3f} argmin {1e3*(h[3]-h[2]):6.3f} wait {1e3*(h[4]-h[3]):8.3f}", flush=True)
