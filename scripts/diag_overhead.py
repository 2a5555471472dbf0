"""Where does per-call time go?  (development aid)"""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_02256_b200 as masw  # noqa: E402
import synth  # noqa: E402

M = int(os.environ.get("M", "100000"))
w = synth.workload("ensemble", M=M)
m = w.models
d = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda")
args = [d(x) for x in (m.h, m.alpha, m.beta, m.rho)]
lam, c, ce = d(w.lam), d(w.c), d(w.ce)
ct = torch.empty((M, 40), dtype=torch.float64, device="cuda")
idx = torch.empty((M, 40), dtype=torch.int32, device="cuda")
mis = torch.empty((M,), dtype=torch.float64, device="cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")


def one(label, fn, reps=5, do_flush=True):
    fn()
    torch.cuda.synchronize()
    for _ in range(reps):
        if do_flush:
            flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        fn()
        e1.record()
        t1 = time.perf_counter()
        e1.synchronize()
        t2 = time.perf_counter()
        print(f"{label:40s} event {e0.elapsed_time(e1):8.3f} ms  host-call {1e3*(t1-t0):8.3f} ms  "
              f"wall {1e3*(t2-t0):8.3f} ms  scan {masw.masw_last_scan_ms():8.3f}", flush=True)


ens = lambda: masw.masw_curves_ensemble(*args, lam, c, ce, ct_out=ct, idx_out=idx, misfit_out=mis,
                                        flags=masw.TIME_SCAN)
one("ensemble (flush)", ens)
one("ensemble (no flush)", ens, do_flush=False)
one("ensemble ASYNC", lambda: masw.masw_curves_ensemble(*args, lam, c, ce, ct_out=ct, idx_out=idx,
                                                        misfit_out=mis, flags=masw.TIME_SCAN | masw.ASYNC))
one("argmin", lambda: masw.masw_argmin(mis))
p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv", "-lms", "200"],
                     stdout=subprocess.DEVNULL)
time.sleep(0.5)
one("ensemble with nvidia-smi polling", ens)
p.terminate()
one("ensemble after polling", ens)
