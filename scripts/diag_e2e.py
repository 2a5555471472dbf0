"""e2e (host-buffer) call breakdown, development aid."""
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
pin = lambda a: torch.as_tensor(np.ascontiguousarray(a)).pin_memory()
hh, ha, hb, hr = (pin(x) for x in (m.h, m.alpha, m.beta, m.rho))
hlam, hc, hce = pin(w.lam), pin(w.c), pin(w.ce)
hct = torch.empty((M, 40), dtype=torch.float64).pin_memory()
hidx = torch.empty((M, 40), dtype=torch.int32).pin_memory()
hmis = torch.empty((M,), dtype=torch.float64).pin_memory()
for _ in range(3):
    masw.masw_curves_ensemble(hh, ha, hb, hr, hlam, hc, hce, ct_out=hct, idx_out=hidx, misfit_out=hmis)
for it in range(8):
    t0 = time.perf_counter()
    masw.masw_curves_ensemble(hh, ha, hb, hr, hlam, hc, hce, ct_out=hct, idx_out=hidx,
                              misfit_out=hmis, flags=masw.TIME_SCAN)
    t1 = time.perf_counter()
    scan = masw.masw_last_scan_ms()
    b, v = masw.masw_argmin(hmis)
    t2 = time.perf_counter()
    print(f"host call {1e3*(t1-t0):8.3f} ms (scan {scan:7.3f})  argmin {1e3*(t2-t1):6.3f} ms", flush=True)
