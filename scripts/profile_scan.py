"""Small ensemble run for ncu captures of scan_kernel (development aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_02256_b200 as masw  # noqa: E402
import synth  # noqa: E402

M = int(os.environ.get("M", "5000"))
REPS = int(os.environ.get("REPS", "2"))
w = synth.workload("ensemble", M=M)
m = w.models
d = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda")
args = [d(x) for x in (m.h, m.alpha, m.beta, m.rho)]
for _ in range(REPS):
    r = masw.masw_curves_ensemble(*args, d(w.lam), d(w.c), d(w.ce), flags=masw.TIME_SCAN)
torch.cuda.synchronize()
print("scan ms", masw.masw_last_scan_ms(), "work", masw.masw_last_work())
