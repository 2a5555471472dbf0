"""Warp finish-time tail of the C5 model-major scan (development aid).

Needs a library built with -DMASW_TAIL_PROBE (each warp writes its %globaltimer finish time
into the MASW_TEAM_STATS slots):  python -m paper_2003_02256_b200.build -DMASW_TAIL_PROBE=1
--out=build/var/libmasw_tail.so;  MASW_LIB=build/var/libmasw_tail.so python scripts/tail_probe.py
"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2003_02256_b200 as masw, synth
w = synth.workload("ensemble", M=100000)
m = w.models
d = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda")
args = [d(x) for x in (m.h, m.alpha, m.beta, m.rho)]
for _ in range(2):
    masw.masw_curves_ensemble(*args, d(w.lam), d(w.c), d(w.ce), flags=masw.TEAM_STATS | masw.TIME_SCAN)
t = masw.masw_last_team_dets().astype(np.float64)
kms = masw.masw_last_scan_ms()
t = (t - t.max()) / 1e6   # ms before the last warp finished
print("kernel ms", kms, "warps", len(t))
print("finish before end (ms): mean %.3f median %.3f p10 %.3f max %.3f" % (-t.mean(), -np.median(t), -np.percentile(t, 10), -t.min()))
print("idle fraction of kernel: %.4f" % ((-t).mean() / kms))
