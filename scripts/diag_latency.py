"""Host overhead of a small single-curve call (C2), development aid."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_02256_b200 as masw  # noqa: E402
from paper_2003_02256_b200 import masw as mb  # noqa: E402
import synth  # noqa: E402

w = synth.workload("maswaves")
m = w.models
d = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda")
args = [d(x[0]) for x in (m.h, m.alpha, m.beta, m.rho)]
lam, c = d(w.lam), d(w.c)
ct = torch.empty(40, dtype=torch.float64, device="cuda")
idx = torch.empty(40, dtype=torch.int32, device="cuda")
L = mb.lib()
mod = mb._Model(5, *[a.data_ptr() for a in args])
ex = mb._Exec(0, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream), 0, 0)
exa = mb._Exec(0, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream), 0, masw.ASYNC)


def bench(label, fn, n=200):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"{label:50s} {1e6 * (t1 - t0) / n:9.1f} us/call", flush=True)


bench("binding masw_curve (device ptrs)", lambda: masw.masw_curve(*args, lam, c))
bench("binding masw_curve, outputs given", lambda: masw.masw_curve(*args, lam, c, ct_out=ct, idx_out=idx))
bench("raw ctypes masw_curve", lambda: L.masw_curve(ctypes.byref(mod), lam.data_ptr(), 40, c.data_ptr(), 1000,
                                                 ct.data_ptr(), idx.data_ptr(), ctypes.byref(ex)))
bench("raw ctypes masw_curve ASYNC", lambda: L.masw_curve(ctypes.byref(mod), lam.data_ptr(), 40, c.data_ptr(),
                                                       1000, ct.data_ptr(), idx.data_ptr(), ctypes.byref(exa)))
hm = [np.ascontiguousarray(x[0]) for x in (m.h, m.alpha, m.beta, m.rho)]
bench("binding masw_curve (host numpy)", lambda: masw.masw_curve(*hm, w.lam, w.c))
