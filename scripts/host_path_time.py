"""Host-buffer path timing (development aid): one C5-size masw_curves_ensemble call with
pinned host buffers, CUDA-event timed, once per command-line argument, each in its own process
with MASW_HOST_CHUNKS set to it (a knob of the measured, rejected pipelined-path build --
DESIGN.md §10b; the current library ignores it, so every argument times the one-launch path).

    python scripts/host_path_time.py 1 2 4 8
"""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child():
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import paper_2003_02256_b200 as masw
    import synth

    w = synth.workload("ensemble", M=100_000)
    m = w.models
    pin = lambda a: torch.as_tensor(np.ascontiguousarray(a)).pin_memory()
    hp = [pin(x) for x in (m.h, m.alpha, m.beta, m.rho)]
    lam, c, ce = pin(w.lam), pin(w.c), pin(w.ce)
    M, L = m.h.shape[0], len(w.lam)
    hct = torch.empty((M, L), dtype=torch.float64).pin_memory()
    hidx = torch.empty((M, L), dtype=torch.int32).pin_memory()
    hmis = torch.empty((M,), dtype=torch.float64).pin_memory()
    ts = []
    for k in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        masw.masw_curves_ensemble(*hp, lam, c, ce, ct_out=hct, idx_out=hidx, misfit_out=hmis)
        e1.record()
        e1.synchronize()
        if k >= 2:
            ts.append(e0.elapsed_time(e1))
    print("RESULT " + json.dumps({"ms": ts, "median": statistics.median(ts)}), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child()
    else:
        for k in sys.argv[1:]:
            env = dict(os.environ, MASW_HOST_CHUNKS=k)
            p = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True,
                               text=True)
            line = [x for x in p.stdout.splitlines() if x.startswith("RESULT ")]
            print(k, json.loads(line[0][7:])["median"] if line else p.stderr[-500:], flush=True)
