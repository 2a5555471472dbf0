"""Same-box A/B of scan time between flag sets, interleaved (development aid).

    FLAGSETS="0,0x400" CONFIGS=ensemble,realistic,uniform python scripts/ab_time.py

Prints, per config and flag set, the median of MASW_TIME_SCAN scan times (the library's own
CUDA events on the launching stream) over REPS interleaved repetitions, and the idx agreement
with the first flag set."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_02256_b200 as masw  # noqa: E402
import synth  # noqa: E402


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda")


def main():
    flagsets = [int(f, 0) for f in os.environ.get("FLAGSETS", "0,0x400").split(",")]
    only = os.environ.get("CONFIGS", "ensemble,realistic,uniform").split(",")
    reps = int(os.environ.get("REPS", "7"))
    M = int(os.environ.get("M", "100000"))
    for name, kw in [("tiny", {}), ("maswaves", {}), ("uniform", {"tier": 200.0}),
                     ("realistic", {}), ("ensemble", {"M": M})]:
        if name not in only:
            continue
        w = synth.workload(name, **kw)
        m = w.models
        args = [dev(x) for x in (m.h, m.alpha, m.beta, m.rho)]
        lam, c = dev(w.lam), dev(w.c)
        ce = dev(w.ce) if w.ce is not None else None

        def run(fl):
            if name == "ensemble":
                r = masw.masw_curves_ensemble(*args, lam, c, ce, flags=masw.TIME_SCAN | fl)
                return r.idx
            st, ct, idx = masw.masw_curve(*[a[0] for a in args], lam, c,
                                          flags=masw.TIME_SCAN | fl)
            return idx

        ref = None
        times = {f: [] for f in flagsets}
        same = {}
        pref = {}
        for f in flagsets:
            run(f)
        for _ in range(reps):
            for f in flagsets:
                idx = run(f)
                torch.cuda.synchronize()
                times[f].append(masw.masw_last_scan_ms())
                if ref is None:
                    ref = idx.clone()
                same[f] = int((idx == ref).sum().item()), int(idx.numel())
                pref[f] = masw.masw_last_prefix()
        for f in flagsets:
            t = statistics.median(times[f])
            print(f"{name:10s} flags={f:#06x} scan {t:9.3f} ms (min {min(times[f]):.3f})  "
                  f"idx equal to first {same[f][0]}/{same[f][1]}"
                  f"  prefix rows/dets {pref[f]}", flush=True)


if __name__ == "__main__":
    main()
