"""Quick device timings of every config (development aid; bench.py is the contract)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_02256_b200 as masw  # noqa: E402
import synth  # noqa: E402


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda")


def time_call(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    print("lib:", masw.masw.LIB_PATH, flush=True)
    if not os.environ.get("NOPROBE"):
        tf, ms = masw.masw_probe_fp64_peak(-1, 300.0)
        print(f"fp64 probe: {tf:.2f} TFLOP/s ({ms:.1f} ms)", flush=True)
    team_env = int(os.environ.get("TEAM", "0"))
    xflags = int(os.environ.get("FLAGS", "0"), 0)   # e.g. FLAGS=0x20 (rows) / 0x40 (models)
    only = os.environ.get("CONFIGS", "tiny,maswaves,uniform,realistic,ensemble").split(",")
    for name, kw in [("tiny", {}), ("maswaves", {}), ("uniform", {"tier": 200.0}),
                     ("realistic", {}), ("ensemble", {"M": 100_000})]:
        if name not in only:
            continue
        w = synth.workload(name, **kw)
        m = w.models
        args = [dev(x) for x in (m.h, m.alpha, m.beta, m.rho)]
        lam, c = dev(w.lam), dev(w.c)
        ce = dev(w.ce) if w.ce is not None else None
        for team in ([team_env] if team_env >= 0 else [0]) if "TEAM" in os.environ else [0, 1, 2, 4, 8]:
            if name == "ensemble":
                fn = lambda: masw.masw_curves_ensemble(*args, lam, c, ce, team_warps=team,
                                                       flags=masw.TIME_SCAN | xflags)
            else:
                fn = lambda: masw.masw_curve(*[a[0] for a in args], lam, c, team_warps=team,
                                             flags=masw.TIME_SCAN | xflags)
            t = time_call(fn)
            alg, ev = masw.masw_last_work()
            kms = masw.masw_last_scan_ms()
            fb = masw.masw_last_fallbacks()
            print(f"{name:10s} team={team:2d} call {t:9.3f} ms  scan {kms:9.3f} ms  "
                  f"alg {alg:12d} eval {ev:12d} gepp-fallback {fb:9d}  "
                  f"{alg / (kms * 1e-3) / 1e9:8.3f} Gdet/s", flush=True)


if __name__ == "__main__":
    main()
