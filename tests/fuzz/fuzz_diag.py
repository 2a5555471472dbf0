"""Re-runs one call of the randomised sweep (FUZZ_MODE / FUZZ_SEED as for fuzz_parity.py)
through every scan and sign method and counts the rows whose index differs from the oracle's
(development aid).

    FUZZ_MODE=big FUZZ_SEED=21 python tests/fuzz/fuzz_diag.py <call> [<call> ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import fuzz_parity as F  # noqa: E402
import oracle  # noqa: E402
import paper_2003_02256_b200 as masw  # noqa: E402


def main():
    want = sorted(int(x) for x in sys.argv[1:])
    oracle.build()
    dev = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda")
    rng = np.random.Generator(np.random.PCG64(F.SEED))
    for call in range(1, max(want) + 1):
        N, M, mods, fine, khmax, lam, c, kern, flag, ce, host = F.make_call(rng, call)
        if call not in want:
            continue
        o = oracle.ensemble(mods, lam, c, None)
        print(f"call {call}: N={N} M={M} L={len(lam)} V={len(c)} fine={fine} c0={c[0]:.4g} "
              f"dc={c[1] - c[0]:.4g} lam=[{lam.min():.4g}, {lam.max():.4g}]", flush=True)
        args = [dev(x) for x in (mods.h, mods.alpha, mods.beta, mods.rho)]
        for lab, fl in (("auto", 0), ("models", masw.SCHED_MODELS), ("pairs", masw.SCHED_PAIRS),
                        ("rows", masw.SCHED_ROWS), ("auto+pivoted", masw.PIVOTED),
                        ("auto+direct", masw.DIRECT)):
            r = masw.masw_curves_ensemble(*args, dev(lam), dev(c), flags=fl)
            g = r.idx.cpu().numpy()
            bad = np.argwhere(g != o["idx"])
            ex = [(int(m), int(i), int(g[m, i]), int(o["idx"][m, i])) for m, i in bad[:4]]
            print(f"   {lab:13s} rows differing {len(bad):6d}  e.g. (model, row, gpu, oracle) {ex}",
                  flush=True)


if __name__ == "__main__":
    main()
