"""Randomised det-value sweep (evidence run): masw_det_grid (banded GEPP values, direct or
stable element) against the oracle's dense complex LU on random layered models and grids,
1e-9 relative inside the det-parity domain (readings S15, S15': c >= 0.5 beta_min,
|det| >= 1e-12 of the row maximum, kappa <= 1e-10), and the sign of Re det wherever the det
is in that domain.  Writes one JSON summary.

    python tests/fuzz/fuzz_detgrid.py [seconds] [out.json]
"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import masw_parity as parity  # noqa: E402
import oracle  # noqa: E402
import paper_2003_02256_b200 as masw  # noqa: E402
import synth  # noqa: E402


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
    out = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "fuzz_detgrid.json")
    oracle.build()
    rng = np.random.Generator(np.random.PCG64(int(os.environ.get("FUZZ_SEED", "31"))))
    t_end = time.time() + budget
    st = {"calls": 0, "points": 0, "in_domain": 0, "worst_rel_in_domain": 0.0, "bad_points": 0,
          "sign_bad": 0, "stable_calls": 0, "bad_cases": []}
    call = 0
    while time.time() < t_end:
        call += 1
        N = int(rng.integers(1, 11))
        mods = synth.random_models(1, N, 50_000 + call)
        a = (mods.h[0], mods.alpha[0], mods.beta[0], mods.rho[0])
        stable = bool(rng.integers(0, 4) == 0)
        khmax = float(rng.uniform(1.0, 340.0))
        lam_min = 2 * math.pi * float(a[0].max()) / khmax
        L = int(rng.integers(1, 9))
        lam = synth.geom(float(rng.uniform(lam_min * 1.2, lam_min * 200.0)), lam_min, L) if L > 1 \
            else np.array([lam_min])
        V = int(rng.integers(16, 160))
        c_hi = float(rng.uniform(0.8, 2.5)) * float(a[1].max())
        c_lo = float(rng.uniform(0.3, 1.0)) * float(a[2].min())
        c = np.linspace(c_lo, c_hi, V)
        gre, gim, gex = masw.masw_det_grid(*a, lam, c, flags=masw.STABLE if stable else 0)
        ost, omant, oex, _ = oracle.det_grid(*a, lam, c)
        kap = oracle.det_grid_kappa(*a, lam, c)
        rel = parity.det_grid_rel_err(gre + 1j * gim, gex, omant, oex)
        dom = parity.det_domain(omant, oex, c, float(a[2].min()), kap)
        st["calls"] += 1
        st["stable_calls"] += int(stable)
        st["points"] += int(dom.size)
        st["in_domain"] += int(dom.sum())
        if dom.any():
            w = float(np.nanmax(rel[dom]))
            st["worst_rel_in_domain"] = max(st["worst_rel_in_domain"], w)
            nb = int((rel[dom] > parity.DET_RTOL).sum())
            sb = int((np.sign(gre)[dom] != np.sign(omant.real)[dom]).sum())
            st["bad_points"] += nb
            st["sign_bad"] += sb
            if nb or sb:
                st["bad_cases"].append({"call": call, "N": N, "stable": stable, "khmax": khmax,
                                        "bad": nb, "sign_bad": sb, "worst": w})
    json.dump(st, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in st.items() if k != "bad_cases"}), flush=True)


if __name__ == "__main__":
    main()
