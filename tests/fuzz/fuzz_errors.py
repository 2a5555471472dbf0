"""Randomised validation sweep (evidence run): valid random ensembles with one to three
random corruptions -- NaN / Inf / zero / negative entries in h, alpha, beta, rho, lambda, c or
C_e, alpha <= beta, a non-increasing grid, c_0 <= 0, k h beyond the 350 guard -- through
masw_curves_ensemble (device or host buffers, with or without C_e), the returned status
against the oracle's (the precedence of include/masw.h), and on an error the caller's output
buffers untouched.  Writes one JSON summary.

    python tests/fuzz/fuzz_errors.py [seconds] [out.json]
"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2003_02256_b200 as masw  # noqa: E402
import synth  # noqa: E402


def corrupt(rng, arrs):
    """One corruption of the dict of arrays (in place); returns its label."""
    kind = int(rng.integers(0, 9))
    if kind == 0:                                          # a non-finite entry somewhere
        name = ["h", "alpha", "beta", "rho", "lam", "c", "ce"][int(rng.integers(0, 7))]
        a = arrs[name]
        a.flat[int(rng.integers(0, a.size))] = [np.nan, np.inf, -np.inf][int(rng.integers(0, 3))]
        return f"nonfinite:{name}"
    if kind == 1:                                          # zero / negative model parameter
        name = ["h", "alpha", "beta", "rho"][int(rng.integers(0, 4))]
        a = arrs[name]
        a.flat[int(rng.integers(0, a.size))] = [0.0, -1.0][int(rng.integers(0, 2))]
        return f"nonpositive:{name}"
    if kind == 2:                                          # alpha <= beta in one layer
        i = int(rng.integers(0, arrs["alpha"].size))
        arrs["alpha"].flat[i] = arrs["beta"].flat[i] * float(rng.uniform(0.5, 1.0))
        return "alpha<=beta"
    if kind == 3:                                          # wavelength <= 0
        arrs["lam"][int(rng.integers(0, arrs["lam"].size))] = [0.0, -2.0][int(rng.integers(0, 2))]
        return "lambda<=0"
    if kind == 4:                                          # c_0 <= 0
        arrs["c"][0] = [0.0, -1.0][int(rng.integers(0, 2))]
        return "c0<=0"
    if kind == 5:                                          # grid not strictly increasing
        c = arrs["c"]
        j = int(rng.integers(1, c.size))
        c[j] = c[j - 1] - float(rng.uniform(0.0, 1.0))
        return "c not increasing"
    if kind == 6:                                          # k h beyond the guard
        arrs["lam"][int(rng.integers(0, arrs["lam"].size))] = 2 * math.pi * float(arrs["h"].max()) / 360.0
        return "kh>350"
    if kind == 7:                                          # C_e <= 0
        arrs["ce"][int(rng.integers(0, arrs["ce"].size))] = [0.0, -3.0][int(rng.integers(0, 2))]
        return "ce<=0"
    return "none"


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
    out = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "fuzz_errors.json")
    oracle.build()
    rng = np.random.Generator(np.random.PCG64(int(os.environ.get("FUZZ_SEED", "41"))))
    dev = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda")
    st = {"calls": 0, "mismatch": 0, "touched": 0, "by_code": {}, "bad_cases": []}
    t_end = time.time() + budget
    call = 0
    while time.time() < t_end:
        call += 1
        N = int(rng.integers(1, 9))
        M = int(rng.integers(1, 40))
        mods = synth.random_models(M, N, 70_000 + call)
        L = int(rng.integers(1, 20))
        lam = synth.geom(80.0, 2.0, L) if L > 1 else np.array([10.0])
        c = 20.0 + 1.0 * np.arange(int(rng.integers(2, 300)), dtype=np.float64)
        arrs = {"h": mods.h.copy(), "alpha": mods.alpha.copy(), "beta": mods.beta.copy(),
                "rho": mods.rho.copy(), "lam": lam.copy(), "c": c.copy(),
                "ce": np.full(L, 150.0)}
        labels = [corrupt(rng, arrs) for _ in range(int(rng.integers(1, 4)))]
        with_ce = bool(rng.integers(0, 2))
        host = bool(rng.integers(0, 2))
        ce = arrs["ce"] if with_ce else None
        om = synth.Models(arrs["h"], arrs["alpha"], arrs["beta"], arrs["rho"])
        o = oracle.ensemble(om, arrs["lam"], arrs["c"], ce)
        ost = int(o["status"])
        ct = np.full((M, L), 7.0) if host else torch.full((M, L), 7.0, dtype=torch.float64,
                                                               device="cuda")
        conv = (lambda a: np.ascontiguousarray(a)) if host else dev
        try:
            r = masw.masw_curves_ensemble(*[conv(arrs[k]) for k in ("h", "alpha", "beta", "rho")],
                                          conv(arrs["lam"]), conv(arrs["c"]),
                                          conv(ce) if ce is not None else None, ct_out=ct)
            gst = int(r.status)
        except masw.MaswError as e:
            gst = int(e.code)
            still = bool((ct == 7.0).all()) if host else bool((ct == 7.0).all().item())
            if not still:
                st["touched"] += 1
        st["calls"] += 1
        st["by_code"][str(gst)] = st["by_code"].get(str(gst), 0) + 1
        if gst != ost:
            st["mismatch"] += 1
            st["bad_cases"].append({"call": call, "labels": labels, "gpu": gst, "oracle": ost,
                                    "with_ce": with_ce, "host": host})
    json.dump(st, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in st.items() if k != "bad_cases"}), flush=True)


if __name__ == "__main__":
    main()
