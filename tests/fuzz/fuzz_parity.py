"""Randomised parity sweep (evidence run, not a unit test): many seeded calls with random
shapes -- N = 1..12 layers, random layered models (synth.random_models: reversals, stiff lids,
soft channels), random wavelength ranges on both sides of the fine/coarse cosh/sinh table
boundary (k h_max <= 50.5 or above), grids from 0.5 m/s or from near the slowest layer, every
scan (model-major, pair, row) -- each compared with the CPU oracle row by row under the S16
near-root rule (tests/masw_parity.py::ct_acceptable).  Writes one JSON summary.

    python tests/fuzz/fuzz_parity.py [seconds] [out.json]
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
import torch  # noqa: E402

import masw_parity as parity  # noqa: E402
import oracle  # noqa: E402
import paper_2003_02256_b200 as masw  # noqa: E402
import synth  # noqa: E402


KH_LO = float(os.environ.get("FUZZ_KH_LO", "50.6"))   # coarse calls: k h_max range
KH_HI = float(os.environ.get("FUZZ_KH_HI", "300"))
SEED = int(os.environ.get("FUZZ_SEED", "2003"))
# FUZZ_MODE: "default" as above; "stable" -- every call with MASW_STABLE (k h_max up to 340);
# "wide" -- N up to 24 and grids reaching 2.5 x the fastest P wave (both waves trigonometric,
# complex half-space node); "misc" -- N up to 40, host or device buffers, a random C_e
# (misfit against the oracle's misfit of the GPU's C_t), random MASW_PIVOTED (MASW_DIRECT, an
# A/B switch that drops the small-c pre-pass, is excluded: its small-c signs are noise,
# reading S15'')
# "big" -- 3000-8000 models per call, N = 3..8, the automatic kernel choice (model-major scan
# with its tail pieces, or the pair scan), no forced schedule
# "curve" -- one model, 3000-12000 wavelengths in random order (single long curves: whole
# pairs plus tail segments of the pair scan), the automatic kernel choice
# "s4" -- grids containing the models' own layer velocities and points within 1e-4 of them
# (the perturbation rule, reading S4), 1-5 models per call
MODE = os.environ.get("FUZZ_MODE", "default")
EXTRA_FLAGS = int(os.environ.get("FUZZ_FLAGS", "0"), 0)   # OR-ed into every call's flags


def make_call(rng, call):
    """One call of the sweep (the seeded draws in their fixed order): the models, wavelengths,
    grid, kernel label, flags, C_e (or None) and whether host buffers are used."""
    N = int(rng.integers(1, {"wide": 25, "misc": 41}.get(MODE, 13)))
    M = int(rng.integers(1, 12 if N > 12 else 60))
    if MODE == "s4":
        M = int(rng.integers(1, 6))
    if MODE == "big":
        N = int(rng.integers(3, 9))
        M = int(rng.integers(3000, 8001))
    if MODE == "curve":
        M = 1
    mods = synth.random_models(M, N, 10_000 + call)
    hmax = float(mods.h.max())
    fine = bool(rng.integers(0, 2))
    khmax = float(rng.uniform(5.0, 50.4)) if fine else float(rng.uniform(KH_LO, KH_HI))
    if MODE == "stable" and not fine:
        khmax = float(rng.uniform(50.6, 340.0))   # (the oracle validates k h <= 350)
    lam_min = 2 * math.pi * hmax / khmax
    L = int(rng.integers(1, 48))
    if MODE == "curve":
        L = int(rng.integers(3000, 12001))
    lam = synth.geom(float(rng.uniform(max(lam_min * 1.5, 2.0), 120.0)), lam_min, L) if L > 1 \
        else np.array([lam_min])
    if MODE == "curve":
        lam = rng.permutation(lam)
    V = int(rng.integers(64, 1500))
    if MODE == "wide" and rng.integers(0, 2):
        c_hi = 2.5 * float(mods.alpha.max())
        c0 = float(rng.uniform(0.3, 1.0)) * float(mods.beta.min())
        c = c0 + (c_hi - c0) / V * np.arange(V, dtype=np.float64)
    elif rng.integers(0, 2):
        c = 0.5 * (np.arange(V, dtype=np.float64) + 1.0)           # from 0.5 m/s
    else:
        c0 = float(mods.beta.min()) * float(rng.uniform(0.5, 0.95))
        c = c0 + float(rng.uniform(0.05, 1.0)) * np.arange(V, dtype=np.float64)
    if MODE == "s4":   # the models' velocities, and points just inside / outside 1e-4 of them
        vel = np.concatenate([mods.alpha.ravel(), mods.beta.ravel()])
        off = rng.choice(np.array([0.0, 0.0, 5e-5, -5e-5, 9.9e-5, -1.5e-4, 2e-4]), vel.size)
        c = np.unique(np.concatenate([c, vel + off]))
        c = c[c > 0]
    kern = ["models", "pairs", "rows"][int(rng.integers(0, 3))]
    flag = {"models": masw.SCHED_MODELS, "pairs": masw.SCHED_PAIRS, "rows": masw.SCHED_ROWS}[kern]
    if MODE == "stable":
        flag |= masw.STABLE
    if MODE in ("big", "curve"):
        flag = 0
        kern = "auto"
    flag |= EXTRA_FLAGS
    ce = None
    host = False
    if MODE == "misc":
        flag |= [0, masw.PIVOTED][int(rng.integers(0, 2))]
        host = bool(rng.integers(0, 2))
        ce = float(mods.beta.min()) * rng.uniform(0.6, 1.1, len(lam))
    return N, M, mods, fine, khmax, lam, c, kern, flag, ce, host


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
    out = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "fuzz_parity.json")
    stats = run(budget)
    json.dump(stats, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in stats.items() if k != "bad_cases"}), flush=True)


def run(budget: float, max_calls: int = 1 << 62) -> dict:
    """The sweep for `budget` seconds or `max_calls` calls (whichever ends first)."""
    oracle.build()
    dev = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda")
    rng = np.random.Generator(np.random.PCG64(SEED))
    t_end = time.time() + budget
    stats = {"mode": MODE, "seed": SEED, "extra_flags": EXTRA_FLAGS, "calls": 0, "rows": 0, "rows_equal": 0, "rows_one_step_S16": 0, "rows_bad": 0,
             "fine_calls": 0, "coarse_calls": 0, "by_kernel": {}, "bad_cases": []}
    call = 0
    while time.time() < t_end and call < max_calls:
        call += 1
        N, M, mods, fine, khmax, lam, c, kern, flag, ce, host = make_call(rng, call)
        conv = (lambda a: np.ascontiguousarray(a)) if host else dev
        try:
            r = masw.masw_curves_ensemble(*[conv(x) for x in (mods.h, mods.alpha, mods.beta,
                                                                 mods.rho)], conv(lam), conv(c),
                                          conv(ce) if ce is not None else None, flags=flag)
        except masw.MaswError as e:   # (e.g. k h > 350 cannot occur here; report anyway)
            stats["bad_cases"].append({"call": call, "error": e.code})
            continue
        gidx = r.idx if host else r.idx.cpu().numpy()
        o = oracle.ensemble(mods, lam, c, None)
        if ce is not None:   # misfit of the GPU's own C_t (reading S13), 1e-9 relative
            gct = r.ct if host else r.ct.cpu().numpy()
            gmis = r.misfit if host else r.misfit.cpu().numpy()
            for m in range(M):
                if not parity.misfit_ok(oracle, gct[m], ce, float(gmis[m])):
                    stats["misfit_bad"] = stats.get("misfit_bad", 0) + 1
        stats["calls"] += 1
        stats["fine_calls" if fine else "coarse_calls"] += 1
        k = stats["by_kernel"].setdefault(kern, {"calls": 0, "rows": 0, "bad": 0})
        k["calls"] += 1
        k["rows"] += gidx.size
        stats["rows"] += gidx.size
        eq = gidx == o["idx"]
        stats["rows_equal"] += int(eq.sum())
        for m in range(M):
            if eq[m].all():
                continue
            a = (mods.h[m], mods.alpha[m], mods.beta[m], mods.rho[m])
            ok, exact, one = parity.ct_acceptable(oracle, a, lam, c, gidx[m], o["idx"][m])
            nb = int((~ok).sum())
            stats["rows_one_step_S16"] += int(one)
            stats["rows_bad"] += nb
            k["bad"] += nb
            if nb:
                bad_i = np.nonzero(~ok)[0]
                stats["bad_cases"].append({"call": call, "model": m, "N": N, "kernel": kern,
                                           "fine": fine, "rows_bad": nb, "flags": int(flag),
                                           "host": host,
                                           "kh_model": [float(2 * math.pi / lam[i] * mods.h[m].max())
                                                        for i in bad_i]})
        kh_rows = 2 * math.pi / lam[None, :] * mods.h.max(axis=1)[:, None]
        for lo in (50, 80, 100, 120, 140, 160):
            key = f"rows_kh_ge_{lo}"
            stats[key] = stats.get(key, 0) + int((kh_rows >= lo).sum())
    return stats


if __name__ == "__main__":
    main()
