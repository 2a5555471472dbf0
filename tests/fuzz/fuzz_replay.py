"""Replays tests/fuzz/fuzz_parity.py's seeded call sequence and, for the calls listed in its
JSON summary's bad_cases, prints per disagreeing row: the GPU and oracle indices, and around
both the sign of Re det K from the oracle in fp64 and in binary128 (det_quad) -- which side
is right (development aid).

    python tests/fuzz/fuzz_replay.py gpurun_out/fuzz_parity.json [max_cases]
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2003_02256_b200 as masw  # noqa: E402
import synth  # noqa: E402


def gen(rng, call):
    N = int(rng.integers(1, 13))
    M = int(rng.integers(1, 60))
    mods = synth.random_models(M, N, 10_000 + call)
    hmax = float(mods.h.max())
    fine = bool(rng.integers(0, 2))
    khmax = float(rng.uniform(5.0, 50.4)) if fine else float(rng.uniform(50.6, 300.0))
    lam_min = 2 * math.pi * hmax / khmax
    L = int(rng.integers(1, 48))
    lam = synth.geom(float(rng.uniform(max(lam_min * 1.5, 2.0), 120.0)), lam_min, L) if L > 1 \
        else np.array([lam_min])
    V = int(rng.integers(64, 1500))
    if rng.integers(0, 2):
        c = 0.5 * (np.arange(V, dtype=np.float64) + 1.0)
    else:
        c0 = float(mods.beta.min()) * float(rng.uniform(0.5, 0.95))
        c = c0 + float(rng.uniform(0.05, 1.0)) * np.arange(V, dtype=np.float64)
    kern = ["models", "pairs", "rows"][int(rng.integers(0, 3))]
    return N, M, mods, fine, khmax, lam, c, kern


def sgn_quad(a, l, cj):
    mq, e, st = oracle.det_quad(*a, l, cj)
    if st != 0:
        return None
    v = mq[0] + mq[1]
    return 0 if v == 0 else (1 if v > 0 else -1)


def main():
    summ = json.load(open(sys.argv[1]))
    maxc = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    brief = len(sys.argv) > 3 and sys.argv[3] == "brief"   # headers only
    want = {}
    for b in summ["bad_cases"]:
        if "model" in b:
            want.setdefault(b["call"], []).append(b["model"])
    oracle.build()
    dev = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda")
    rng = np.random.Generator(np.random.PCG64(2003))
    shown = 0
    call = 0
    last = max(want) if want else 0
    while call < last and shown < maxc:
        call += 1
        N, M, mods, fine, khmax, lam, c, kern = gen(rng, call)
        if call not in want:
            continue
        flag = {"models": masw.SCHED_MODELS, "pairs": masw.SCHED_PAIRS, "rows": masw.SCHED_ROWS}[kern]
        r = masw.masw_curves_ensemble(*[dev(x) for x in (mods.h, mods.alpha, mods.beta, mods.rho)],
                                      dev(lam), dev(c), flags=flag)
        gidx = r.idx.cpu().numpy()
        o = oracle.ensemble(mods, lam, c, None)
        for m in want[call]:
            a = (mods.h[m], mods.alpha[m], mods.beta[m], mods.rho[m])
            for i in np.nonzero(gidx[m] != o["idx"][m])[0]:
                g, oi = int(gidx[m, i]), int(o["idx"][m, i])
                k = 2 * math.pi / lam[i]
                print(f"call {call} model {m} N={N} kern={kern} kh_max(call)={khmax:.1f} "
                      f"lam={lam[i]:.4g} k*h_max(model)={k * a[0].max():.1f} gpu idx {g} "
                      f"oracle idx {oi} c_g={c[g] if g >= 0 else None} c_o={c[oi] if oi >= 0 else None}")
                shown += 1
                if brief:
                    continue
                shown -= 1
                for lab, fl in (("pivoted", masw.PIVOTED), ("stable", masw.STABLE),
                                ("direct", masw.DIRECT)):
                    st2, ct2, i2 = masw.masw_curve(*[dev(x) for x in a], dev(lam[i:i + 1]),
                                                    dev(c), flags=fl)
                    print(f"    gpu {lab:8s} idx {int(i2.cpu()[0])}")
                gre, gim, gex = masw.masw_det_grid(*a, lam[i:i + 1], c)
                lo = max(0, min(x for x in (g, oi) if x >= 0) - 2)
                hi = max(g, oi) + 1
                for j in range(lo, min(hi + 1, len(c))):
                    mnt, e, st = oracle.det(*a, float(lam[i]), float(c[j]))
                    s64 = 0 if mnt.real == 0 else (1 if mnt.real > 0 else -1)
                    print(f"    j={j} c={c[j]:.4f} oracle64 sgn {s64:+d} |Re|=2^{e}*{abs(mnt.real):.3g}"
                          f"  quad sgn {sgn_quad(a, float(lam[i]), float(c[j]))}"
                          f"  gpu det_grid {gre[0, j]:+.3g}*2^{int(gex[0, j])}")
                print("   beta", np.round(a[2], 1), "h", np.round(a[0], 2), "alpha/beta",
                      np.round(a[1] / a[2], 2))
                shown += 1
                if shown >= maxc:
                    break


if __name__ == "__main__":
    main()
