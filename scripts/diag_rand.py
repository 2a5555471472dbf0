import os, sys, math
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import synth, oracle
import paper_2003_02256_b200 as masw
oracle.build()
N, seed = int(sys.argv[1]), int(sys.argv[2])
mods = synth.random_models(160, N, seed)
lam = synth.geom(60.0, 0.8, 24)
c = 0.5 * (np.arange(1000, dtype=np.float64) + 1.0)
o = oracle.ensemble(mods, lam, c, None)
for fl, name in ((masw.SCHED_MODELS, "models"), (masw.SCHED_ROWS, "rows"), (masw.SCHED_ROWS | masw.PIVOTED, "rows-pivoted")):
    r = masw.masw_curves_ensemble(mods.h, mods.alpha, mods.beta, mods.rho, lam, c, None, flags=fl)
    mm = np.argwhere(r.idx != o["idx"])
    print(name, "mismatches", len(mm))
    for m, i in mm[:6]:
        a = (mods.h[m], mods.alpha[m], mods.beta[m], mods.rho[m])
        jg, jo = int(r.idx[m, i]), int(o["idx"][m, i])
        vals = []
        for j in sorted(set([max(jg - 1, 0), max(jg, 0), max(jo - 1, 0), max(jo, 0)])):
            mt, e, st = oracle.det(*a, float(lam[i]), float(c[j]))
            vals.append((j, float(c[j]), float(mt.real * 2.0 ** e)))
        print(f"  m={m} i={i} lam={lam[i]:.3f} gpu={jg} oracle={jo} h={a[0]} b={a[2]} al={a[1]} rho={a[3]}")
        print("     ", vals)
