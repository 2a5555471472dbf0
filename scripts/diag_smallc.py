"""Small-c sign check of the direct element (reading S15): oracle fp64 vs long double vs
mpmath (50 digits) vs the GPU direct and stable (MASW_STABLE) scans (development aid)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import synth, oracle
import paper_2003_02256_b200 as masw
oracle.build()
mods = synth.random_models(160, 1, 101)
m = 28
a = (mods.h[m], mods.alpha[m], mods.beta[m], mods.rho[m])
lam = synth.geom(60.0, 0.8, 24)[:2]
c = 0.5 * (np.arange(1000, dtype=np.float64) + 1.0)
for j in range(0, 4):
    for l in lam:
        m64, e64, _ = oracle.det(*a, float(l), float(c[j]))
        mld, eld, _ = oracle.det(*a, float(l), float(c[j]), extended=True)
        print(f"lam={l:.3f} c={c[j]}: fp64 {m64.real * 2.0**e64:+.6e}  long double {mld.real * 2.0**eld:+.6e}")
for fl, name in ((0, "direct"), (masw.STABLE, "stable"), (masw.SCHED_ROWS, "rows")):
    st, ct, idx = masw.masw_curve(*a, lam, c, flags=fl)
    print(name, st, idx)
st, ct, idx, nd = oracle.curve(*a, lam, c)
print("oracle", st, idx)
try:
    import mpmath  # noqa: F401
    sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
    from test_oracle_pins import _mp_det
    for j in range(0, 3):
        print("mpmath", c[j], [float(_mp_det(*a, float(l), float(c[j]), k_double=True).real) for l in lam])
except Exception as e:
    print("mpmath unavailable:", str(e)[:200])
