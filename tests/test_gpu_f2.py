"""§8(f) f2: the dense-LU comparison arm of scripts/dense_lu_baseline.py
and the banded det grid, both checked against the oracle on a seeded sample of the C4 and C3
grids the throughput comparison runs on (profiles/r2/dense_lu_baseline.json).

  * sign of Re det K: dense assembly + batched LU, banded GEPP values (masw_det_grid) and the
    oracle agree wherever the oracle's sign is decided (|Re det| >= 1e-6 |det|);
  * banded values within the north star's 1e-9 inside the det-parity domain (S15, S15').
"""
import os
import sys

import numpy as np
import pytest

import synth
import masw_parity as parity

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                "scripts"))


@pytest.fixture(scope="module")
def masw():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2003_02256_b200 as m

    m.lib()
    return m


def sample_points(L, V, n_rows, per_row, seed):
    rng = np.random.default_rng(seed)
    rows = np.sort(rng.choice(L, size=n_rows, replace=False))
    return [(int(i), np.sort(rng.choice(V, size=per_row, replace=False))) for i in rows]


@pytest.mark.parametrize("name,lam_override", [
    ("realistic", None),
    ("uniform", np.tile([1.0, 30.0, 200.0], 334)[:1000]),
])
def test_dense_lu_and_banded_signs_vs_oracle(masw, orc, name, lam_override):
    import dense_lu_baseline as dlb

    w = synth.workload(name)
    lam = w.lam if lam_override is None else lam_override
    m = w.models
    a = (m.h[0], m.alpha[0], m.beta[0], m.rho[0])
    ta = [torch.as_tensor(x, device="cuda") for x in a]
    pts = sample_points(len(lam), len(w.c), 12, 25, seed=2003 + len(lam))
    n_dec = n_agree = n_dom = 0
    worst = 0.0
    for i, js in pts:
        # banded values of the whole row (the grid kernel's launch), then the sampled points
        gre, gim, gex = masw.masw_det_grid(*a, lam[i:i + 1], w.c)
        lam_pts = torch.full((len(js),), float(lam[i]), dtype=torch.float64, device="cuda")
        c_pts = torch.as_tensor(w.c[js], device="cuda")
        dd = dlb.dense_det_points(*ta, lam_pts, c_pts).cpu().numpy()
        for t, j in enumerate(js):
            om, oe, st = orc.det(*a, float(lam[i]), float(w.c[j]))
            assert st == 0
            if abs(om.real) < 1e-6 * abs(om):
                continue          # the oracle's sign is not decided to this margin
            n_dec += 1
            so = np.sign(om.real)
            sb = np.sign(gre[0, j])
            sd = np.sign(dd[t].real)
            n_agree += int(so == sb == sd)
            kap = orc.det_kappa(*a, float(lam[i]), float(w.c[j]))
            if w.c[j] >= 0.5 * m.beta[0].min() and kap <= parity.KAPPA_MAX:
                n_dom += 1
                rel = parity.det_grid_rel_err(np.array([gre[0, j] + 1j * gim[0, j]]),
                                              np.array([gex[0, j]]), np.array([om]),
                                              np.array([oe]))[0]
                worst = max(worst, float(rel))
    assert n_dec >= 250, n_dec
    assert n_agree == n_dec, (n_agree, n_dec)
    assert n_dom >= 100, n_dom
    assert worst <= parity.DET_RTOL, worst
