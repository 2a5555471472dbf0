"""Seeded synthetic inputs for the five workloads (SURVEY.md §8(d) "Concrete synthetic inputs").

This module is the ONLY code shared by the oracle side (``oracle/``, ``tests/``) and the
CUDA side (``paper_2003_02256_b200``).  It holds none of the method's arithmetic: it only
lays out model parameters, wavelength lists and test-velocity grids as fp64 arrays, and
loads experimental curves C_e that a committed oracle-only script wrote under
``tests/golden/`` (``scripts/make_golden.py``).

Shapes follow the paper's workloads:
  * PAPER.md:76  "up to 100 wavelengths and 1,000 test velocities"
  * PAPER.md:170 "uniform" (identical wavelengths) and "variable" (decreasing) datasets
  * PAPER.md:216 "the variable dispersion curve has 40 entries"
  * PAPER.md:99  "an exhaustive quantity of plausible model parameters" (ensemble)

Layout (the C-ABI's, include/masw.h): structure-of-arrays, row-major
``h[M][N]``, ``alpha/beta/rho[M][N+1]`` (index N is the half-space), SI units.
"""
from __future__ import annotations

import dataclasses
import os
from typing import Optional

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")

#: PCG64 seed of the Monte-Carlo ensemble.
ENSEMBLE_SEED = 200302256


def geom(a: float, b: float, n: int) -> np.ndarray:
    """``geom(a,b,n)`` of SURVEY.md §8(d): a·(b/a)^{i/(n−1)}, i = 0..n−1 (fp64)."""
    i = np.arange(n, dtype=np.float64)
    return (a * (b / a) ** (i / (n - 1))).astype(np.float64)


@dataclasses.dataclass
class Models:
    """Structure-of-arrays layered models: ``h[M][N]``, ``alpha, beta, rho[M][N+1]``."""

    h: np.ndarray
    alpha: np.ndarray
    beta: np.ndarray
    rho: np.ndarray

    @property
    def n_models(self) -> int:
        return int(self.h.shape[0])

    @property
    def n_layers(self) -> int:
        return int(self.h.shape[1])

    def model(self, m: int) -> "Models":
        return Models(self.h[m:m + 1], self.alpha[m:m + 1], self.beta[m:m + 1], self.rho[m:m + 1])

    def slice(self, lo: int, hi: int) -> "Models":
        return Models(self.h[lo:hi], self.alpha[lo:hi], self.beta[lo:hi], self.rho[lo:hi])

    def take(self, ids) -> "Models":
        ids = np.asarray(ids, dtype=np.int64)
        return Models(self.h[ids], self.alpha[ids], self.beta[ids], self.rho[ids])


@dataclasses.dataclass
class Workload:
    name: str
    models: Models
    lam: np.ndarray          # [L] wavelengths, m
    c: np.ndarray            # [V] test velocities, m/s, strictly increasing
    ce: Optional[np.ndarray]  # [L] experimental curve C_e (or None)
    note: str = ""


def _single(h, alpha, beta, rho) -> Models:
    f = lambda x: np.ascontiguousarray(np.asarray(x, dtype=np.float64)[None, :])
    return Models(f(h), f(alpha), f(beta), f(rho))


# ---------------------------------------------------------------- the five configs

def tiny_model() -> Models:
    """C1: N=2, h=[2,4] m, β=[120,200,320], α=2β (ν=1/3), ρ=[1800,1900,2000]."""
    beta = np.array([120.0, 200.0, 320.0])
    return _single([2.0, 4.0], 2.0 * beta, beta, [1800.0, 1900.0, 2000.0])


def maswaves_model(twin: bool = False) -> Models:
    """C2: MASWaves-style 5 layers + half-space.

    ``twin=True`` gives the N=6 twin whose extra 5 m layer equals the half-space (P6).
    """
    h = [1.0, 1.0, 2.0, 2.0, 4.0]
    beta = [75.0, 90.0, 150.0, 180.0, 240.0, 290.0]
    if twin:
        h = h + [5.0]
        beta = beta + [290.0]
    n1 = len(beta)
    return _single(h, [1440.0] * n1, beta, [1850.0] * n1)


def uniform_model() -> Models:
    """C3: N=10, h_e=1.5 m, β_e=100+25e, ν=0.3 ⇒ α=β·√3.5, ρ_e=1800+20e."""
    e = np.arange(11, dtype=np.float64)
    beta = 100.0 + 25.0 * e
    return _single(np.full(10, 1.5), beta * np.sqrt(3.5), beta, 1800.0 + 20.0 * e)


def ensemble_models(M: int = 100_000, seed: int = ENSEMBLE_SEED) -> Models:
    """C5: M random 6-layer models, PCG64(seed).

    Each model draws 20 uniforms u in [0, 1) in order (row-major over models, so any prefix
    of a larger ensemble is bit-identical): β_e = β_ref,e·(0.6 + 0.8 u_e) (e < 7),
    h_e = h_ref,e·(0.5 + u_{7+e}) (e < 6), ρ_e = 1700 + 300 u_{13+e} (e < 7); α = 1440.
    Velocity reversals are allowed.
    """
    beta_ref = np.array([75.0, 90.0, 150.0, 180.0, 240.0, 290.0, 290.0])
    h_ref = np.array([1.0, 1.0, 2.0, 2.0, 4.0, 5.0])
    rng = np.random.Generator(np.random.PCG64(seed))
    u = rng.random((M, 20))
    beta = np.ascontiguousarray(beta_ref[None, :] * (0.6 + 0.8 * u[:, 0:7]))
    h = np.ascontiguousarray(h_ref[None, :] * (0.5 + u[:, 7:13]))
    rho = np.ascontiguousarray(1700.0 + 300.0 * u[:, 13:20])
    alpha = np.full((M, 7), 1440.0)
    return Models(h, alpha, beta, rho)


def random_models(M: int, N: int, seed: int) -> Models:
    """Property-test models beyond the configs' shapes, PCG64(seed): per model and layer
    β ~ U(60, 500) m/s in any order (reversals, stiff lids, soft channels), Poisson ratios
    through α = β·U(1.6, 3.5), h ~ U(0.3, 8) m, ρ ~ U(1500, 2300) kg/m³."""
    rng = np.random.Generator(np.random.PCG64(seed))
    beta = rng.uniform(60.0, 500.0, (M, N + 1))
    alpha = beta * rng.uniform(1.6, 3.5, (M, N + 1))
    h = rng.uniform(0.3, 8.0, (M, N))
    rho = rng.uniform(1500.0, 2300.0, (M, N + 1))
    return Models(np.ascontiguousarray(h), np.ascontiguousarray(alpha),
                  np.ascontiguousarray(beta), np.ascontiguousarray(rho))


def tiny_lambdas() -> np.ndarray:
    return geom(60.0, 2.0, 20)


def tiny_grid() -> np.ndarray:
    return 40.0 + 0.5 * np.arange(1000, dtype=np.float64)


def variable_lambdas() -> np.ndarray:
    """The paper's 40-entry decreasing "variable" curve."""
    return geom(40.0, 1.0, 40)


def maswaves_grid() -> np.ndarray:
    """c_j = 0.5(j+1), j<1000 (≈1000 test velocities)."""
    return 0.5 * (np.arange(1000, dtype=np.float64) + 1.0)


UNIFORM_TIERS = (1.0, 30.0, 200.0)


def uniform_grid() -> np.ndarray:
    return 20.0 + 0.04 * np.arange(10_000, dtype=np.float64)


def realistic_lambdas() -> np.ndarray:
    return geom(100.0, 0.5, 10_000)


def realistic_grid() -> np.ndarray:
    return 15.0 + 0.03 * np.arange(10_000, dtype=np.float64)


# ---------------------------------------------------------------- experimental curves

def load_golden(name: str) -> np.ndarray:
    """Load a golden fp64 column written by scripts/make_golden.py (oracle only)."""
    path = os.path.join(GOLDEN_DIR, name)
    vals = []
    with open(path) as fh:
        for line in fh:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            vals.append(float(line.split()[-1]))
    return np.asarray(vals, dtype=np.float64)


def perturbed_ce(ce: np.ndarray) -> np.ndarray:
    """Second, non-trivial C_e: C_e,i·(1 + 0.02 sin i)."""
    i = np.arange(ce.shape[0], dtype=np.float64)
    return ce * (1.0 + 0.02 * np.sin(i))


def _ce_or_none(name: str) -> Optional[np.ndarray]:
    try:
        return load_golden(name)
    except FileNotFoundError:
        return None


# ---------------------------------------------------------------- workload factory

def workload(name: str, **kw) -> Workload:
    """Return a named workload: tiny | maswaves | maswaves_twin | uniform | realistic | ensemble."""
    if name == "tiny":
        lam = tiny_lambdas()
        ce = _ce_or_none("c1_ct_oracle.txt")
        return Workload(name, tiny_model(), lam, tiny_grid(), ce, "C1 tiny N=2, 20 λ × 1000 c")
    if name in ("maswaves", "maswaves_twin"):
        ce = _ce_or_none("c2_ct_oracle.txt")
        return Workload(name, maswaves_model(twin=name.endswith("twin")), variable_lambdas(),
                        maswaves_grid(), ce, "C2 MASWaves-style, 40 λ × 1000 c")
    if name == "uniform":
        tier = float(kw.get("tier", 200.0))
        L = int(kw.get("L", 10_000))
        lam = np.full(L, tier, dtype=np.float64)
        ce = None
        g = _ce_or_none("c3_ct_oracle.txt")
        if g is not None:
            tiers = load_golden_tiers()
            if tier in tiers:
                ce = np.full(L, tiers[tier], dtype=np.float64)
        return Workload(name, uniform_model(), lam, uniform_grid(), ce,
                        f"C3 uniform N=10, {L} × λ={tier} m × 10k c")
    if name == "realistic":
        ce = _ce_or_none("c4_ct_oracle.txt")
        return Workload(name, maswaves_model(), realistic_lambdas(), realistic_grid(), ce,
                        "C4 realistic N=5, 10k λ (100→0.5 m) × 10k c")
    if name == "ensemble":
        M = int(kw.get("M", 100_000))
        ce = _ce_or_none("c2_ct_oracle.txt")
        return Workload(name, ensemble_models(M), variable_lambdas(), maswaves_grid(), ce,
                        f"C5 ensemble {M} random N=6 models × 40 λ × 1000 c")
    raise KeyError(name)


def load_golden_tiers() -> dict:
    """C3 tier → oracle C_t (file rows: 'lambda idx ct')."""
    out = {}
    path = os.path.join(GOLDEN_DIR, "c3_ct_oracle.txt")
    with open(path) as fh:
        for line in fh:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            parts = line.split()
            out[float(parts[0])] = float(parts[-1])
    return out


WORKLOADS = ("tiny", "maswaves", "maswaves_twin", "uniform", "realistic", "ensemble")
