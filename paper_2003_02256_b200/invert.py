"""Monte-Carlo inversion driver on top of masw_curves_ensemble.

The paper's method is a forward model used inside an optimisation loop: "the only way to
minimize the misfit is to compute theoretical dispersion curves for an exhaustive quantity
of plausible model parameters"; its stated future work is an I/O system and
command-line arguments.  This driver draws candidate layered models
uniformly within per-layer bounds, evaluates their misfits against an experimental curve in
batches on the GPU (sharded over ranks under torchrun, models in contiguous blocks with one
NCCL all-gather per batch), and keeps the best models (ties -> lowest id).

    python -m paper_2003_02256_b200.invert --curve ce.csv --bounds bounds.json \\
        --models 1000000 --batch 100000 --grid 0.5:500:0.5 --top 10 --out best.csv
    torchrun --nproc-per-node 8 -m paper_2003_02256_b200.invert ...

Files
  curve CSV:   header "wavelength_m,velocity_m_per_s", one row per wavelength (C_e).
  bounds JSON: {"h": [[lo, hi], ...N], "beta": [[lo, hi], ...N+1], "alpha": [[lo, hi], ...]
                or "alpha_over_beta": [lo, hi], "rho": [[lo, hi], ...N+1]}.
  output CSV:  rank, model_id, misfit, then h_0..h_{N-1}, alpha_0.., beta_0.., rho_0..
"""
from __future__ import annotations

import argparse
import csv
import json
import os
import sys
from typing import List, Optional, Tuple

import numpy as np


# ------------------------------------------------------------------ files

def read_curve(path: str) -> Tuple[np.ndarray, np.ndarray]:
    lam, vel = [], []
    with open(path) as fh:
        for row in csv.reader(fh):
            if not row or row[0].strip().startswith("#"):
                continue
            try:
                a, b = float(row[0]), float(row[1])
            except ValueError:
                continue                       # header
            lam.append(a)
            vel.append(b)
    if not lam:
        raise ValueError(f"{path}: empty curve")
    return np.asarray(lam), np.asarray(vel)


def write_curve(path: str, lam, vel) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["wavelength_m", "velocity_m_per_s"])
        for a, b in zip(lam, vel):
            w.writerow([repr(float(a)), repr(float(b))])


def parse_grid(spec: str) -> np.ndarray:
    """'lo:hi:step' -> [lo, lo+step, ...] up to and including the largest value <= hi."""
    lo, hi, step = (float(x) for x in spec.split(":"))
    if not (lo > 0 and step > 0 and hi > lo):
        raise ValueError("grid needs 0 < lo < hi and step > 0")
    n = int(np.floor((hi - lo) / step + 1e-9)) + 1
    if n < 2:
        raise ValueError("grid needs at least 2 velocities")
    return lo + step * np.arange(n, dtype=np.float64)


class Bounds:
    def __init__(self, spec: dict):
        self.h = np.asarray(spec["h"], dtype=np.float64)
        self.beta = np.asarray(spec["beta"], dtype=np.float64)
        self.rho = np.asarray(spec["rho"], dtype=np.float64)
        self.alpha = np.asarray(spec["alpha"], dtype=np.float64) if "alpha" in spec else None
        self.aob = np.asarray(spec["alpha_over_beta"], dtype=np.float64) if "alpha_over_beta" in spec else None
        self.N = self.h.shape[0]
        if self.beta.shape != (self.N + 1, 2) or self.rho.shape != (self.N + 1, 2):
            raise ValueError("bounds: beta and rho need N+1 [lo, hi] pairs")
        if self.alpha is None and self.aob is None:
            raise ValueError("bounds: give alpha or alpha_over_beta")

    def draw(self, rng: np.random.Generator, M: int):
        """M models, drawn per model row-major (prefix-stable for a given seed)."""
        N = self.N
        u = rng.random((M, 4 * N + 3))
        lerp = lambda b, x: b[:, 0] + (b[:, 1] - b[:, 0]) * x
        h = lerp(self.h, u[:, :N])
        beta = lerp(self.beta, u[:, N:2 * N + 1])
        rho = lerp(self.rho, u[:, 2 * N + 1:3 * N + 2])
        if self.alpha is not None:
            alpha = np.maximum(lerp(self.alpha, u[:, 3 * N + 2:4 * N + 3]), beta * (1 + 1e-6))
        else:
            alpha = beta * lerp(np.repeat(self.aob[None, :], N + 1, 0), u[:, 3 * N + 2:4 * N + 3])
        c = lambda x: np.ascontiguousarray(x, dtype=np.float64)
        return c(h), c(alpha), c(beta), c(rho)


# ------------------------------------------------------------------ search

def invert(lam, ce, c, bounds: Bounds, n_models: int, batch: int, seed: int, top: int,
           device=None, ops=None):
    """Returns (best list of (misfit, model_id, (h, alpha, beta, rho) row), models evaluated).

    Single process or under torch.distributed (each rank evaluates a contiguous block of
    every batch; misfits are all-gathered).  `ops` injects the per-rank compute (tests).
    """
    import torch
    import torch.distributed as dist

    from . import distributed as D

    rng = np.random.Generator(np.random.PCG64(seed))
    world = dist.get_world_size() if dist.is_initialized() else 1
    dev = device if device is not None else (torch.device("cuda", torch.cuda.current_device())
                                             if torch.cuda.is_available() else torch.device("cpu"))
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=dev)
    lam_t, c_t, ce_t = t(lam), t(c), t(ce)
    best: List[Tuple[float, int, tuple]] = []
    done = 0
    while done < n_models:
        B = min(batch, n_models - done)
        h, a, b, r = bounds.draw(rng, B)              # every rank draws the same batch
        out = D.ensemble_sharded((t(h), t(a), t(b), t(r)), lam_t, c_t, ce_t, ops=ops)
        mis = out.misfit.cpu().numpy() if hasattr(out.misfit, "cpu") else np.asarray(out.misfit)
        order = np.lexsort((np.arange(B), mis))[:top]  # misfit, then lowest id
        for k in order:
            best.append((float(mis[k]), done + int(k), (h[k], a[k], b[k], r[k])))
        best.sort(key=lambda x: (x[0], x[1]))
        best = best[:top]
        done += B
    return best, done


def write_report(path: str, best, N: int) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["rank", "model_id", "misfit"] + [f"h_{e}" for e in range(N)]
                   + [f"alpha_{e}" for e in range(N + 1)] + [f"beta_{e}" for e in range(N + 1)]
                   + [f"rho_{e}" for e in range(N + 1)])
        for k, (m, mid, (h, a, b, r)) in enumerate(best):
            w.writerow([k, mid, repr(m)] + [repr(float(x)) for x in (*h, *a, *b, *r)])


def main(argv: Optional[list] = None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--curve", required=True)
    ap.add_argument("--bounds", required=True)
    ap.add_argument("--models", type=int, default=100_000)
    ap.add_argument("--batch", type=int, default=100_000)
    ap.add_argument("--grid", default="0.5:500:0.5", help="test velocities lo:hi:step (m/s)")
    ap.add_argument("--top", type=int, default=10)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--out", default="best_models.csv")
    args = ap.parse_args(argv)
    if args.models < 1 or args.batch < 1 or args.top < 1:
        print("invert: --models, --batch and --top must be >= 1", file=sys.stderr)
        return 2

    import torch
    import torch.distributed as dist

    if int(os.environ.get("WORLD_SIZE", "1")) > 1 and not dist.is_initialized():
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    lam, ce = read_curve(args.curve)
    bounds = Bounds(json.load(open(args.bounds)))
    c = parse_grid(args.grid)
    best, n = invert(lam, ce, c, bounds, args.models, args.batch, args.seed, args.top)
    rank = dist.get_rank() if dist.is_initialized() else 0
    if rank == 0:
        write_report(args.out, best, bounds.N)
        print(f"invert: {n} models, best misfit {best[0][0]:.6g} (model {best[0][1]}) -> {args.out}")
    if dist.is_initialized():
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
