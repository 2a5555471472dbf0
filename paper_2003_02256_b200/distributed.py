"""Multi-GPU sharding of the forward model: one process per GPU, torch.distributed (NCCL over
NVLink/NVSwitch) for the single exchange step.

Two shardings, both from the paper's MPI design, re-done for a box of GPUs:

* ensemble (config C5): models are independent ("each of these curves and their
  misfits can be computed independently"), so each rank runs ``masw_curves_ensemble`` on a
  contiguous block of models; C_t, idx and misfits are then all-gathered (the one
  collective) and every rank takes the argmin (ties -> lowest global id).
* one huge curve (configs C3/C4): wavelengths are partitioned modularly, i mod s
  (the paper's fix for decreasing curves), each rank scans its
  wavelengths (no communication), C_t/idx are all-gathered and inverse-permuted,
  and the misfit is evaluated once on the gathered curve by the same kernel on every rank,
  so results are bitwise identical to one GPU (the paper's "one reduction").

The per-rank compute goes through ``ops`` (default: the CUDA library); tests inject a CPU
implementation to exercise this host logic with the gloo backend.
"""
from __future__ import annotations

import dataclasses
from typing import Callable, List, Optional, Sequence

import torch
import torch.distributed as dist


# ------------------------------------------------------------------ partitions

def partition_wavelengths(W: int, s: int, strategy: str = "modular") -> List[List[int]]:
    """Wavelength index lists per worker.

    contiguous: worker k gets a contiguous run, earlier workers take the extra element
                ("assign wavelengths contiguously"; W=40, s=3 -> 14,13,13,
                PAPER.md:216).
    modular:    worker k gets every index i with i mod s == k.
    """
    if W < 0 or s < 1:
        raise ValueError("need W >= 0, s >= 1")
    if strategy == "modular":
        return [list(range(k, W, s)) for k in range(s)]
    if strategy == "contiguous":
        base, extra = divmod(W, s)
        out, lo = [], 0
        for k in range(s):
            n = base + (1 if k < extra else 0)
            out.append(list(range(lo, lo + n)))
            lo += n
        return out
    raise ValueError(f"unknown strategy {strategy!r}")


_INDEX_CACHE: dict = {}


def partition_index(W: int, s: int, rank: int, strategy: str, device) -> tuple:
    """(this rank's wavelength indices, the concatenated order of all ranks' indices) as
    int64 tensors on `device` -- partition_wavelengths as device index vectors, built once
    per (W, s, rank, strategy, device) (a 10k-entry Python list per call cost ~1 ms)."""
    key = (W, s, rank, strategy, str(device))
    hit = _INDEX_CACHE.get(key)
    if hit is not None:
        return hit
    parts = partition_wavelengths(W, s, strategy)
    mine = torch.as_tensor(parts[rank], dtype=torch.int64).to(device)
    order = torch.as_tensor([i for p in parts for i in p], dtype=torch.int64).to(device)
    if len(_INDEX_CACHE) > 64:
        _INDEX_CACHE.clear()
    _INDEX_CACHE[key] = (mine, order, [len(p) for p in parts])
    return _INDEX_CACHE[key]


def shard_bounds(M: int, world: int, rank: int):
    """Contiguous model block [lo, hi) of `rank` (earlier ranks take the extra model)."""
    base, extra = divmod(M, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


# ------------------------------------------------------------------ per-rank compute hooks

@dataclasses.dataclass
class Ops:
    """Per-rank compute used by the sharded drivers (tensors on the rank's device)."""

    curves_ensemble: Callable  # (h, alpha, beta, rho, lam, c, ce) -> (status, ct, idx, misfit)
    curve: Callable            # (h, alpha, beta, rho, lam, c) -> (status, ct, idx)
    misfit: Callable           # (ct, ce) -> float
    argmin: Callable           # (misfit) -> (best, value)


def cuda_ops(flags: int = 0, team_warps: int = 0) -> Ops:
    """The CUDA library as per-rank compute.  A failing call (invalid model in this rank's
    shard, out-of-range k h, ...) does NOT raise here: it returns its negative status with
    NaN / -1 outputs, so every rank still reaches the status all-gather and the drivers raise
    on ALL ranks together (raising on one rank would leave the others blocked in the
    collective)."""
    from . import masw

    def ens(h, a, b, r, lam, c, ce):
        try:
            res = masw.masw_curves_ensemble(h, a, b, r, lam, c, ce, flags=flags,
                                            team_warps=team_warps)
            return res.status, res.ct, res.idx, res.misfit
        except masw.MaswError as e:
            M, L = h.shape[0], lam.shape[0]
            return (e.code, _filled((M, L), float("nan"), torch.float64, lam),
                    _filled((M, L), -1, torch.int32, lam),
                    _filled((M,), float("nan"), torch.float64, lam))

    def cur(h, a, b, r, lam, c):
        try:
            return tuple(masw.masw_curve(h, a, b, r, lam, c, flags=flags, team_warps=team_warps))
        except masw.MaswError as e:
            L = lam.shape[0]
            return (e.code, _filled((L,), float("nan"), torch.float64, lam),
                    _filled((L,), -1, torch.int32, lam))

    def argmin(v):
        b, val = masw.masw_argmin(v)
        return b, val

    return Ops(ens, cur, masw.masw_misfit, argmin)


def _filled(shape, value, dtype, like):
    return torch.full(shape, value, dtype=dtype, device=like.device)


class ShardError(RuntimeError):
    """A rank's shard failed (worst status over all ranks < 0); raised on every rank."""

    def __init__(self, code: int, statuses):
        self.code = int(code)
        self.statuses = [int(x) for x in statuses]
        super().__init__(f"sharded call failed: worst status {code} (per rank {self.statuses})")


def worst_status(st: int, device, group=None) -> int:
    """Worst status over ranks (errors negative, the warning positive); raises ShardError on
    every rank if any rank failed."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    sts = [int(st)]
    if dist.is_initialized():   # (also at world size 1: the same collective code path)
        t = torch.tensor([int(st)], dtype=torch.int64, device=device)
        sts = _all_gather_padded(t, [1] * world, group).tolist()
    lo, hi = min(sts), max(sts)
    if lo < 0:
        raise ShardError(lo, sts)
    return hi


# ------------------------------------------------------------------ collectives

def _all_gather_padded(x: torch.Tensor, counts: Sequence[int], group=None) -> torch.Tensor:
    """Concatenate per-rank first-dim blocks of unequal size (pad to the max, one
    all_gather_into_tensor, trim).  The same collective on every backend (NCCL on the GPU
    box, gloo in the CPU tests)."""
    world = len(counts)
    if world == 1 and not dist.is_initialized():
        return x
    mx = max(counts)
    if x.shape[0] == mx:
        pad = x.contiguous()
    else:
        pad = torch.zeros((mx,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        pad[: x.shape[0]] = x
    out = torch.empty((world * mx,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    if all(cnt == mx for cnt in counts):
        return out
    return torch.cat([out[k * mx: k * mx + counts[k]] for k in range(world)], dim=0)


@dataclasses.dataclass
class EnsembleOut:
    status: int
    ct: torch.Tensor       # [M][L] all models (gathered)
    idx: torch.Tensor      # [M][L]
    misfit: torch.Tensor   # [M]
    best: int
    best_misfit: float


def ensemble_sharded(models_all, lam, c, ce, ops: Optional[Ops] = None, group=None,
                     device=None) -> EnsembleOut:
    """C5 driver: shard models contiguously, compute, all-gather, argmin on every rank.

    ``models_all`` is a tuple (h, alpha, beta, rho) of the FULL ensemble (host or device);
    each rank slices its block.  Returns gathered results identical on every rank.
    """
    ops = ops or cuda_ops()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    h, a, b, r = models_all
    M = h.shape[0]
    lo, hi = shard_bounds(M, world, rank)
    mv = lambda t: t[lo:hi].to(device) if device is not None else t[lo:hi]
    counts = [shard_bounds(M, world, k)[1] - shard_bounds(M, world, k)[0] for k in range(world)]
    L = lam.shape[0]
    if hi > lo:
        st, ct, idx, mis = ops.curves_ensemble(mv(h), mv(a), mv(b), mv(r), lam, c, ce)
    else:   # more ranks than models: an empty shard takes part in the collectives only
        st, ct, idx, mis = (0, _filled((0, L), 0.0, torch.float64, lam),
                            _filled((0, L), 0, torch.int32, lam),
                            _filled((0,), 0.0, torch.float64, lam))
    # worst status over ranks; every rank raises together if one failed
    st = worst_status(st, ct.device, group)
    ct_all = _all_gather_padded(ct, counts, group)
    idx_all = _all_gather_padded(idx, counts, group)
    mis_all = _all_gather_padded(mis, counts, group)
    best, bval = ops.argmin(mis_all)
    return EnsembleOut(st, ct_all, idx_all, mis_all, int(best[0]), float(bval[0]))


@dataclasses.dataclass
class CurveOut:
    status: int
    ct: torch.Tensor
    idx: torch.Tensor
    misfit: Optional[float]


def curve_sharded(model, lam: torch.Tensor, c, ce=None, strategy: str = "modular",
                  ops: Optional[Ops] = None, group=None) -> CurveOut:
    """C3/C4 driver: one model, wavelengths partitioned over ranks."""
    ops = ops or cuda_ops()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    W = lam.shape[0]
    mine, order, counts = partition_index(W, world, rank, strategy, lam.device)
    if counts[rank] > 0:
        st, ct, idx = ops.curve(*model, lam[mine], c)
    else:   # W < world: an empty shard takes part in the collectives only
        st, ct, idx = (0, _filled((0,), 0.0, torch.float64, lam),
                       _filled((0,), 0, torch.int32, lam))
    st = worst_status(st, ct.device, group)
    ct_g = _all_gather_padded(ct, counts, group)
    idx_g = _all_gather_padded(idx, counts, group)
    order = order.to(ct_g.device)
    ct_full = torch.empty_like(ct_g)
    idx_full = torch.empty_like(idx_g)
    ct_full[order] = ct_g
    idx_full[order] = idx_g
    mis = ops.misfit(ct_full, ce) if ce is not None else None
    return CurveOut(st, ct_full, idx_full, mis)
