"""B200-native MASW theoretical dispersion-curve forward model (arXiv:2003.02256).

The compute lives in libmasw.so (hand-written sm_100a CUDA, C ABI in include/masw.h);
this package is the thin ctypes binding (``masw``), the multi-GPU sharding over
torch.distributed/NCCL (``distributed``) and the nvcc build (``build``).
"""
from .masw import (  # noqa: F401
    ASYNC, E_ARG, E_CUDA, E_GRID, E_MODEL, E_NOMEM, E_NONFINITE, E_RANGE, IDX_NO_CHANGE,
    IDX_NONFINITE, OK, PIVOTED, DIRECT, SCHED_CONTIGUOUS, SCHED_MODELS, SCHED_MODULAR, SCHED_PAIRS,
    SCHED_ROWS, STABLE, TEAM_STATS, TIME_SCAN, WARN_NO_SIGN_CHANGE, MaswError, lib, masw_argmin,
    masw_curve, masw_curves_ensemble, masw_det_grid, masw_kernel_launches, masw_last_scan_ms,
    masw_last_fallbacks, masw_last_prefix, masw_last_team_dets, masw_last_work, masw_misfit, masw_recent_scan_ms,
    masw_misfit_batch, masw_probe_fp64_peak)

__all__ = [n for n in dir() if n.startswith("masw_")] + ["MaswError", "lib"]
