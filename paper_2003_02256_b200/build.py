"""Build libmasw.so in-tree with nvcc for sm_100a (SASS only, no PTX JIT).

    python -m paper_2003_02256_b200.build [--force] [--verbose]
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libmasw.so")
SOURCES = ["masw_kernels.cu", "masw_capi.cu", "masw_probe.cu"]
HEADERS = ["masw_det.cuh", "masw_exp_table.h", "masw_internal.h"]
PUBLIC_HEADERS = [os.path.join(ROOT, "include", "masw.h"), os.path.join(ROOT, "include", "masw_probe.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "--expt-relaxed-constexpr",
         # ptxas register-usage heuristic at its most register-hungry setting (same-box A/B,
         # profiles/r2/ptxas_reglevel_ab.txt: C4 -2.1 %, C3 -0.3 %, C5 unchanged; idx identical)
         "-Xptxas", "-regUsageLevel=10"]


def _inputs():
    return ([os.path.join(CSRC, s) for s in SOURCES + HEADERS] + PUBLIC_HEADERS +
            [os.path.abspath(__file__)])


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _inputs())


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple = ()) -> str:
    """Compile libmasw.so (or a variant with extra -D defines into `out`)."""
    target = out or LIB
    if out is None and not force and not stale():
        return LIB
    objdir = os.path.join(PKG, "build")
    if out is not None:   # variant builds: their own objects (parallel builds do not collide)
        objdir = os.path.join(objdir, os.path.basename(out).replace(".", "_"))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for s in SOURCES:
        obj = os.path.join(objdir, s.replace(".cu", ".o"))
        extra = os.environ.get("MASW_NVCC_EXTRA", "").split() if out is not None else []
        cmd = [NVCC, *ARCH, *FLAGS, *extra, *[f"-D{d}" for d in defines], "-c",
               os.path.join(CSRC, s), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        objs.append(obj)
    tmp = target + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-cudart", "static"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    defs = tuple(a[2:] for a in sys.argv[1:] if a.startswith("-D"))
    outs = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv,
                out=outs[0] if outs else None, defines=defs))
