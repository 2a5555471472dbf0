"""CPU-only checks of the C ABI: libmasw.so builds for sm_100a, loads without a GPU, and
exports every function include/*.h declares; the product fails loudly without CUDA."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = []
    for fn in sorted(os.listdir(os.path.join(ROOT, "include"))):
        if not fn.endswith(".h"):
            continue
        src = open(os.path.join(ROOT, "include", fn)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(masw_\w+)\s*\(", src, re.M):
            names.append(m.group(1))
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    from paper_2003_02256_b200 import build

    build.build()
    return ctypes.CDLL(build.LIB)


def test_header_declares_the_boundary():
    names = declared_functions()
    for need in ("masw_curve", "masw_misfit", "masw_curves_ensemble", "masw_argmin",
                 "masw_det_grid", "masw_strerror", "masw_probe_fp64_peak"):
        assert need in names


def test_every_declared_symbol_is_exported(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_sass_is_sm100a_without_ptx(lib):
    from paper_2003_02256_b200 import build

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    ptx = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-ptx", build.LIB],
                         capture_output=True, text=True).stdout
    assert ".ptx" not in ptx


def test_strerror_and_version(lib):
    lib.masw_strerror.restype = ctypes.c_char_p
    assert lib.masw_version() == 1
    for code in (0, 1, -1, -2, -3, -4, -5, -6, -7):
        assert lib.masw_strerror(code).startswith(b"MASW_")


def test_arg_errors_need_no_gpu():
    import paper_2003_02256_b200 as m

    L = m.lib()
    assert L.masw_curve(None, None, 0, None, 0, None, None, None) == m.E_ARG
    assert L.masw_misfit(None, None, 0, None, None) == m.E_ARG
    assert L.masw_argmin(None, 0, None, None, None) == m.E_ARG


def test_product_fails_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2003_02256_b200 as m

    with pytest.raises(m.MaswError) as ei:
        m.masw_curve([1.0], [300.0, 300.0], [100.0, 100.0], [1.0, 1.0], [1.0], np.arange(1, 10.0))
    assert ei.value.code == m.E_CUDA


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2003_02256_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "oracle/" not in src.replace(
                    "oracle/ (", "").replace("shares nothing with oracle/", ""), f
