"""A bounded run of the randomised parity sweep (tests/fuzz/fuzz_parity.py, seed 2003, the first
450 calls: random layered models N = 1..12, wavelength ranges on both sides of the fine/coarse
cosh/sinh table boundary up to k h = 300, grids from 0.5 m/s or near the slowest layer, every
scan), each call's C_t against the CPU oracle under the S16 rule.  The full sweeps and their
results are in profiles/r2/fuzz_parity_*.json; this run includes three calls that exposed the
block-sign certificate's reciprocal-range bug."""
import os
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_random_sweep_first_450_calls():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sys.path.insert(0, os.path.join(ROOT, "tests", "fuzz"))
    os.environ.setdefault("FUZZ_SEED", "2003")
    import fuzz_parity

    st = fuzz_parity.run(budget=600.0, max_calls=450)
    assert st["calls"] + sum(1 for b in st["bad_cases"] if "error" in b) == 450
    assert st["rows"] > 250_000
    assert st["rows_bad"] == 0, st["bad_cases"][:5]
    assert st.get("misfit_bad", 0) == 0
