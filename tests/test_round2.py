"""The device's division-free round2 quotient (csrc/router.cuh) equals the
reference's std::round(x * 100.0) / 100.0 (env.hpp:82) on its fast range.
A sample here; `python tools/check_round2.py` walks every k in [1, 2^22]."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tools"))
import check_round2  # noqa: E402


def test_round2_fast_quotient_sample():
    rng = np.random.default_rng(7)
    ks = np.concatenate([np.arange(1, 20001),                      # capacity, small T^_c
                         rng.integers(20001, 1 << 22, 20000),      # the rest of the range
                         [(1 << 22) - 1, 1 << 22]])
    assert check_round2.check(ks) == []
