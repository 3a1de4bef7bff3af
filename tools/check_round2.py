#!/usr/bin/env python
"""Exhaustive check of the device round2 quotient (csrc/router.cuh): for every
integer k in [1, K], q0 = RN(k * RN(0.01)), r = RN(k - 100 q0) (one FMA) is
exact, and RN(q0 + r * RN(0.01)) (one FMA) equals RN(k / 100).

    python tools/check_round2.py [K]      # default 2^22, the device's fast range (~1 min)

Exact rational arithmetic (fractions); float(Fraction) rounds to nearest even,
i.e. it is one correctly rounded FMA.
"""
import sys
from fractions import Fraction as F

import numpy as np


def check(ks):
    """Return the k (integers, as a numpy array) whose fast quotient is wrong."""
    y = 0.01
    fy = F(y)
    q0s = (np.asarray(ks, dtype=np.float64) * y).tolist()  # one RN multiply each
    bad = []
    for k, q in zip(np.asarray(ks).tolist(), q0s):
        r_exact = int(k) - 100 * F(q)
        r = float(r_exact)
        if F(r) != r_exact or float(F(q) + F(r) * fy) != float(F(int(k), 100)):
            bad.append(int(k))
    return bad


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
    bad = check(np.arange(1, K + 1))
    print(f"k in [1, {K}]: {len(bad)} mismatches" + (f", first {bad[:5]}" if bad else ""))
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
