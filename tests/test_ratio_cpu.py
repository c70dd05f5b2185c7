"""The fusion's integer ratio cnt / pc (csrc/common.cuh ratio_rn) replaces
__ddiv_rn by a float reciprocal refined once in double, q0 = RN(cnt * r), the
exact fma residual and one correction fma.  This restates those operations
with exact rational arithmetic (an fma rounds once: float(Fraction) is the
correctly rounded double) and checks the result equals the correctly rounded
quotient -- for the float reciprocal exactly rounded and perturbed by one ulp
either way (MUFU.RCP is an approximation) -- over random and edge operands
below 2^24.  The GPU tests pin the fusion's priorities to the oracle."""
from fractions import Fraction

import numpy as np


def _fma(a: float, b: float, c: float) -> float:
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def _ratio(cnt: int, pc: int, pert: int) -> float:
    r0 = np.float32(1.0) / np.float32(pc)
    if pert:
        r0 = np.nextafter(r0, np.float32(np.inf if pert > 0 else -np.inf))
    r0 = float(r0)
    y, x = float(pc), float(cnt)
    r = _fma(r0, _fma(-y, r0, 1.0), r0)
    q0 = x * r
    return _fma(_fma(-q0, y, x), r, q0)


def test_ratio_rn_equals_correctly_rounded_division():
    rng = np.random.default_rng(11)
    pairs = [(1, 1), (1, 3), (2, 3), (7, 7), ((1 << 24) - 1, 1), (1, (1 << 24) - 1), ((1 << 24) - 1, (1 << 24) - 3),
             (5, 1 << 20), (3, 1 << 23), ((1 << 23) + 1, 3)]
    for _ in range(1500):
        pc = int(rng.integers(1, 1 << 24)) if rng.random() < 0.5 else int(rng.integers(1, 2048))
        cnt = int(rng.integers(1, 1 << 24)) if rng.random() < 0.5 else int(rng.integers(1, pc + 1))
        pairs.append((cnt, pc))
    for cnt, pc in pairs:
        want = cnt / pc  # Python float division is correctly rounded
        for pert in (-1, 0, 1):
            assert _ratio(cnt, pc, pert) == want, (cnt, pc, pert)
