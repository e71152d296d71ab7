"""CPU pins of the roofline numerator bench.py reports:
M_alg = the number of (odd prime p, odd multiple m) pairs with
wheel < p <= isqrt(hi - 1) and max(lo, p^2) <= m < hi.

bench.algorithmic_marks counts them in closed form per prime; here they are
enumerated one by one on small ranges, and the config-3 totals are checked
against the values SURVEY.md 8(d) D2 quotes (6.02e9 marks at wheel 19) and
the w = 31 count VERDICT.md round 1 recomputed (5,470,683,379)."""
import math
import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def _brute(lo, hi, wheel):
    if hi <= lo:
        return 0
    r = math.isqrt(hi - 1) if hi >= 1 else 0
    total = 0
    for p in range(3, r + 1, 2):
        if p <= wheel or any(p % d == 0 for d in range(3, math.isqrt(p) + 1, 2)):
            continue
        for m in range(p * p, hi, 2 * p):  # odd multiples from p^2 on
            if m >= lo:
                total += 1
    return total


@pytest.mark.parametrize("lo,hi", [(0, 100), (2, 1001), (10, 5000), (4000, 9000), (1, 20000),
                                   (12345, 54321), (99_000, 101_001), (0, 10)])
@pytest.mark.parametrize("wheel", [2, 7, 19, 31])
def test_marks_brute_force(lo, hi, wheel):
    assert bench.algorithmic_marks(lo, hi, wheel) == _brute(lo, hi, wheel)


def test_marks_additive_over_blocks():
    # a range split into contiguous blocks: the per-block counts add up
    lo, hi = 2, 3_000_001
    cuts = [lo, 123_457, 1_000_003, 2_222_223, hi]
    parts = sum(bench.algorithmic_marks(a, b, 31) for a, b in zip(cuts, cuts[1:]))
    assert parts == bench.algorithmic_marks(lo, hi, 31)


def test_marks_config3():
    lo, hi = 2, 10**10 + 1
    assert bench.algorithmic_marks(lo, hi, 31) == 5_470_683_379
    m19 = bench.algorithmic_marks(lo, hi, 19)
    assert m19 == 6_021_778_759
    assert round(m19 / 1e9, 2) == 6.02
