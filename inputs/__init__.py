"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the sieve method: it only defines the
workloads of BASELINE.json (``configs``) as integer ranges and draws the
seeded random intervals.  Both the tests/bench (which drive the oracle and the
CUDA path) import it; neither side's arithmetic lives here.

Readings:
  R1  ranges are half-open [lo, hi); "[2, N]" means [2, N+1).
  R11 config 5 "drawn from seed 0": splitmix64 with state 0; per interval
      draw lo = 1e9 + x mod (1e13 - 1e9 + 1) then width = 1e5 + y mod
      (1e7 - 1e5 + 1); interval [lo, lo + width).
  R12 config 4 sub-windows: K = 16 windows of width 1e7, starts
      L + x_i mod (W - 1e7 + 1), x_i from splitmix64 with state 1.
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1


class SplitMix64:
    """splitmix64 (Steele, Lea, Flood 2014), all arithmetic mod 2^64."""

    def __init__(self, state: int):
        self.s = state & MASK64

    def next(self) -> int:
        self.s = (self.s + 0x9E3779B97F4A7C15) & MASK64
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)


# ---- the five workloads of BASELINE.json "configs" ----------------------
CONFIG1 = (2, 10**7 + 1)            # [2, 10^7]
CONFIG2 = (2, 10**9 + 1)            # [2, 10^9]
CONFIG3 = (2, 10**10 + 1)           # [2, 10^10]  -- the headline metric
CONFIG4 = (10**12, 10**12 + 10**10)  # [L, L+W)
CONFIG5_N = 4096


def config5_intervals(n: int = CONFIG5_N, seed: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """Reading R11: (lo[], hi[]) uint64 of the config-5 batch."""
    g = SplitMix64(seed)
    lo = np.zeros(n, dtype=np.uint64)
    hi = np.zeros(n, dtype=np.uint64)
    for i in range(n):
        a = 10**9 + g.next() % (10**13 - 10**9 + 1)
        w = 10**5 + g.next() % (10**7 - 10**5 + 1)
        lo[i] = a
        hi[i] = a + w
    return lo, hi


def config4_subwindows(k: int = 16, width: int = 10**7, seed: int = 1) -> list[tuple[int, int]]:
    """Reading R12: K seeded sub-windows [s, s+width) of config 4's window."""
    L, H = CONFIG4
    W = H - L
    g = SplitMix64(seed)
    out = []
    for _ in range(k):
        s = L + g.next() % (W - width + 1)
        out.append((s, s + width))
    return out


def random_intervals(n: int, seed: int, lo_max: int, width_max: int) -> list[tuple[int, int]]:
    """Generic seeded intervals for parity sweeps: lo uniform in [0, lo_max],
    width uniform in [0, width_max] (empty intervals included)."""
    g = SplitMix64(seed)
    out = []
    for _ in range(n):
        a = g.next() % (lo_max + 1)
        w = g.next() % (width_max + 1)
        out.append((a, a + w))
    return out


def u64_stream(n: int, seed: int) -> np.ndarray:
    """n seeded uniform 64-bit values (splitmix64): the rand() draws of Alg. 3
     and random operands for the F2 parity tests.  Vectorised
    form of SplitMix64 (same sequence)."""
    s = (np.arange(1, n + 1, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
         + np.uint64(seed & MASK64))
    z = s
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))
