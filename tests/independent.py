"""Independent checkers that pin the oracle to something other than itself.

None of these share code with ``oracle/`` or the CUDA path; each is a
different algorithm for the same mathematical object, written from its
textbook definition:

* ``is_prime_td``      -- trial division, the definition quoted at PAPER.md:29
                          (Sec. 1: n is prime iff no prime <= sqrt(n) divides it).
* ``is_prime_mr``      -- deterministic Miller-Rabin with the first 12 prime
                          bases (exact for n < 3.3e24).  PAPER.md:237 names
                          Rabin-Miller as the improvement over Alg. 3.
* ``lucy_pi_sum``      -- the Lucy-Hedgehog recurrence (a Legendre-style
                          combinatorial count, cf. the "counting argument
                          based on the sieve of Eratosthenes"):
                          pi(x) and (sum of primes <= x) mod 2^64 without
                          enumerating the primes.
"""
from __future__ import annotations

import math

import numpy as np

MASK64 = (1 << 64) - 1


def is_prime_td(n: int) -> bool:
    if n < 2:
        return False
    if n < 4:
        return True
    if n % 2 == 0:
        return False
    d = 3
    while d * d <= n:
        if n % d == 0:
            return False
        d += 2
    return True


def primes_td(lo: int, hi: int) -> list[int]:
    return [n for n in range(lo, hi) if is_prime_td(n)]


_MR_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def is_prime_mr(n: int) -> bool:
    if n < 2:
        return False
    for p in _MR_BASES:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in _MR_BASES:
        x = pow(a, d, n)
        if x == 1 or x == n - 1:
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def _tri_mod64(v: np.ndarray) -> np.ndarray:
    """v(v+1)/2 mod 2^64 for uint64 arrays (halve the even factor first)."""
    v = v.astype(np.uint64)
    even = (v % np.uint64(2)) == 0
    a = np.where(even, v // np.uint64(2), v)
    b = np.where(even, v + np.uint64(1), (v + np.uint64(1)) // np.uint64(2))
    with np.errstate(over="ignore"):
        return a * b


def lucy_pi_sum(x: int) -> tuple[int, int]:
    """(pi(x), sum of primes <= x mod 2^64) by the Lucy-Hedgehog recurrence.

    S(v, p) = S(v, p-1) - [p prime] * (S(v//p, p-1) - S(p-1, p-1)), over the
    set V = { x//i } of all distinct floor quotients; the sum variant weights
    each removed integer by its value (the removed set is p * {survivors in
    [p, v//p]}).  All sums are taken mod 2^64 with numpy uint64 wraparound.
    """
    if x < 2:
        return 0, 0
    r = math.isqrt(x)
    # V sorted descending: x//1, x//2, ..., x//r, then the small values down to 1
    big = np.array([x // i for i in range(1, r + 1)], dtype=np.uint64)
    small_max = int(big[-1]) - 1
    small = np.arange(small_max, 0, -1, dtype=np.uint64)
    V = np.concatenate([big, small])
    nV = V.size
    cnt = V.astype(np.int64) - 1                  # integers 2..v
    with np.errstate(over="ignore"):
        sm = _tri_mod64(V) - np.uint64(1)         # sum of 2..v mod 2^64

    def idx(v: np.ndarray) -> np.ndarray:
        # position of value v in V: big part if v > small_max, else small part
        v = v.astype(np.int64)
        out = np.empty(v.shape, dtype=np.int64)
        isbig = v > small_max
        out[isbig] = (x // v[isbig]) - 1
        out[~isbig] = nV - v[~isbig]
        return out

    for p in range(2, r + 1):
        ip = nV - p                                # index of v = p
        ipm1 = nV - (p - 1)                        # index of v = p-1
        if cnt[ip] == cnt[ipm1]:
            continue                               # p not prime
        c_pm1 = cnt[ipm1]
        s_pm1 = sm[ipm1]
        p2 = p * p
        k = int(np.searchsorted(-V.astype(np.int64), -p2, side="right"))  # V[:k] >= p^2
        if k == 0:
            break
        vv = V[:k]
        j = idx(vv // np.uint64(p))
        cnt[:k] -= cnt[j] - c_pm1
        with np.errstate(over="ignore"):
            sm[:k] -= np.uint64(p) * (sm[j] - s_pm1)
    return int(cnt[0]), int(sm[0])


def lucy_interval(lo: int, hi: int) -> tuple[int, int]:
    """(count, sum mod 2^64) of primes in [lo, hi) as a Lucy difference."""
    if hi <= lo:
        return 0, 0
    c1, s1 = lucy_pi_sum(hi - 1)
    c0, s0 = lucy_pi_sum(lo - 1) if lo >= 2 else (0, 0)
    return c1 - c0, (s1 - s0) & MASK64
