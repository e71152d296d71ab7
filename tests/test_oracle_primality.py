"""Pins of the F2 oracle (oracle/primality.c: PAPER.md Alg. 2 and Alg. 3)
against things other than itself: SPEC.md's worked examples, naive repeated
multiplication, Python's built-in three-argument pow (an independent
library routine), trial division, Fermat's little theorem on primes, and the
Carmichael numbers below 2000 (561, 1105, 1729: SPEC.md carmichael_scan)."""
import math

import numpy as np

import inputs
import oracle
from independent import is_prime_td

U64MAX = (1 << 64) - 1


def test_modpow_spec_examples():
    # SPEC.md mod_pow: (2,10,1000) -> 24; (2,340,341) -> 1; (a,0,c) -> 1 mod c (0 for c = 1)
    assert oracle.modpow(2, 10, 1000) == 24
    assert oracle.modpow(2, 340, 341) == 1
    assert oracle.modpow(3, 340, 341) == 56   # SPEC.md fermat_test example for 341
    assert oracle.modpow(12345, 0, 97) == 1
    assert oracle.modpow(12345, 0, 1) == 0
    assert oracle.modpow(0, 0, 7) == 1          # Alg. 2: the loop never runs, x = 1
    assert oracle.modpow(5, 7, 0) == U64MAX     # c = 0: domain error marker


def test_modpow_vs_naive_exhaustive():
    """a, b < 24 and 1 <= c < 24: the O(b) repeated multiplication of PAPER.md:178."""
    for c in range(1, 24):
        for a in range(24):
            x = 1 % c
            for b in range(24):
                assert oracle.modpow(a, b, c) == x, (a, b, c)
                x = (x * a) % c


def test_modpow_vs_python_pow_random_64bit():
    r = inputs.u64_stream(3 * 3000, seed=11).reshape(3, -1)
    cs = [int(x) | 1 if k % 3 else int(x) for k, x in enumerate(r[2])]
    cs[:8] = [1, 2, 3, U64MAX, U64MAX - 1, (1 << 63), (1 << 61) - 1, 4]
    for a, b, c in zip(r[0].tolist(), r[1].tolist(), cs):
        c = max(c, 1)
        assert oracle.modpow(a, b, c) == pow(a, b, c), (a, b, c)
    got = oracle.modpow_batch(r[0], r[1], np.maximum(np.array(cs, dtype=np.uint64), 1))
    assert got.tolist() == [pow(a, b, max(c, 1)) for a, b, c in zip(r[0].tolist(), r[1].tolist(), cs)]


def test_fermat_guard_and_primes():
    d = inputs.u64_stream(20, seed=3)
    assert oracle.fermat(1, 5, d) is False          # Alg. 3: "if p = 1 return false"
    assert oracle.fermat(0, 5, d) is False          # domain error reported as false
    assert oracle.fermat(2, 5, d) is True           # a = rand mod 1 + 1 = 1 (SPEC.md note)
    primes = [n for n in range(2, 10**4) if is_prime_td(n)]
    draws = inputs.u64_stream(len(primes) * 20, seed=4)
    verdict = oracle.fermat_batch(np.array(primes, dtype=np.uint64), draws, 20)
    assert verdict.all()                             # Eq. 6: a prime is never rejected


def test_fermat_341_forced_bases():
    # SPEC.md: base 2 passes (341 = 11*31 is a base-2 pseudoprime), base 3 rejects
    assert oracle.fermat(341, 1, [1]) is True        # a = 1 mod 340 + 1 = 2
    assert oracle.fermat(341, 1, [2]) is False       # a = 3
    assert oracle.fermat(341, 2, [1, 2]) is False


def test_carmichael_numbers_below_2000():
    """Composite n whose every coprime base passes Alg. 3's test: exactly
    561, 1105, 1729 below 2000 (SPEC.md carmichael_scan)."""
    found = []
    for n in range(3, 2000):
        if is_prime_td(n):
            continue
        bases = np.array([a for a in range(2, n) if math.gcd(a, n) == 1], dtype=np.uint64)
        got = oracle.modpow_batch(bases, np.full(bases.size, n - 1, dtype=np.uint64),
                                  np.full(bases.size, n, dtype=np.uint64))
        if bases.size and (got == 1).all():
            found.append(n)
    assert found == [561, 1105, 1729]
    assert 561 == 3 * 11 * 17 and 1105 == 5 * 13 * 17 and 1729 == 7 * 13 * 19


def test_fermat_composites_mostly_rejected():
    """Composites that are not Carmichael numbers fail for most draws."""
    comps = np.array([n for n in range(4, 3000) if not is_prime_td(n) and n not in (561, 1105, 1729)],
                     dtype=np.uint64)
    verdict = oracle.fermat_batch(comps, inputs.u64_stream(comps.size * 8, seed=5), 8)
    assert verdict.mean() < 0.01
