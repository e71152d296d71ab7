"""GPU parity for SURVEY.md 8(f) F2 (paper_1205_4883_b200/csrc/primality.cu,
through the C ABI): Alg. 2 batched modpow and Alg. 3 batched Fermat against
the CPU oracle (oracle/primality.c) element by element, and the
deterministic Miller-Rabin verifier against the oracle's sieve."""
import numpy as np
import pytest

import inputs
import oracle
import paper_1205_4883_b200 as sv
from independent import is_prime_mr, is_prime_td

pytestmark = pytest.mark.gpu
U64MAX = (1 << 64) - 1


def _operands(n, seed):
    r = inputs.u64_stream(3 * n, seed=seed).reshape(3, n)
    a, b, c = r[0].copy(), r[1].copy(), r[2].copy()
    c[1::3] |= np.uint64(1)                     # odd moduli (Montgomery path)
    c[2::3] &= ~np.uint64(1)                    # even moduli (128-bit remainder path)
    c[2::9] >>= np.uint64(40)                   # small moduli
    edges = [(5, 7, 0), (5, 7, 1), (0, 0, 7), (U64MAX, U64MAX, U64MAX), (U64MAX, 2, U64MAX - 1),
             (3, 340, 341), (2, 10, 1000), (12345, 0, 97), (1 << 63, 3, (1 << 61) - 1), (7, 1, 2)]
    for k, (x, y, z) in enumerate(edges):
        a[k], b[k], c[k] = x, y, z
    return a, b, c


def test_modpow_vs_oracle():
    a, b, c = _operands(20000, seed=21)
    got = sv.modpow(a, b, c)
    assert np.array_equal(got, oracle.modpow_batch(a, b, c))
    assert int(got[0]) == U64MAX and int(got[1]) == 0 and int(got[5]) == 56


def test_modpow_device_pointers():
    import torch
    a, b, c = _operands(4096, seed=22)
    t = [torch.from_numpy(x.view(np.int64)).cuda() for x in (a, b, c)]
    out = torch.zeros(4096, dtype=torch.int64, device="cuda")
    sv.modpow(*t, out=out)
    assert np.array_equal(out.cpu().numpy().view(np.uint64), oracle.modpow_batch(a, b, c))


@pytest.mark.parametrize("iterations", [1, 3, 8])
def test_fermat_vs_oracle(iterations):
    small = np.arange(0, 20000, dtype=np.uint64)
    big = inputs.u64_stream(4000, seed=30 + iterations) | np.uint64(1)
    carm = np.array([561, 1105, 1729, 2465, 2821, 6601, 8911, 41041, 825265, 321197185],
                    dtype=np.uint64)
    p = np.concatenate([small, big, carm])
    draws = inputs.u64_stream(p.size * iterations, seed=40 + iterations)
    got = sv.fermat(p, draws, iterations)
    assert np.array_equal(got, oracle.fermat_batch(p, draws, iterations))
    assert got[1] == 0 and got[0] == 0 and got[2] == 1


def test_fermat_iterations_zero_rejected():
    with pytest.raises(sv.SieveError):
        sv.fermat([7], [1], 0)


def test_is_prime_vs_trial_division_and_sieve():
    n = np.arange(0, 100000, dtype=np.uint64)
    got = sv.is_prime(n)
    assert got.tolist() == [int(is_prime_td(int(x))) for x in n]
    lo, hi = 10**12 - 1000, 10**12 + 10**6
    win = np.arange(lo, hi, dtype=np.uint64)
    expect = np.zeros(win.size, dtype=np.uint8)
    expect[(oracle.primes(lo, hi) - np.uint64(lo)).astype(np.int64)] = 1
    assert np.array_equal(sv.is_prime(win), expect)


def test_is_prime_64bit_pins():
    # 2^61-1 (Mersenne prime), 2^64-59 (largest 64-bit prime), and composites
    # that fool small-base tests: 3215031751 = 151*751*28351 (strong pseudoprime
    # to bases 2, 3, 5, 7), Carmichael numbers, products of two large primes
    pr = [(1 << 61) - 1, (1 << 64) - 59]
    co = [3215031751, 151 * 751 * 28351, 561, 41041, ((1 << 31) - 1) * ((1 << 31) - 19),
          4294967291 * 4294967279]
    assert 3215031751 == 151 * 751 * 28351
    got = sv.is_prime(np.array(pr + co, dtype=np.uint64))
    assert got.tolist() == [1] * len(pr) + [0] * len(co)
    r = inputs.u64_stream(3000, seed=50) | np.uint64(1)
    assert sv.is_prime(r).tolist() == [int(is_prime_mr(int(x))) for x in r]


def test_is_prime_verifies_config4_subwindow_list():
    """The verifier role: every element of a config-4 sub-window list is prime
    and every odd non-member is not."""
    s0 = inputs.config4_subwindows()[0][0]
    lst, c = sv.primes(s0, s0 + 10**6)
    assert sv.is_prime(lst).all()
    odd = np.arange(s0 | 1, s0 + 10**6, 2, dtype=np.uint64)
    non = np.setdiff1d(odd, lst)
    assert not sv.is_prime(non).any()
