"""Pin the CPU oracle to things other than itself (-m "not gpu").

Each test names what it pins against: trial division, the
pi values stated in BASELINE.json north_star, SPEC.md worked examples,
the Lucy-Hedgehog combinatorial count, deterministic Miller-Rabin, and
invariants that hold at any size.  A plausible oracle bug (a dropped base
prime, a wrong start index p^2 vs 2p, an off-by-one on hi, evens in the
bitmap, a non-wrapping sum) fails at least one of them.
"""
import numpy as np
import pytest

import inputs
import oracle
from golden_io import kv, pairs, spec_examples, subwindows
from independent import is_prime_mr, is_prime_td, lucy_interval, lucy_pi_sum, primes_td

MASK64 = (1 << 64) - 1


def test_isqrt_exact():
    for x in list(range(0, 2000)) + [2**48 - 1, 2**48, 10**12 + 10**10 - 1, (2**24) ** 2,
                                     (2**24) ** 2 - 1, 999999999999]:
        r = oracle.isqrt(x)
        assert r * r <= x < (r + 1) * (r + 1), x


def test_base_primes_vs_trial_division():
    # PAPER.md:29 definition, every n <= 10^5
    got = oracle.base_primes(10**5)
    exp = primes_td(0, 10**5 + 1)
    assert got.tolist() == exp
    assert oracle.base_primes(1).size == 0
    assert oracle.base_primes(2).tolist() == [2]


def test_list_vs_trial_division_all_n_le_1e5():
    # north_star: "checked against trial division on all n <= 10^5"
    got = oracle.primes(0, 10**5 + 1)
    assert got.tolist() == primes_td(0, 10**5 + 1)


@pytest.mark.parametrize("threads", [1, 3, 8])
def test_thread_count_invariance(threads):
    lo, hi = 123456789, 123456789 + 3 * (1 << 24) + 12345  # several chunks + ragged tail
    assert oracle.stats(lo, hi, threads) == oracle.stats(lo, hi, 1)
    bm1, _, _ = oracle.bitmap(lo, hi, 1)
    bmt, _, _ = oracle.bitmap(lo, hi, threads)
    assert np.array_equal(bm1, bmt)


def test_spec_worked_examples():
    for lo, hi, ps, cnt in spec_examples():
        got = oracle.primes(lo, hi)
        assert len(got) == cnt, (lo, hi)
        if ps is not None:
            assert got.tolist() == ps, (lo, hi)


def test_known_pi_values_upto_1e9():
    # BASELINE.json north_star: pi(10^6)=78498 ... pi(10^9)=50847534
    for x, pi in pairs("known_pi.txt"):
        if x > 10**9:
            continue
        assert oracle.stats(0, x + 1)[0] == pi, x


@pytest.mark.slow
def test_known_pi_1e10_and_sum():
    # BASELINE.json north_star pi(10^10)=455052511; sum pinned by Lucy
    c, s = oracle.stats(2, 10**10 + 1)
    assert c == 455052511
    assert (c, s) == lucy_pi_sum(10**10)


def test_prime_sums_vs_lucy():
    # golden sums are re-derived by Lucy (independent of oracle/), then the oracle must match
    for x, s in pairs("prime_sums.txt"):
        if x <= 10**8:
            assert lucy_pi_sum(x)[1] == s
            assert oracle.stats(0, x + 1)[1] == s, x
    assert oracle.stats(0, 10**9 + 1)[1] == 24739512092254535


def test_random_intervals_vs_lucy():
    for lo, hi in inputs.random_intervals(6, seed=7, lo_max=10**9, width_max=5 * 10**6):
        assert oracle.stats(lo, hi) == lucy_interval(lo, hi), (lo, hi)


def test_random_windows_vs_miller_rabin():
    # windows high up (10^12 .. 10^13) where trial division is too slow
    for lo, hi in inputs.random_intervals(4, seed=11, lo_max=10**13, width_max=3000):
        lo += 10**12
        hi += 10**12
        got = oracle.primes(lo, hi).tolist()
        exp = [n for n in range(lo, hi) if is_prime_mr(n)]
        assert got == exp, (lo, hi)


def test_brute_force_all_tiny_intervals():
    # every [lo, hi) with 0 <= lo <= hi <= 256 vs trial division
    isp = [is_prime_td(n) for n in range(257)]
    for lo in range(0, 257):
        for hi in range(lo, 257):
            c, s = oracle.stats(lo, hi, 1)
            ps = [n for n in range(lo, hi) if isp[n]]
            assert (c, s) == (len(ps), sum(ps)), (lo, hi)


def test_p_squared_boundaries():
    # around p^2 for every prime p <= 1000: the first composite each base prime owns
    for p in primes_td(2, 1001):
        lo, hi = p * p - 2, p * p + 3
        got = oracle.primes(max(lo, 0), hi).tolist()
        assert got == [n for n in range(max(lo, 0), hi) if is_prime_td(n)], p


def test_bitmap_convention_and_invariants():
    # reading R5: bit j <-> (lo|1) + 2j, 1 = prime, zero padding; popcount + [2 in range] = count
    for lo, hi in [(0, 1), (0, 3), (2, 3), (1, 200), (2, 10**5 + 1), (7, 7 + 64 * 5 + 17), (100, 101),
                   (10**6 - 100, 10**6 + 1)]:
        bm, c, s = oracle.bitmap(lo, hi)
        o0 = lo | 1
        B = hi // 2 - lo // 2
        assert bm.size == (B + 31) // 32
        bits = np.unpackbits(bm.view(np.uint8), bitorder="little")
        assert not bits[B:].any()
        odd_primes = [n for n in range(lo, hi) if n % 2 and is_prime_td(n)]
        assert [o0 + 2 * j for j in np.nonzero(bits[:B])[0]] == odd_primes
        assert int(bits.sum()) + (1 if lo <= 2 < hi else 0) == c


def test_config1_pins():
    k = kv("config_pins.txt")
    lo, hi = int(k["config1.lo"]), int(k["config1.hi"])
    bm, c, s = oracle.bitmap(lo, hi)
    assert c == int(k["config1.count"]) and s == int(k["config1.sum"])
    assert bm.size == int(k["config1.words"])
    assert oracle.fnv1a64(bm) == int(k["config1.fnv"], 16)
    assert [int(x) for x in bm[:3]] == [int(k[f"config1.word{i}"], 16) for i in range(3)]
    lst = oracle.primes(lo, hi)
    assert lst.size == c and int(lst.sum(dtype=np.uint64)) == s
    assert (c, s) == lucy_interval(lo, hi)


def test_fnv1a64_reference_vectors():
    # FNV-1a 64 published test vectors (Fowler/Noll/Vo): "" and "a"
    assert oracle.fnv1a64(np.frombuffer(b"", dtype=np.uint8)) == 0xcbf29ce484222325
    assert oracle.fnv1a64(np.frombuffer(b"a", dtype=np.uint8)) == 0xaf63dc4c8601ec8c
    assert oracle.fnv1a64(np.frombuffer(b"foobar", dtype=np.uint8)) == 0x85944171f73967e8


def test_truncated_list():
    full = oracle.primes(0, 1000)
    part = oracle.primes(0, 1000, cap=10)
    assert part.tolist() == full[:10].tolist()


def test_errors_and_empty():
    assert oracle.stats(5, 5) == (0, 0)
    with pytest.raises(ValueError):
        oracle.stats(10, 5)
    with pytest.raises(ValueError):
        oracle.stats(0, 2**48 + 1)


def test_config4_subwindow0_and_config5_intervals():
    sw = subwindows()
    wins = inputs.config4_subwindows()
    assert [w[0] for w in wins] == [s[0] for s in sw]
    s0, c0, sum0, h0 = sw[0]
    lst = oracle.primes(s0, s0 + 10**7)
    assert lst.size == c0
    assert int(lst.sum(dtype=np.uint64)) == sum0
    assert oracle.fnv1a64(lst.astype("<u8")) == h0
    k = kv("config_pins.txt")
    lo, hi = inputs.config5_intervals()
    for i in (0, 1, 2, 4095):
        v = k[f"config5.i{i}"]
        assert (int(lo[i]), int(hi[i])) == (int(v[0]), int(v[1]))
    c, s = oracle.batch(lo[[0, 1, 2, 3, 4095]], hi[[0, 1, 2, 3, 4095]])
    for j, i in enumerate((0, 1, 2, 3, 4095)):
        v = k[f"config5.i{i}"]
        assert (int(c[j]), int(s[j])) == (int(v[2]), int(v[3])), i
    # one interval also element-wise by Miller-Rabin (window of 10^4 inside interval 0)
    a = int(lo[0])
    got = oracle.primes(a, a + 10**4).tolist()
    assert got == [n for n in range(a, a + 10**4) if is_prime_mr(n)]
