"""The oracle reproduces every stored expected value (-m "not gpu", slow).

Every value in tests/golden/ that the GPU parity tests compare against is
recomputed here by oracle/ alone, so that no stored value is trusted on the
survey's word only (SURVEY.md:60-62 "the builder must re-derive them with
the oracle").  The survey values came from methods independent of oracle/
(numpy / numba sieves, Lucy-Hedgehog differences, sympy spot checks:
SURVEY.md 8(c) C3), so an agreement here pins the oracle, and a stored value
the oracle does not reproduce fails the suite.

config5_oracle.txt is the one file written by a script (tools/regen_golden.py,
oracle/ + inputs/ only); its aggregate is pinned to the survey's digest.
"""
import numpy as np
import pytest

import inputs
import oracle
from golden_io import config3_blocks, config5_oracle, kv, subwindows

PINS = kv("config_pins.txt")
MASK64 = (1 << 64) - 1


def _pairs_digest(c, s):
    inter = np.empty(2 * c.size, dtype="<u8")
    inter[0::2] = c
    inter[1::2] = s
    return oracle.fnv1a64(inter)


def test_config2_bitmap_fnv_count_sum():
    # config 2 bitmap FNV-1a64 0xe4b98535dc2fea3d, 15,625,000 words
    lo, hi = inputs.CONFIG2
    bm, c, s = oracle.bitmap(lo, hi)
    assert (c, s) == (int(PINS["config2.count"]), int(PINS["config2.sum"]))
    assert bm.size == int(PINS["config2.words"])
    assert oracle.fnv1a64(bm) == int(PINS["config2.fnv"], 16)


@pytest.mark.slow
def test_config3_blocks_every_G():
    # SURVEY.md C3 per-GPU block values (Lucy differences) for G = 2, 4, 8;
    # the G = 8 blocks are computed once and the coarser blocks are unions of them
    blocks = config3_blocks()
    lo, hi = inputs.CONFIG3
    eight = {g: (a, b, c, s) for G, g, a, b, c, s in blocks if G == 8}
    got = {g: oracle.stats(a, b) for g, (a, b, _, _) in eight.items()}
    for g, (_, _, c, s) in eight.items():
        assert got[g] == (c, s), g
    for G, g, a, b, c, s in blocks:
        k = 8 // G
        assert (a, b) == (eight[g * k][0], eight[g * k + k - 1][1])
        tc = sum(got[g * k + i][0] for i in range(k))
        ts = sum(got[g * k + i][1] for i in range(k)) & MASK64
        assert (tc, ts) == (c, s), (G, g)
    assert (sum(v[0] for v in got.values()), sum(v[1] for v in got.values()) & MASK64) == \
        (int(PINS["config3.count"]), int(PINS["config3.sum"]))
    assert oracle.base_primes(oracle.isqrt(hi - 1)).size == int(PINS["config3.nbase"])


@pytest.mark.slow
def test_config4_full_window_count_sum():
    # Lucy difference + independent segmented sieve
    lo, hi = inputs.CONFIG4
    assert (lo, hi) == (int(PINS["config4.lo"]), int(PINS["config4.hi"]))
    assert oracle.stats(lo, hi) == (int(PINS["config4.count"]), int(PINS["config4.sum"]))
    # reading R3: base primes <= isqrt(hi - 1) = 1,004,987, not <= 10^6
    assert oracle.isqrt(hi - 1) == 1004987
    assert oracle.base_primes(1004987).size == int(PINS["config4.nbase"])


def test_config4_all_subwindows_lists():
    # SURVEY.md C3 (numba window sieve; sub-window 0 also by sympy.isprime):
    # all 16 sub-windows (reading R12), count, sum and FNV of the u64 list
    wins = inputs.config4_subwindows()
    sw = subwindows()
    assert [w[0] for w in wins] == [s[0] for s in sw]
    for (s0, s1), (start, c, sm, h) in zip(wins, sw):
        lst = oracle.primes(s0, s1)
        assert lst.size == c, start
        assert int(lst.sum(dtype=np.uint64)) == sm, start
        assert oracle.fnv1a64(lst.astype("<u8")) == h, start


@pytest.mark.slow
def test_config5_all_intervals_file_and_digest():
    # the per-interval file the GPU test compares with is exactly the oracle's
    # output, and its aggregate is the survey's
    lo, hi = inputs.config5_intervals()
    flo, fhi, fc, fs = config5_oracle()
    assert np.array_equal(lo, flo) and np.array_equal(hi, fhi)
    c, s = oracle.batch(lo, hi)
    assert np.array_equal(c, fc) and np.array_equal(s, fs)
    assert int(c.sum()) == int(PINS["config5.count_total"])
    assert int(s.sum(dtype=np.uint64)) == int(PINS["config5.sum_total"])
    assert _pairs_digest(c, s) == int(PINS["config5.digest"], 16)
    for i in (0, 1, 2, 3, 4095):
        v = PINS[f"config5.i{i}"]
        assert (int(c[i]), int(s[i])) == (int(v[2]), int(v[3])), i
    assert int(c.min()) == 3630 and int(c.max()) == 407836  # SURVEY.md C3 range


def test_config5_file_aggregate_matches_survey():
    # fast check of the committed file alone (no oracle run)
    _, _, c, s = config5_oracle()
    assert c.size == inputs.CONFIG5_N
    assert _pairs_digest(c, s) == int(PINS["config5.digest"], 16)
