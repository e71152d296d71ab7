#!/usr/bin/env python
"""Write the oracle-derived golden files (tests/golden/) -- TEST INFRASTRUCTURE.

This script imports ONLY ``oracle`` (the CPU reference, test infrastructure)
and ``inputs`` (the seeded workload definitions): no value it writes comes
from the CUDA path.  It writes

  tests/golden/config5_oracle.txt   per-interval (count, sum mod 2^64) of the
                                    4096 config-5 intervals (reading R11),
                                    computed by oracle.batch

and, with --check, recomputes every survey-supplied value in the other golden
files with the oracle and reports any disagreement (the same comparisons the
slow CPU tests in tests/test_oracle_golden.py make).

Usage:  python tools/regen_golden.py [--check]
"""
from __future__ import annotations

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import inputs  # noqa: E402
import oracle  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")


def fnv_pairs(c: np.ndarray, s: np.ndarray) -> int:
    """FNV-1a64 over the LE bytes of [count_0, sum_0, count_1, ...] (SURVEY.md C3 digest)."""
    inter = np.empty(2 * c.size, dtype="<u8")
    inter[0::2] = c
    inter[1::2] = s
    return oracle.fnv1a64(inter)


def write_config5() -> None:
    lo, hi = inputs.config5_intervals()
    t0 = time.time()
    c, s = oracle.batch(lo, hi)
    dt = time.time() - t0
    path = os.path.join(GOLDEN, "config5_oracle.txt")
    with open(path, "w") as f:
        f.write("# Config 5 (BASELINE.json configs[4]; reading R11: splitmix64 state 0) per-interval\n")
        f.write("# results, written by tools/regen_golden.py from oracle.batch ONLY (oracle/oracle.c,\n")
        f.write("# the byte-per-integer Eratosthenes of PAPER.md:131).  The aggregate of these lines is\n")
        f.write("# pinned to SURVEY.md 8(c) C3 (independent numba sieve): sum count = 715907351,\n")
        f.write("# sum of sums mod 2^64 = 5308460821128448155, FNV-1a64 of LE [count_i, sum_i] =\n")
        f.write(f"# 0x0dc0f9dd19ee6192 (this file: {int(c.sum())}, {int(s.sum(dtype=np.uint64))}, "
                f"{fnv_pairs(c, s):#018x}).\n")
        f.write("# Format: i lo hi count sum_mod_2^64\n")
        for i in range(c.size):
            f.write(f"{i} {int(lo[i])} {int(hi[i])} {int(c[i])} {int(s[i])}\n")
    print(f"wrote {path} ({c.size} intervals, oracle {dt:.1f} s)")


def check() -> int:
    from golden_io import config3_blocks, config5_oracle, kv, pairs, subwindows

    bad = 0

    def eq(name, got, want):
        nonlocal bad
        ok = got == want
        bad += not ok
        print(f"{'ok ' if ok else 'BAD'} {name}: oracle {got} vs golden {want}")

    k = kv("config_pins.txt")
    for x, pi in pairs("known_pi.txt"):
        eq(f"pi({x})", oracle.stats(0, x + 1)[0], pi)
    for x, sm in pairs("prime_sums.txt"):
        eq(f"sum<= {x}", oracle.stats(0, x + 1)[1], sm)
    lo, hi = inputs.CONFIG2
    bm, c, s = oracle.bitmap(lo, hi)
    eq("config2", (c, s, bm.size, oracle.fnv1a64(bm)),
       (int(k["config2.count"]), int(k["config2.sum"]), int(k["config2.words"]), int(k["config2.fnv"], 16)))
    for G, g, a, b, cnt, sm in config3_blocks():
        eq(f"config3 G={G} g={g}", oracle.stats(a, b), (cnt, sm))
    lo, hi = inputs.CONFIG4
    eq("config4", oracle.stats(lo, hi), (int(k["config4.count"]), int(k["config4.sum"])))
    eq("config4 nbase", int(oracle.base_primes(oracle.isqrt(hi - 1)).size), int(k["config4.nbase"]))
    for s0, cnt, sm, h in subwindows():
        lst = oracle.primes(s0, s0 + 10**7)
        eq(f"subwindow {s0}", (int(lst.size), int(lst.sum(dtype=np.uint64)), oracle.fnv1a64(lst.astype("<u8"))),
           (cnt, sm, h))
    lo5, hi5, c5, s5 = config5_oracle()
    c, s = oracle.batch(lo5, hi5)
    eq("config5 file", bool(np.array_equal(c, c5) and np.array_equal(s, s5)), True)
    eq("config5 aggregate", (int(c.sum()), int(s.sum(dtype=np.uint64)), fnv_pairs(c, s)),
       (int(k["config5.count_total"]), int(k["config5.sum_total"]), int(k["config5.digest"], 16)))
    print(f"{bad} disagreement(s)")
    return 1 if bad else 0


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--check", action="store_true")
    args = ap.parse_args()
    if args.check:
        return check()
    write_config5()
    return 0


if __name__ == "__main__":
    sys.exit(main())
