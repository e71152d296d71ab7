"""Parsers for tests/golden/*.txt (each line carries its citation)."""
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _lines(name):
    with open(os.path.join(GOLDEN, name)) as f:
        for raw in f:
            line = raw.split("#", 1)[0].strip() if not raw.lstrip().startswith("#") else ""
            if line:
                yield line


def pairs(name):
    """'x y' lines -> list of (int, int)."""
    return [tuple(int(t, 0) for t in l.split()[:2]) for l in _lines(name)]


def kv(name):
    out = {}
    for l in _lines(name):
        k, *v = l.split()
        out[k] = v if len(v) > 1 else v[0]
    return out


def spec_examples():
    out = []
    for l in _lines("spec_examples.txt"):
        rng, exp = l.split("|")
        lo, hi = (int(t) for t in rng.split())
        exp = exp.strip()
        if exp.startswith("count="):
            out.append((lo, hi + 1, None, int(exp[6:])))
        else:
            ps = [int(t) for t in exp.split()]
            out.append((lo, hi + 1, ps, len(ps)))
    return out


def subwindows():
    out = []
    for l in _lines("config4_subwindows.txt"):
        s, c, sm, h = l.split()
        out.append((int(s), int(c), int(sm), int(h, 16)))
    return out


def config3_blocks():
    """tests/golden/config3_blocks.txt -> list of (G, g, lo, hi, count, sum)."""
    return [tuple(int(t) for t in l.split()) for l in _lines("config3_blocks.txt")]


def config5_oracle():
    """tests/golden/config5_oracle.txt (written by tools/regen_golden.py from
    oracle/ only) -> (lo, hi, count, sum) uint64 arrays in interval order."""
    import numpy as np

    rows = [l.split() for l in _lines("config5_oracle.txt")]
    assert [int(r[0]) for r in rows] == list(range(len(rows)))
    cols = [np.array([int(r[k]) for r in rows], dtype=np.uint64) for k in range(1, 5)]
    return tuple(cols)
