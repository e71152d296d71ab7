"""Step A2 (K1, base primes) on the GPU against the oracle: the odd primes
<= r ascending, their count, and their Barrett reciprocals floor((2^64-1)/p)
(the definition, in Python integers).  r spans the special cases of the
kernel: below/at the pattern primes (3..31) and the mini-sieve primes
(37..61), squares of small primes, slice edges (a slice is 8192 odd numbers:
n = 16385, 32769, ...), the configs' bounds and the 2^24 cap."""
import numpy as np
import pytest
import torch

import oracle
import paper_1205_4883_b200 as sv
from paper_1205_4883_b200 import dist as D

pytestmark = pytest.mark.gpu

R_VALUES = [0, 1, 2, 3, 4, 5, 8, 9, 10, 24, 25, 30, 31, 32, 36, 37, 60, 61, 62, 120, 121,
            960, 961, 1369, 3720, 3721, 16383, 16385, 16387, 32767, 32769, 32771, 35355,
            100000, 1004987, 3162277, 4096 * 4096 - 1, 1 << 24]


@pytest.fixture(scope="module")
def dev():
    sv.set_device(0)
    return torch.device("cuda", 0)


def _run(r, dev):
    base = D.alloc_base(sv.base_capacity(r), dev)
    base.packed.fill_(-1)  # stale contents must not leak through
    with torch.cuda.stream(torch.cuda.current_stream()):
        sv.set_stream(torch.cuda.current_stream())
        sv.base_primes_async(r, base.primes, base.recips, base.nbase)
        torch.cuda.synchronize()
        sv.set_stream(None)
    n = int(base.nbase.item())
    return (base.primes[:n].cpu().numpy().astype(np.int64),
            base.recips[:n].cpu().numpy().view(np.uint64))


@pytest.mark.parametrize("r", R_VALUES)
def test_base_primes_match_oracle(dev, r):
    got, rec = _run(r, dev)
    want = oracle.base_primes(r)
    want = want[want > 2].astype(np.int64)
    assert got.size == want.size, (r, got.size, want.size)
    assert np.array_equal(got, want), r
    # Barrett reciprocals: the definition, exactly (sampled for the big r)
    idx = np.arange(got.size) if got.size <= 4096 else np.random.default_rng(r).choice(got.size, 4096)
    for i in idx:
        assert int(rec[i]) == ((1 << 64) - 1) // int(got[i]), (r, int(got[i]))


def test_base_primes_back_to_back_epochs(dev):
    """Alternating sizes reuse the look-back flags across launches (epoch tags)."""
    for r in [10**6, 10**4, 3 * 10**6, 10**5, 10**6]:
        got, _ = _run(r, dev)
        want = oracle.base_primes(r)
        assert np.array_equal(got, want[want > 2].astype(np.int64)), r


@pytest.mark.parametrize("lo,hi", [(2, 10**7 + 1), (0, 10), (2, 3), (10**10 - 10**8, 10**10 + 1),
                                   (10**12, 10**12 + 10**9), (2**48 - 3 * 10**6, 2**48),
                                   (3 * 10**13, 3 * 10**13 + 2 * 10**8 + 7)])
def test_fused_base_launch(dev, lo, hi):
    """sieve_stats_base_async: A2 inside the sieve launch (or K1 first when a
    CTA's slice would not fit) -- the base-prime buffers it fills and the
    stats, against the oracle."""
    r = D.isqrt(hi - 1) if hi >= 2 else 0
    base = D.alloc_base(sv.base_capacity(r), dev)
    base.packed.fill_(-1)
    res = torch.zeros(2, dtype=torch.int64, device=dev)
    sv.set_stream(torch.cuda.current_stream())
    try:
        for _ in range(2):  # the grid barrier counter must be back at 0 for the second launch
            sv.stats_base_async(lo, hi, base.primes, base.recips, base.nbase, res)
            torch.cuda.synchronize()
            got = [int(x) & ((1 << 64) - 1) for x in res.cpu().tolist()]
            assert tuple(got) == oracle.stats(lo, hi), (lo, hi)
    finally:
        sv.set_stream(None)
    want = oracle.base_primes(r)
    want = want[want > 2].astype(np.int64)
    n = int(base.nbase.item())
    if hi - lo >= 2:  # an empty odd range launches no sieve: K1 fills the buffers
        assert n == want.size
        assert np.array_equal(base.primes[:n].cpu().numpy().astype(np.int64), want)
        rec = base.recips[:n].cpu().numpy().view(np.uint64)
        for i in np.random.default_rng(7).choice(n, min(n, 2048), replace=False) if n else []:
            assert int(rec[i]) == ((1 << 64) - 1) // int(want[i])
