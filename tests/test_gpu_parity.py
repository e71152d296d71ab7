"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle and pins.

Every comparison is bit-exact (integer work: counts, sums mod 2^64, bitmap
words, prime lists).  Inputs are seeded (inputs/), sized so the oracle
finishes in seconds while spanning several segments and a ragged tail; the
full BASELINE configs are checked against pinned values (tests/golden/) and
on oracle-computable samples.
"""
import math

import numpy as np
import pytest

import inputs
import oracle
import paper_1205_4883_b200 as sv
from paper_1205_4883_b200.dist import block_of
from golden_io import config3_blocks, config5_oracle, kv, subwindows
from independent import is_prime_td

pytestmark = pytest.mark.gpu
PINS = kv("config_pins.txt")
MASK64 = (1 << 64) - 1


@pytest.fixture(autouse=True)
def _defaults():
    sv.set_options()
    yield
    sv.set_options()


def _fnv(a):
    return oracle.fnv1a64(np.ascontiguousarray(a))


# ---------------------------------------------------------------- config 1
def test_config1_count_sum_bitmap_list():
    lo, hi = inputs.CONFIG1
    assert sv.count(lo, hi) == int(PINS["config1.count"])
    assert sv.stats(lo, hi) == (int(PINS["config1.count"]), int(PINS["config1.sum"]))
    bm, c = sv.bitmap(lo, hi)
    assert c == int(PINS["config1.count"])
    assert bm.size == int(PINS["config1.words"])
    assert _fnv(bm) == int(PINS["config1.fnv"], 16)
    obm, oc, os_ = oracle.bitmap(lo, hi)
    assert np.array_equal(bm, obm)
    lst, c2 = sv.primes(lo, hi)
    assert c2 == oc
    assert np.array_equal(lst, oracle.primes(lo, hi))
    assert int(lst.sum(dtype=np.uint64)) == os_


# ------------------------------------------------------- tiny / edge cases
def test_all_tiny_intervals_exhaustive():
    isp = [is_prime_td(n) for n in range(257)]
    los, his = [], []
    for lo in range(257):
        for hi in range(lo, 257):
            los.append(lo)
            his.append(hi)
    c, s = sv.batch(los, his)
    for k, (lo, hi) in enumerate(zip(los, his)):
        ps = [n for n in range(lo, hi) if isp[n]]
        assert (int(c[k]), int(s[k])) == (len(ps), sum(ps)), (lo, hi)


def test_tiny_intervals_single_calls_and_bitmaps():
    for lo in range(0, 70):
        for hi in (lo, lo + 1, lo + 2, lo + 63, lo + 64, lo + 65, lo + 200):
            assert sv.stats(lo, hi) == oracle.stats(lo, hi, 1), (lo, hi)
            bm, c = sv.bitmap(lo, hi)
            obm, oc, _ = oracle.bitmap(lo, hi, 1)
            assert c == oc
            assert np.array_equal(bm[:obm.size], obm), (lo, hi)
            lst, c3 = sv.primes(lo, hi)
            assert c3 == oc and lst[:c3].tolist() == oracle.primes(lo, hi, threads=1).tolist()


def test_errors():
    with pytest.raises(sv.SieveError):
        sv.count(10, 5)
    with pytest.raises(sv.SieveError):
        sv.count(0, (1 << 48) + 1)
    assert sv.count(7, 7) == 0


def test_p_squared_and_wheel_boundaries():
    ps = [p for p in range(3, 1200) if is_prime_td(p)]
    los = [max(0, p * p - 3) for p in ps] + list(range(0, 140))
    his = [p * p + 4 for p in ps] + [x + 3 for x in range(0, 140)]
    c, s = sv.batch(los, his)
    oc, os_ = oracle.batch(los, his, threads=None)
    assert np.array_equal(c, oc) and np.array_equal(s, os_)


# ------------------------------------------------ random seeded intervals
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random_intervals_stats(seed):
    iv = inputs.random_intervals(40, seed=seed, lo_max=10**13, width_max=10**6)
    for lo, hi in iv[:10]:
        assert sv.stats(lo, hi) == oracle.stats(lo, hi), (lo, hi)
    lo = np.array([a for a, _ in iv], dtype=np.uint64)
    hi = np.array([b for _, b in iv], dtype=np.uint64)
    c, s = sv.batch(lo, hi)
    oc, os_ = oracle.batch(lo, hi)
    assert np.array_equal(c, oc) and np.array_equal(s, os_)


def test_random_intervals_10k_batch_and_single_calls():
    """SURVEY.md 8(c) random parity: 10^4 seeded intervals, lo uniform in
    [0, 10^13], width uniform in [0, 10^6] (empty ones included), through
    sieve_batch, element-wise against oracle.batch; 500 of them also through
    the single-call path (one fused launch each)."""
    iv = inputs.random_intervals(10**4, seed=2024, lo_max=10**13, width_max=10**6)
    lo = np.array([a for a, _ in iv], dtype=np.uint64)
    hi = np.array([b for _, b in iv], dtype=np.uint64)
    c, s = sv.batch(lo, hi)
    oc, os_ = oracle.batch(lo, hi)
    bad = np.nonzero((c != oc) | (s != os_))[0]
    assert bad.size == 0, [(int(lo[i]), int(hi[i])) for i in bad[:5]]
    for k in range(0, 10**4, 20):
        assert sv.stats(int(lo[k]), int(hi[k])) == (int(oc[k]), int(os_[k])), (int(lo[k]), int(hi[k]))


@pytest.mark.parametrize("seg_kb", [32, 64, 128, 192])
@pytest.mark.parametrize("wheel", [11, 17, 23, 31, 41, 47])
def test_bitmap_multi_segment_ragged(seg_kb, wheel):
    if seg_kb == 192 and wheel == 47:
        pytest.skip("192 KiB + 25 KiB of wheel tables exceed shared memory")
    sv.set_options(segment_kb=seg_kb, wheel=wheel)
    for lo, hi in [(0, 3 * 10**7 + 17), (10**12 + 3, 10**12 + 2 * 10**7 + 1), (999_999_999_989, 1_000_040_000_000)]:
        bm, c = sv.bitmap(lo, hi)
        obm, oc, os_ = oracle.bitmap(lo, hi)
        assert c == oc
        assert np.array_equal(bm, obm), (lo, hi, seg_kb, wheel)
        assert sv.stats(lo, hi) == (oc, os_)


@pytest.mark.parametrize("threads", [256, 512, 768, 1024])
def test_thread_and_occupancy_invariance(threads):
    sv.set_options(threads=threads, segment_kb=64, ctas_per_sm=2)
    lo, hi = 10**11, 10**11 + 5 * 10**7 + 3
    assert sv.stats(lo, hi) == oracle.stats(lo, hi)
    # the write-back and list paths at every thread count (in-register
    # transpose: 2 lanes per block, tail lanes duplicating the last block)
    lo, hi = 10**11 + 7, 10**11 + 2 * 10**7 + 5
    obm, oc, _ = oracle.bitmap(lo, hi)
    bm, c = sv.bitmap(lo, hi)
    assert c == oc and np.array_equal(bm, obm)
    lst, c = sv.primes(lo, hi)
    assert c == oc and np.array_equal(lst, oracle.primes(lo, hi))


def test_primes_list_truncation_and_device_out():
    torch = pytest.importorskip("torch")
    lo, hi = 10**9, 10**9 + 10**7
    full = oracle.primes(lo, hi)
    lst, c = sv.primes(lo, hi, cap=1000)
    assert c == full.size and lst.tolist() == full[:1000].tolist()
    _, c0 = sv.primes(lo, hi, cap=0)
    assert c0 == full.size
    d = torch.zeros(full.size, dtype=torch.int64, device="cuda")
    _, c1 = sv.primes(lo, hi, out=d)
    assert c1 == full.size
    assert np.array_equal(d.cpu().numpy().view(np.uint64), full)
    # an output 8 bytes past a 16-byte boundary (the emission pairs primes
    # into 16-byte stores once aligned)
    d2 = torch.zeros(full.size + 1, dtype=torch.int64, device="cuda")
    _, c2 = sv.primes(lo, hi, cap=full.size, out=d2[1:])
    assert c2 == full.size
    assert np.array_equal(d2[1:].cpu().numpy().view(np.uint64), full) and int(d2[0]) == 0
    w = sv.bitmap_words(lo, hi)
    db = torch.zeros(w, dtype=torch.int32, device="cuda")
    _, cb = sv.bitmap(lo, hi, out=db)
    obm, oc, _ = oracle.bitmap(lo, hi)
    assert cb == oc and np.array_equal(db.cpu().numpy().view(np.uint32), obm)


@pytest.mark.parametrize("seg_kb,threads", [(8, 1024), (16, 1024), (16, 256), (32, 512), (208, 1024)])
def test_list_staged_emission_edges(seg_kb, threads):
    """A8 staged emission (kernels.cu list_emit, SIEVE_LIST_STAGE): warps whose
    word range is shorter than half a pass (direct only), one partial staged
    pass, many passes; ranges too dense for the staging room (direct
    fallback pass by pass), ranges where dense and sparse passes mix, and
    config 4's density; the list cut inside a staged pass, with guard
    elements past the cap, at both 16-byte phases of the output."""
    torch = pytest.importorskip("torch")
    sv.set_options(segment_kb=seg_kb, threads=threads)
    for lo, hi in [(2, 4 * 10**6 + 1), (3 * 10**3, 10**6), (10**7 + 1, 10**7 + 3 * 10**6),
                   (10**12 + 11, 10**12 + 5 * 10**6)]:
        full = oracle.primes(lo, hi)
        for off in (0, 1):
            for cap in (full.size, full.size - 37, full.size // 2 + 1):
                d = torch.full((off + cap + 64,), -7, dtype=torch.int64, device="cuda")
                _, c = sv.primes(lo, hi, cap=cap, out=d[off:off + cap])
                h = d.cpu().numpy()
                assert c == full.size
                assert np.array_equal(h[off:off + cap].view(np.uint64), full[:cap]), (lo, hi, off, cap)
                assert (h[:off] == -7).all() and (h[off + cap:] == -7).all(), (lo, hi, off, cap)


@pytest.mark.parametrize("shift", [0, 1, 2, 3])
def test_bitmap_bulk_copy_edges(shift):
    """A7 by TMA bulk copy (csrc/kernels.cu epilogue<kBitmap>): device outputs
    at 4-byte offsets 0..3 words past a 16-byte boundary (0: the bulk copy;
    else the 32-bit store path), ranges whose word count ends 0..3 words past
    a 16-byte multiple (the last < 4 words go by plain stores) and spanning
    several segments, and guard words before and after the output that must
    stay untouched."""
    torch = pytest.importorskip("torch")
    sv.set_options(segment_kb=16)
    try:
        for k, lo in enumerate([10**9 + 1, 3, 10**12 + 7]):
            for tail in range(4):
                w = 4 * (997 + 13 * k) + tail + 32 * 4096   # several 16 KiB segments
                hi = lo + 64 * w - (5 if lo % 2 else 6)     # last word partially valid
                assert sv.bitmap_words(lo, hi) == w
                buf = torch.full((w + 8,), -1, dtype=torch.int32, device="cuda")
                out = buf[shift: shift + w]
                _, cb = sv.bitmap(lo, hi, out=out)
                obm, oc, _ = oracle.bitmap(lo, hi)
                got = buf.cpu().numpy().view(np.uint32)
                assert cb == oc, (lo, tail, shift)
                assert np.array_equal(got[shift: shift + w], obm), (lo, tail, shift)
                assert (got[:shift] == 0xFFFFFFFF).all() and (got[shift + w:] == 0xFFFFFFFF).all()
    finally:
        sv.set_options()


def test_managed_memory_outputs():
    """Managed (unified) memory counts as device memory at the ABI
    (runtime.cu is_device_ptr): the kernels write it directly -- the bitmap
    by the TMA bulk copy, the list by its 16-byte stores -- and the host
    reads it after the call."""
    import ctypes
    torch = pytest.importorskip("torch")
    torch.cuda.init()
    rt = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so.12")
    lo, hi = 10**11 + 1, 10**11 + 3 * 10**6 + 2
    w = sv.bitmap_words(lo, hi)
    full = oracle.primes(lo, hi)
    ptrs = []
    try:
        for nbytes in (4 * w, 8 * full.size):
            p = ctypes.c_void_p()
            assert rt.cudaMallocManaged(ctypes.byref(p), ctypes.c_size_t(nbytes), 1) == 0
            ptrs.append(p.value)
        L = sv.lib()
        cb = L.sieve_bitmap(lo, hi, ptrs[0])
        cl = L.sieve_primes(lo, hi, ptrs[1], full.size)
        assert rt.cudaDeviceSynchronize() == 0
        obm, oc, _ = oracle.bitmap(lo, hi)
        got_bm = np.ctypeslib.as_array(ctypes.cast(ptrs[0], ctypes.POINTER(ctypes.c_uint32)), (w,)).copy()
        got_l = np.ctypeslib.as_array(ctypes.cast(ptrs[1], ctypes.POINTER(ctypes.c_uint64)), (full.size,)).copy()
        assert cb == oc and np.array_equal(got_bm, obm)
        assert cl == full.size and np.array_equal(got_l, full)
    finally:
        for p in ptrs:
            rt.cudaFree(ctypes.c_void_p(p))


def test_repeat_determinism():
    lo, hi = 2, 2 * 10**8 + 1
    a = [sv.stats(lo, hi) for _ in range(3)]
    assert a[0] == a[1] == a[2] == oracle.stats(lo, hi)


# ---------------------------------------------------------------- config 2
@pytest.mark.parametrize("seg_kb", [32, 64, 128, 192])
def test_config2_bitmap_hash_every_segment_size(seg_kb):
    sv.set_options(segment_kb=seg_kb)
    lo, hi = inputs.CONFIG2
    bm, c = sv.bitmap(lo, hi)
    assert c == int(PINS["config2.count"])
    assert bm.size == int(PINS["config2.words"])
    assert _fnv(bm) == int(PINS["config2.fnv"], 16)


def test_config2_vs_oracle_bitmap():
    lo, hi = inputs.CONFIG2
    bm, c = sv.bitmap(lo, hi)
    obm, oc, os_ = oracle.bitmap(lo, hi)
    assert c == oc and np.array_equal(bm, obm)
    assert sv.stats(lo, hi) == (oc, os_) == (int(PINS["config2.count"]), int(PINS["config2.sum"]))


# ---------------------------------------------------------------- config 3
def test_config3_count_sum_and_blocks():
    lo, hi = inputs.CONFIG3
    assert sv.stats(lo, hi) == (int(PINS["config3.count"]), int(PINS["config3.sum"]))
    # the G-block split (reading R10): blocks add up, whatever G
    for G in (2, 4, 8):
        tot_c, tot_s = 0, 0
        for g in range(G):
            a, b = block_of(lo, hi, g, G)
            c, s = sv.stats(a, b)
            tot_c += c
            tot_s = (tot_s + s) & MASK64
        assert (tot_c, tot_s) == (int(PINS["config3.count"]), int(PINS["config3.sum"]))
    # the cost-weighted split (dist.block_of split="cost") adds up as well
    for G in (2, 8):
        tot_c, tot_s = 0, 0
        for g in range(G):
            c, s = sv.stats(*block_of(lo, hi, g, G, "cost"))
            tot_c += c
            tot_s = (tot_s + s) & MASK64
        assert (tot_c, tot_s) == (int(PINS["config3.count"]), int(PINS["config3.sum"]))
    # every block of G = 2, 4, 8 against tests/golden/config3_blocks.txt
    # (reproduced by the oracle in test_oracle_golden.py)
    for G, g, a, b, c, s in config3_blocks():
        assert block_of(lo, hi, g, G) == (a, b)
        assert sv.stats(a, b) == (c, s), (G, g)


# ---------------------------------------------------------------- config 4
def test_config4_count_sum_and_subwindows():
    lo, hi = inputs.CONFIG4
    for seg_kb in (32, 192):
        sv.set_options(segment_kb=seg_kb)
        assert sv.stats(lo, hi) == (int(PINS["config4.count"]), int(PINS["config4.sum"]))
    sv.set_options()
    for (s, c, sm, h) in subwindows():
        lst, cnt = sv.primes(s, s + 10**7)
        assert cnt == c
        assert int(lst.sum(dtype=np.uint64)) == sm
        assert oracle.fnv1a64(lst.astype("<u8")) == h
    s0 = subwindows()[0][0]
    lst, _ = sv.primes(s0, s0 + 10**7)
    assert np.array_equal(lst, oracle.primes(s0, s0 + 10**7))


# ---------------------------------------------------------------- config 5
def test_config5_batch_digest_and_samples():
    lo, hi = inputs.config5_intervals()
    c, s = sv.batch(lo, hi)
    inter = np.empty(2 * c.size, dtype="<u8")
    inter[0::2] = c
    inter[1::2] = s
    assert int(c.sum()) == int(PINS["config5.count_total"])
    assert int(s.sum(dtype=np.uint64)) == int(PINS["config5.sum_total"])
    assert oracle.fnv1a64(inter) == int(PINS["config5.digest"], 16)
    # every interval element-wise against the oracle's values
    # (tests/golden/config5_oracle.txt, written by tools/regen_golden.py)
    flo, fhi, fc, fs = config5_oracle()
    assert np.array_equal(lo, flo) and np.array_equal(hi, fhi)
    assert np.array_equal(c, fc) and np.array_equal(s, fs)
    idx = np.array([0, 1, 2, 3, 4095] + list(range(7, 4096, 409)))
    oc, os_ = oracle.batch(lo[idx], hi[idx])
    assert np.array_equal(c[idx], oc) and np.array_equal(s[idx], os_)


# ------------------------------------------------- step A5: bucket path
@pytest.mark.parametrize("seg_kb", [4, 8, 32])
@pytest.mark.parametrize("buckets", [0, 1])
def test_bucket_path_vs_oracle(seg_kb, buckets):
    """Large primes (p > S) through per-segment buckets (buckets=1) and
    through per-segment Barrett first hits (buckets=0) agree with the oracle:
    ranges from 2 (p^2 inside the run: entries parked ahead), windows at
    10^12 (p up to 10^6 > 30 S at 4 KiB: the ring clamps at 32), ragged
    ends, and bitmap/list outputs."""
    sv.set_options(segment_kb=seg_kb, buckets=buckets)
    assert sv.get_options()["buckets"] == buckets
    cases = [(2, 3 * 10**8), (10**12 - 7, 10**12 + 2 * 10**7 + 3),
             (999_999_999_989, 1_000_000_031_000)]
    cases += inputs.random_intervals(4, seed=20 + seg_kb, lo_max=10**12, width_max=10**7)
    for lo, hi in cases:
        assert sv.stats(lo, hi) == oracle.stats(lo, hi), (lo, hi)
    lo, hi = 10**12 - 7, 10**12 + 3 * 10**6 + 3
    bm, c = sv.bitmap(lo, hi)
    obm, oc, _ = oracle.bitmap(lo, hi)
    assert c == oc and np.array_equal(bm, obm)
    lst, c2 = sv.primes(lo, hi)
    assert c2 == oc and np.array_equal(lst, oracle.primes(lo, hi))


def test_bucket_path_config4_full_window():
    """Config 4 with the bucket path carrying 71% of the base primes (32 KiB
    segments) and with the default segment, against the pinned values."""
    lo, hi = inputs.CONFIG4
    for seg_kb, buckets in ((32, 1), (32, 0), (64, 1)):
        sv.set_options(segment_kb=seg_kb, buckets=buckets)
        assert sv.stats(lo, hi) == (int(PINS["config4.count"]), int(PINS["config4.sum"]))


def test_config4_full_list_on_device_subwindows():
    """Config 4 at full size, as the benchmark runs it: the whole prime list
    of [10^12, 10^12 + 10^10) compacted into device memory (361,840,208 u64,
    2.9 GB), then the 16 seeded sub-windows (reading R12) sliced out of it by
    binary search and compared with their pinned count / sum / list FNV, and
    sub-window 0 element by element with the oracle.  Whole-list properties:
    count, sum mod 2^64, strictly ascending, all odd."""
    import torch
    lo, hi = inputs.CONFIG4
    n = int(PINS["config4.count"])
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    _, c = sv.primes(lo, hi, cap=n, out=out)
    assert c == n
    assert int(out.sum().item()) & MASK64 == int(PINS["config4.sum"])
    assert bool((out[1:] > out[:-1]).all()) and bool((out & 1).all())
    assert int(out[0]) >= lo and int(out[-1]) < hi
    for k, (s, cnt, sm, h) in enumerate(subwindows()):
        b = torch.tensor([s, s + 10**7], dtype=torch.int64, device="cuda")
        i0, i1 = torch.searchsorted(out, b).tolist()
        sl = out[i0:i1].cpu().numpy().astype(np.uint64)
        assert sl.size == cnt
        assert int(sl.sum(dtype=np.uint64)) == sm
        assert oracle.fnv1a64(sl.astype("<u8")) == h
        if k == 0:
            assert np.array_equal(sl, oracle.primes(s, s + 10**7))
    del out
    torch.cuda.empty_cache()


def test_f1_gather_single_rank_cuda_backend():
    """F1 on the CUDA backend at world size 1 (the box has one GPU; the
    N-rank gather logic runs under gloo in test_dist_gloo.py): the whole
    config-1 bitmap with its decomposable checksum, and the whole list."""
    import torch
    from paper_1205_4883_b200 import dist as D
    lo, hi = inputs.CONFIG1
    words, cs = D.gather_bitmap(lo, hi, device=torch.device("cuda"))
    w = words.cpu().numpy().view(np.uint32)
    assert _fnv(w) == int(PINS["config1.fnv"], 16)
    assert cs == D.bitmap_checksum(w)
    lst = D.gather_primes(lo, hi, device=torch.device("cuda")).cpu().numpy().view(np.uint64)
    assert lst.size == int(PINS["config1.count"]) and int(lst.sum(dtype=np.uint64)) == int(PINS["config1.sum"])


@pytest.mark.parametrize("seg_kb,buckets", [(208, 0), (16, 0), (16, 1)])
def test_top_of_range_2_48(seg_kb, buckets):
    """The largest allowed range end, hi = 2^48 (base primes up to 2^24,
    ~1.08 M of them; the widest K1 launch): count, sum and the list of a
    window just below it, against the oracle, with and without buckets."""
    sv.set_options(segment_kb=seg_kb, buckets=buckets)
    hi = 1 << 48
    lo = hi - 3 * 10**6 - 17
    assert sv.stats(lo, hi) == oracle.stats(lo, hi)
    lst, c = sv.primes(lo, hi)
    assert np.array_equal(lst, oracle.primes(lo, hi))
    bm, cb = sv.bitmap(lo, hi)
    obm, oc, _ = oracle.bitmap(lo, hi)
    assert cb == oc and np.array_equal(bm, obm)


@pytest.mark.parametrize("seg_kb,wheel", [(4, 11), (24, 31), (208, 31), (40, 47), (104, 17)])
def test_skip_residues_random_offsets(seg_kb, wheel):
    """The marking loops skip the hits that are multiples of 3 (and of 5 in
    long (C) walks): which hits those are depends on lo mod 3, lo mod 5, the
    segment offsets and p mod 3 / mod 5.  Random lo of every residue mod 30,
    odd segment sizes and several wheels, count + sum + bitmap vs the oracle."""
    sv.set_options(segment_kb=seg_kb, wheel=wheel)
    rng = np.random.default_rng(1000 + seg_kb + wheel)
    for k in range(12):
        lo = int(rng.integers(10**6, 2**40)) // 30 * 30 + (7 * k + seg_kb) % 30
        hi = lo + int(rng.integers(1, 3 * 10**6))
        assert sv.stats(lo, hi) == oracle.stats(lo, hi), (lo, hi)
        if k % 4 == 0:
            bm, c = sv.bitmap(lo, hi)
            obm, _, _ = oracle.bitmap(lo, hi)
            assert np.array_equal(bm[: obm.size], obm), (lo, hi)


def test_batch_edge_intervals():
    """Batch with duplicates, overlaps, empty and one-element intervals,
    intervals containing 2 / the wheel primes / 1, and a 2^48 top one."""
    iv = [(0, 0), (5, 5), (2, 3), (0, 2), (1, 60), (30, 50), (30, 50), (10**6, 10**6 + 1),
          (10**6 - 17, 10**6 + 10**5), (10**6, 10**6 + 10**5), (2**48 - 10**5, 2**48),
          (10**12 - 1, 10**12 + 1), (3, 4), (41, 48), (10**9 + 7, 10**9 + 8)]
    lo = np.array([a for a, _ in iv], dtype=np.uint64)
    hi = np.array([b for _, b in iv], dtype=np.uint64)
    c, s = sv.batch(lo, hi)
    for k, (a, b) in enumerate(iv):
        assert (int(c[k]), int(s[k])) == oracle.stats(a, b), (a, b)


@pytest.mark.parametrize("seg_kb", [16, 64, 208])
def test_batch_plain_pass_magnitudes(seg_kb):
    """The batch kernel's plain pass (primes with <= 8 hits per item) takes
    the 32-bit scaled first hit when every such prime exceeds 2^t, a < 2^(32+t)
    (default segment: everywhere below 2^48), else the 64-bit Barrett one
    (16 KiB segments above ~2^46): random intervals from 2^20 to 2^48 over
    both, with full and partial passes, vs the oracle."""
    sv.set_options(segment_kb=seg_kb)
    rng = np.random.default_rng(4242 + seg_kb)
    iv = []
    for e in range(20, 49, 2):
        for _ in range(3):
            b = int(rng.integers(1, 4 * 10**5))
            a = int(rng.integers(1 << (e - 1), (1 << e) - b)) if e < 48 else (1 << 48) - b
            iv.append((a, a + b))
    lo = np.array([a for a, _ in iv], dtype=np.uint64)
    hi = np.array([b for _, b in iv], dtype=np.uint64)
    c, s = sv.batch(lo, hi)
    for k, (a, b) in enumerate(iv):
        assert (int(c[k]), int(s[k])) == oracle.stats(a, b), (seg_kb, a, b)


@pytest.mark.parametrize("shift", [0, 1, 2, 3])
def test_plain_pass_list_alignment(shift):
    """Caller-owned base-prime buffers at any 4-byte offset (views shifted
    by 0-3 primes) through the base-buffer calls of the plain-pass kernels
    (r > S/8): count, sum and the bitmap of a 3*10^7 window at 10^12
    (r ~ 10^6) against the oracle."""
    torch = pytest.importorskip("torch")
    lo, hi = 10**12 + 17, 10**12 + 3 * 10**7 + 5
    r = int(np.sqrt(hi)) + 1
    cap = sv.base_capacity(r) + 4
    dev = torch.device("cuda")
    pbuf = torch.zeros(cap + 4, dtype=torch.int32, device=dev)
    rbuf = torch.zeros(cap + 4, dtype=torch.int64, device=dev)
    nb = torch.zeros(1, dtype=torch.int32, device=dev)
    primes, recips = pbuf[shift: shift + cap], rbuf[shift: shift + cap]
    res = torch.zeros(2, dtype=torch.int64, device=dev)
    out = torch.empty(sv.bitmap_words(lo, hi), dtype=torch.int32, device=dev)
    sv.set_stream(torch.cuda.current_stream())
    try:
        sv.base_primes_async(math.isqrt(hi - 1), primes, recips, nb)
        sv.stats_async(lo, hi, primes, recips, nb, res)
        torch.cuda.synchronize()
        got = tuple(int(x) & MASK64 for x in res.cpu().tolist())
        sv.bitmap_base_async(lo, hi, primes, recips, nb, out, res)
        torch.cuda.synchronize()
    finally:
        sv.set_stream(None)
    assert got == oracle.stats(lo, hi)
    obm, _, _ = oracle.bitmap(lo, hi)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), obm)


@pytest.mark.parametrize("lo,hi", [(2, 48), (40, 43), (1, 3), (29, 32), (2, 10**6), (999_983, 10**6 + 7)])
def test_small_ranges_fused_sync_paths(lo, hi):
    """Ranges around the wheel primes and tiny ranges through the synchronous
    APIs (fused base-prime launch) in all three modes."""
    assert sv.stats(lo, hi) == oracle.stats(lo, hi)
    bm, c = sv.bitmap(lo, hi)
    obm, oc, _ = oracle.bitmap(lo, hi)
    assert c == oc and np.array_equal(bm[: obm.size], obm)
    lst, n = sv.primes(lo, hi)
    assert np.array_equal(lst[:n], oracle.primes(lo, hi))


def test_lifecycle_shutdown_options_streams():
    """Library state across calls: shutdown and re-initialisation (scratch,
    tickets and grid-barrier counters re-created), option changes between
    fused launches (segment size, wheel, threads), a user stream, and the
    separate K1 path after the fused one -- every result against the oracle."""
    torch = pytest.importorskip("torch")
    want = oracle.stats(10**9, 10**9 + 10**7)
    assert sv.stats(10**9, 10**9 + 10**7) == want
    sv.shutdown()
    assert sv.stats(10**9, 10**9 + 10**7) == want
    for opts in [dict(segment_kb=32), dict(segment_kb=208, wheel=47 - 6), dict(threads=512),
                 dict(segment_kb=96, wheel=17), dict()]:
        sv.set_options(**opts)
        assert sv.stats(10**9, 10**9 + 10**7) == want, opts
        assert sv.stats(2, 10**6) == oracle.stats(2, 10**6), opts
    st = torch.cuda.Stream()
    sv.set_stream(st)
    try:
        assert sv.stats(10**9, 10**9 + 10**7) == want
        lst, n = sv.primes(10**9, 10**9 + 10**5)
        assert np.array_equal(lst[:n], oracle.primes(10**9, 10**9 + 10**5))
    finally:
        sv.set_stream(None)
    sv.shutdown()
    lst, n = sv.primes(2, 10**5)
    assert np.array_equal(lst[:n], oracle.primes(2, 10**5))


def test_batch_async_device_plan():
    """A10 planned on the device (sieve_batch_async): device-resident
    intervals, results element-wise against the oracle; an interval longer
    than the promised width_max gets the sentinel, the others are unaffected;
    repeated calls (the class histogram is re-zeroed by each plan)."""
    torch = pytest.importorskip("torch")
    iv = inputs.random_intervals(300, seed=77, lo_max=10**13, width_max=3 * 10**6) + [(0, 0), (2, 3), (0, 100)]
    lo = np.array([a for a, _ in iv], dtype=np.uint64)
    hi = np.array([b for _, b in iv], dtype=np.uint64)
    oc, os_ = oracle.batch(lo, hi)
    dlo = torch.from_numpy(lo.view(np.int64)).cuda()
    dhi = torch.from_numpy(hi.view(np.int64)).cuda()
    res = torch.zeros(2 * lo.size, dtype=torch.int64, device="cuda")
    sv.set_stream(torch.cuda.current_stream())
    try:
        for _ in range(3):
            res.fill_(-7)
            sv.batch_async(dlo, dhi, int(hi.max()), int((hi - lo).max()), res)
            torch.cuda.synchronize()
            got = res.cpu().numpy().view(np.uint64)
            assert np.array_equal(got[0::2], oc) and np.array_equal(got[1::2], os_)
        w = int(np.sort(hi - lo)[-2])  # the widest interval exceeds this promise
        sv.batch_async(dlo, dhi, int(hi.max()), w, res)
        torch.cuda.synchronize()
        got = res.cpu().numpy().view(np.uint64)
        big = int(np.argmax(hi - lo))
        assert got[2 * big] == got[2 * big + 1] == (1 << 64) - 1
        keep = np.arange(lo.size) != big
        assert np.array_equal(got[0::2][keep], oc[keep]) and np.array_equal(got[1::2][keep], os_[keep])
    finally:
        sv.set_stream(None)


@pytest.mark.parametrize("cfg", ["config3", "config4"])
def test_full_size_bitmaps_sampled_windows(cfg):
    """Bitmap mode at full size, in the launch configuration the bench modes
    time (sieve_bitmap_base_async: base primes, sieve and write-back in one
    launch, device output): config 3's 625 MB bitmap of [2, 10^10] and config
    4's 625 MB bitmap of [10^12, 10^12 + 10^10).  Properties over the whole
    bitmap (popcount = count minus the prime 2, padding bits zero) and 16
    seeded word-aligned windows of 10^6 integers element-wise against the
    oracle's bitmap of the same window (reading R5: word j of the call covers
    the odd integers o0 + 64 j ... o0 + 64 j + 62)."""
    torch = pytest.importorskip("torch")
    from paper_1205_4883_b200 import dist as D
    lo, hi = inputs.CONFIG3 if cfg == "config3" else inputs.CONFIG4
    want = (int(PINS[f"{cfg}.count"]), int(PINS[f"{cfg}.sum"]))
    r = D.isqrt(hi - 1)
    base = D.alloc_base(sv.base_capacity(r), torch.device("cuda"))
    words = sv.bitmap_words(lo, hi)
    out = torch.empty(words, dtype=torch.int32, device="cuda")
    res = torch.zeros(2, dtype=torch.int64, device="cuda")
    sv.set_stream(torch.cuda.current_stream())
    try:
        sv.bitmap_base_async(lo, hi, base.primes, base.recips, base.nbase, out, res)
        torch.cuda.synchronize()
    finally:
        sv.set_stream(None)
    assert tuple(int(x) & MASK64 for x in res.cpu().tolist()) == want
    x = out.to(torch.int64) & 0xFFFFFFFF  # SWAR popcount on the device
    x = x - ((x >> 1) & 0x55555555)
    x = (x & 0x33333333) + ((x >> 2) & 0x33333333)
    x = (x + (x >> 4)) & 0x0F0F0F0F
    pc = int(((x * 0x01010101) >> 24 & 0xFF).sum().item())
    del x
    w = out.cpu().numpy().view(np.uint32)
    assert pc + (1 if lo <= 2 < hi else 0) == want[0]
    B = hi // 2 - lo // 2
    if B % 32:
        assert int(w[-1]) >> (B % 32) == 0
    o0 = lo | 1
    g = inputs.SplitMix64(31 + len(cfg))
    for _ in range(16):
        w0 = g.next() % (words - 20000)
        w1 = w0 + 15625  # 10^6 integers
        a, b = o0 + 64 * w0, o0 + 64 * w1
        obm, _, _ = oracle.bitmap(a, b)
        assert obm.size == w1 - w0
        assert np.array_equal(w[w0:w1], obm), (cfg, w0)
    del out
    torch.cuda.empty_cache()


@pytest.mark.parametrize("count_only", [0, 1])
@pytest.mark.parametrize("seg_kb,threads", [(208, 1024), (64, 256), (32, 512), (8, 1024)])
def test_bitmap_async_sum_and_count_only(count_only, seg_kb, threads):
    """The fused write-back (in-register half-block transpose, count and
    prime sum from the rows and words it holds) against the oracle on ranges
    that span several segments, ragged tails, outputs at 4-byte offsets (no
    bulk copy) and every thread count: with the sum (result = (count, sum))
    and with the option bitmap_count_only (carry-save count, result[1] = 0)."""
    torch = pytest.importorskip("torch")
    from paper_1205_4883_b200 import dist as D
    sv.set_options(segment_kb=seg_kb, threads=threads, bitmap_count_only=count_only)
    g = inputs.SplitMix64(77 + seg_kb)
    ranges = [(0, 3 * 10**7 + 17), (10**12 + 3, 10**12 + 2 * 10**7 + 1), (2, 1025), (2, 64 * 1024 * 33 + 5)]
    ranges += [(a, a + 1 + g.next() % (3 * 10**6)) for a in (10**9 + g.next() % 10**9 for _ in range(4))]
    sv.set_stream(torch.cuda.current_stream())
    try:
        for lo, hi in ranges:
            r = D.isqrt(hi - 1)
            base = D.alloc_base(sv.base_capacity(r), torch.device("cuda"))
            words = sv.bitmap_words(lo, hi)
            obm, oc, os_ = oracle.bitmap(lo, hi)
            for shift in (0, 1):  # 16-byte aligned output (bulk copies) and a 4-byte offset
                buf = torch.zeros(words + 4, dtype=torch.int32, device="cuda")
                out = buf[shift:shift + words]
                res = torch.zeros(2, dtype=torch.int64, device="cuda")
                sv.bitmap_base_async(lo, hi, base.primes, base.recips, base.nbase, out, res)
                torch.cuda.synchronize()
                c, s = (int(x) & MASK64 for x in res.cpu().tolist())
                assert c == oc, (lo, hi, shift)
                assert s == (0 if count_only else os_), (lo, hi, shift)
                assert np.array_equal(out.cpu().numpy().view(np.uint32), obm), (lo, hi, shift)
                assert int(buf[:shift].abs().sum()) == 0 and int(buf[shift + words:].abs().sum()) == 0
    finally:
        sv.set_stream(None)
