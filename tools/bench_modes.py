"""Secondary measurements (one JSON line each) for the non-headline configs:
config 1 (list), config 2 (bitmap to HBM, plus the write-back stage in
isolation), config 4 (interval count), config 5 (batch).  Device-resident
outputs, CUDA events on the library stream, L2 flushed between repetitions.
The headline number is bench.py (config 3)."""
import json
import math
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_1205_4883_b200 as sv  # noqa: E402
from paper_1205_4883_b200 import dist as D  # noqa: E402

HBM_PEAK = 6544.7  # GB/s, MEASURED_PEAKS.json hbm_gbs (copy, read+write)
try:
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                           "MEASURED_PEAKS.json")) as f:
        HBM_PEAK = json.load(f).get("hbm_gbs", HBM_PEAK)
except Exception:  # noqa: BLE001
    pass

dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(device=dev)
sv.set_stream(stream)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
REPS = int(os.environ.get("REPS", "10"))


def timed(fn, reps=REPS):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        with torch.cuda.stream(stream):
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts), min(ts)


def base_for(hi):
    r = math.isqrt(hi - 1)
    b = D.alloc_base(sv.base_capacity(r), dev)
    sv.base_primes_async(r, b.primes, b.recips, b.nbase)
    return r, b


RESULTS = []


def emit(d):
    RESULTS.append(d)
    print(json.dumps(d), flush=True)


def oracle_report(path):
    """SURVEY.md 8(d) D4 / BASELINE.md 5: the oracle on the host cores per
    config (T = all hardware threads; T = 1 for configs 1-2), next to the GPU
    numbers of this run, with nproc and the CPU model -> report.json."""
    import oracle
    import bench

    T = oracle.default_threads()

    def t(fn):
        t0 = time.perf_counter()
        out = fn()
        return time.perf_counter() - t0, out

    rep = {"host": {**bench.host_cpu(), "threads": T}, "gpu": RESULTS, "oracle": {}}
    o = rep["oracle"]
    lo, hi = inputs.CONFIG1
    for th in (T, 1):
        ds, _ = t(lambda: (oracle.stats(lo, hi, th), oracle.primes(lo, hi, threads=th),
                           oracle.bitmap(lo, hi, th)))
        o[f"config1_T{th}"] = {"s": ds, "what": "count+sum, list, bitmap of [2, 1e7+1)"}
    lo, hi = inputs.CONFIG2
    for th in (T, 1):
        ds, (bm, c, _) = t(lambda: oracle.bitmap(lo, hi, th))
        o[f"config2_T{th}"] = {"s": ds, "what": "bitmap + count + sum of [2, 1e9+1)",
                               "ok": c == 50847534 and oracle.fnv1a64(bm) == 0xe4b98535dc2fea3d}
    lo, hi = inputs.CONFIG3
    ds, r = t(lambda: oracle.stats(lo, hi, T))
    o[f"config3_T{T}"] = {"s": ds, "what": "count+sum of [2, 1e10+1)",
                          "ok": r == (455052511, 2220822432581729238)}
    lo, hi = inputs.CONFIG4
    ds, r = t(lambda: oracle.stats(lo, hi, T))
    o[f"config4_T{T}"] = {"s": ds, "what": "count+sum of the whole window [1e12, 1e12+1e10)",
                          "ok": r == (361840208, 13161149016643422504)}
    ds, _ = t(lambda: [oracle.primes(a, b, threads=T) for a, b in inputs.config4_subwindows()])
    o[f"config4_subwindows_T{T}"] = {"s": ds, "what": "the 16 sub-window lists (width 1e7)"}
    l5, h5 = inputs.config5_intervals()
    ds, (c5, _) = t(lambda: oracle.batch(l5, h5, T))
    o[f"config5_T{T}"] = {"s": ds, "what": "all 4096 intervals, count+sum", "ok": int(c5.sum()) == 715907351}
    with open(path, "w") as f:
        json.dump(rep, f, indent=1)
    print(json.dumps({"report": path, "oracle": o}), flush=True)


def config2(opts, lohi=None, tag=2):
    """Bitmap mode (A7) of config 2 -- or, with lohi = config 3's range, a
    625 MB bitmap far larger than the 126 MB L2, where HBM binds.  Times:
    the product call (base primes + sieve + bitmap in one launch,
    sieve_bitmap_base_async) and the write-back stage in isolation (diagnostic flag 1: wheel init +
    transpose + count + store, marking skipped)."""
    if isinstance(opts, int):
        opts = {"segment_kb": opts}
    sv.set_options(**opts)
    seg_kb = sv.get_options()
    lo, hi = lohi or inputs.CONFIG2
    r = math.isqrt(hi - 1)
    b = D.alloc_base(sv.base_capacity(r), dev)
    words = sv.bitmap_words(lo, hi)
    out = torch.empty(words, dtype=torch.int32, device=dev)
    res = torch.zeros(2, dtype=torch.int64, device=dev)
    want = {2: 50847534, 3: 455052511}[tag]
    med, mn = timed(lambda: sv.bitmap_base_async(lo, hi, b.primes, b.recips, b.nbase, out, res))
    ok = res.cpu().tolist()[0] == want
    sv.debug_set_flags(1)
    wmed, wmn = timed(lambda: sv.bitmap_base_async(lo, hi, b.primes, b.recips, b.nbase, out, res))
    sv.debug_set_flags(0)
    # the same calls returning the count only (option bitmap_count_only: no prime sum, the
    # configs' "bitmap + count"; sieve_bitmap's own path)
    sv.set_options(**{**sv.get_options(), "bitmap_count_only": 1})
    cmed, _ = timed(lambda: sv.bitmap_base_async(lo, hi, b.primes, b.recips, b.nbase, out, res))
    ok = ok and res.cpu().tolist()[0] == want
    sv.debug_set_flags(1)
    cwmed, _ = timed(lambda: sv.bitmap_base_async(lo, hi, b.primes, b.recips, b.nbase, out, res))
    sv.debug_set_flags(1 | 256)  # wheel init skipped too: transpose + count + bulk copy alone
    ctmed, _ = timed(lambda: sv.bitmap_base_async(lo, hi, b.primes, b.recips, b.nbase, out, res))
    sv.debug_set_flags(0)
    cmed_count = None
    if tag == 3:  # the same range in count mode: the bitmap's marginal cost over count + sum
        cres = torch.zeros(2, dtype=torch.int64, device=dev)
        cmed_count, _ = timed(lambda: sv.stats_base_async(lo, hi, b.primes, b.recips, b.nbase, cres))
    sv.set_options(**{**sv.get_options(), "bitmap_count_only": 0})
    byts = words * 4
    emit({"config": tag, "mode": "bitmap", "segment_kb": seg_kb, "ok": ok, "kernel_ms": med,
          "integers_per_s": (hi - lo) / (med / 1e3), "bitmap_bytes": byts,
          "bitmap_vs_l2": "larger than the 126 MB L2" if byts > 126e6 else "fits in L2",
          "hbm_gbs_end_to_end": byts / (med / 1e3) / 1e9,
          "hbm_frac_end_to_end": byts / (med / 1e3) / 1e9 / HBM_PEAK,
          "writeback_only_ms": wmed, "writeback_only_gbs": byts / (wmed / 1e3) / 1e9,
          "writeback_only_frac": byts / (wmed / 1e3) / 1e9 / HBM_PEAK,
          "count_only_kernel_ms": cmed, "count_only_hbm_frac_end_to_end": byts / (cmed / 1e3) / 1e9 / HBM_PEAK,
          "count_only_writeback_only_ms": cwmed,
          "count_only_writeback_only_frac": byts / (cwmed / 1e3) / 1e9 / HBM_PEAK,
          "transpose_copy_only_ms": ctmed, "transpose_copy_only_frac": byts / (ctmed / 1e3) / 1e9 / HBM_PEAK,
          "count_mode_ms": cmed_count,
          "marginal_vs_count_mode_frac": (byts / ((cmed - cmed_count) / 1e3) / 1e9 / HBM_PEAK)
          if cmed_count and cmed > cmed_count else None,
          "hbm_peak_gbs": HBM_PEAK, "peak_basis": "MEASURED_PEAKS.json hbm_gbs (copy)",
          "call": "sieve_bitmap_base_async (fused A2 + sieve + write-back, one launch)"})
    del out
    torch.cuda.empty_cache()
    sv.set_options()


def config1():
    lo, hi = inputs.CONFIG1
    n = 664579
    out = torch.empty(n, dtype=torch.int64, device=dev)

    def run():
        sv.primes(lo, hi, out=out)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(REPS):
        t0 = time.perf_counter()
        run()
        ts.append(time.perf_counter() - t0)
    med = statistics.median(ts)
    emit({"config": 1, "mode": "list (sieve_primes, device out, synchronous call)", "ms": med * 1e3,
          "integers_per_s": (hi - lo) / med, "list_bytes": n * 8,
          "list_gbs": n * 8 / med / 1e9})


def config4(seg_kb):
    sv.set_options(segment_kb=seg_kb)
    lo, hi = inputs.CONFIG4
    r, b = base_for(hi)
    res = torch.zeros(2, dtype=torch.int64, device=dev)
    med, mn = timed(lambda: sv.stats_async(lo, hi, b.primes, b.recips, b.nbase, res), reps=5)
    got = [D.i64_to_u64(x) for x in res.cpu().tolist()]
    emit({"config": 4, "mode": "count+sum", "segment_kb": seg_kb, "kernel_ms": med,
          "integers_per_s": (hi - lo) / (med / 1e3),
          "ok": got == [361840208, 13161149016643422504], **config4_frac(med, seg_kb)})
    sv.set_options()


def config4_list(seg_kb=0):
    """Config 4 prime list (361,840,208 u64 = 2.9 GB) compacted into device
    memory through sieve_primes (synchronous call: base primes, bitmap-mode
    sieve into scratch, segment scan, compaction, count read-back)."""
    if seg_kb:
        sv.set_options(segment_kb=seg_kb)
    lo, hi = inputs.CONFIG4
    n = 361840208
    out = torch.empty(n, dtype=torch.int64, device=dev)

    def run():
        return sv.primes(lo, hi, cap=n, out=out)[1]
    for _ in range(2):
        c = run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        with torch.cuda.stream(stream):
            flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        run()
        ts.append(time.perf_counter() - t0)
    med = statistics.median(ts)
    emit({"config": 4, "mode": "list (sieve_primes, device out, synchronous call)",
          "segment_kb": sv.get_options()["segment_kb"], "ms": med * 1e3, "ok": c == n,
          "integers_per_s": (hi - lo) / med, "list_bytes": n * 8, "list_gbs": n * 8 / med / 1e9,
          "list_hbm_frac": n * 8 / med / 1e9 / HBM_PEAK})
    del out
    torch.cuda.empty_cache()
    sv.set_options()


def f2():
    """SURVEY.md 8(f) F2 on the GPU: the deterministic Miller-Rabin verifier
    and Alg. 3 (one round) over the whole config-4 prime list, device-resident
    (361,840,208 candidates of ~40 bits)."""
    lo, hi = inputs.CONFIG4
    n = 361840208
    lst = torch.empty(n, dtype=torch.int64, device=dev)
    sv.primes(lo, hi, cap=n, out=lst)
    out = torch.empty(n, dtype=torch.uint8, device=dev)
    draws = torch.from_numpy(inputs.u64_stream(n, seed=7).view(np.int64)).to(dev)

    def t(fn):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        return statistics.median(ts)
    mr = t(lambda: sv.is_prime(lst, out=out))
    ok_mr = bool(out.all())
    fe = t(lambda: sv.fermat(lst, draws, 1, out=out))
    ok_fe = bool(out.all())
    emit({"config": "F2", "mode": "Miller-Rabin (12 bases) + Fermat (Alg. 3, 1 round) over the config-4 list",
          "candidates": n, "mr_ms": mr * 1e3, "mr_tests_per_s": n / mr, "mr_all_prime": ok_mr,
          "fermat_ms": fe * 1e3, "fermat_tests_per_s": n / fe, "fermat_all_pass": ok_fe})
    del lst, out, draws
    torch.cuda.empty_cache()


def marks_alg_interval(lo: int, hi: int, primes: np.ndarray, wheel: int) -> int:
    """M_alg of one interval (bench.algorithmic_marks, vectorised): odd
    multiples m of every prime wheel < p <= isqrt(hi-1), max(lo, p^2) <= m < hi."""
    if hi <= lo or hi < 10:
        return 0
    r = math.isqrt(hi - 1)
    p = primes[(primes > wheel) & (primes <= r)]
    a = np.maximum(np.int64(lo), p * p)
    m0 = (a + p - 1) // p * p
    m0 = np.where(m0 % 2 == 0, m0 + p, m0)
    ok = m0 < hi
    return int((((hi - 1 - m0[ok]) // (2 * p[ok])) + 1).sum())


def small_primes_np(r: int) -> np.ndarray:
    s = np.ones(r + 1, dtype=bool)
    s[:2] = False
    for q in range(2, math.isqrt(r) + 1):
        if s[q]:
            s[q * q::q] = False
    return np.nonzero(s)[0].astype(np.int64)


def config5():
    """Config 5 (4096 intervals): kernel-only on device-resident intervals
    (sieve_batch_async: K1 + the on-device plan + the batch sieve, CUDA
    events) and end to end through the host API (sieve_batch), with the
    shared-memory-atomic roofline fraction (M_alg at the build's wheel over
    all intervals / kernel time / (148 x R_atom x f))."""
    lo, hi = inputs.config5_intervals()
    total = int((hi - lo).sum())
    hi_max, width_max = int(hi.max()), int((hi - lo).max())
    dlo = torch.from_numpy(lo.view(np.int64)).to(dev)
    dhi = torch.from_numpy(hi.view(np.int64)).to(dev)
    res = torch.zeros(2 * lo.size, dtype=torch.int64, device=dev)
    med, mn = timed(lambda: sv.batch_async(dlo, dhi, hi_max, width_max, res))
    got = res.cpu().numpy().view(np.uint64)
    ok_k = int(got[0::2].sum()) == 715907351
    for _ in range(2):
        c, s = sv.batch(lo, hi)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        c, s = sv.batch(lo, hi)
        ts.append(time.perf_counter() - t0)
    e2e = statistics.median(ts)
    w = sv.get_options()["wheel"]
    pr = small_primes_np(math.isqrt(hi_max))
    m_alg = sum(marks_alg_interval(int(a), int(b), pr, w) for a, b in zip(lo, hi))
    r_atom, _ = sv.debug_k0()
    peak = 148 * r_atom * 1965e6
    emit({"config": 5, "mode": "batch", "kernel_ms": med, "kernel_ms_min": mn,
          "kernel_integers_per_s": total / (med / 1e3), "e2e_ms": e2e * 1e3,
          "e2e_integers_per_s": total / e2e, "ok": ok_k and int(c.sum()) == 715907351,
          "kernel_scope": "sieve_batch_async on device-resident intervals: K1 base primes + plan "
                          "(3 small kernels) + the batch sieve",
          "e2e_scope": "sieve_batch (host arrays): H2D of the intervals, the same device work, D2H",
          "wheel": w, "marks_alg": m_alg, "roofline_frac": m_alg / (med / 1e3) / peak,
          "peak_basis": f"148 x R_atom {r_atom:.2f} (K0) x 1965 MHz"})


def config4_frac(kernel_ms: float, seg_kb: int) -> dict:
    lo, hi = inputs.CONFIG4
    w = sv.get_options()["wheel"]
    pr = small_primes_np(math.isqrt(hi - 1))
    m = marks_alg_interval(lo, hi, pr, w)
    r_atom, _ = sv.debug_k0()
    return {"marks_alg": m, "wheel": w, "roofline_frac": m / (kernel_ms / 1e3) / (148 * r_atom * 1965e6)}


if __name__ == "__main__":
    which = [a for a in sys.argv[1:] if "=" not in a and not a.startswith("--")] or ["1", "2", "3b", "4", "5"]
    if "1" in which:
        config1()
    if "2" in which:
        specs = [a for a in sys.argv[1:] if "=" in a and not a.startswith("--")]
        if specs:
            for spec in specs:
                config2({k: int(v) for k, v in (kv.split("=") for kv in spec.split(","))})
        else:
            for kb in (32, 64, 128, 192, 208):
                config2(kb)
    if "3b" in which:  # config 3's range in bitmap mode: 625 MB, HBM-bound write-back
        config2({}, inputs.CONFIG3, tag=3)
    if "4" in which:
        for kb in (32, 208):
            config4(kb)
        config4_list()
    if "5" in which:
        config5()
    if "f2" in which:
        f2()
    rp = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--report=")]
    if rp:
        oracle_report(rp[0])
