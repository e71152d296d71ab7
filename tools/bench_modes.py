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


def emit(d):
    print(json.dumps(d), flush=True)


def config2(opts):
    if isinstance(opts, int):
        opts = {"segment_kb": opts}
    sv.set_options(**opts)
    seg_kb = sv.get_options()
    lo, hi = inputs.CONFIG2
    r, b = base_for(hi)
    words = sv.bitmap_words(lo, hi)
    out = torch.empty(words, dtype=torch.int32, device=dev)
    res = torch.zeros(2, dtype=torch.int64, device=dev)
    med, mn = timed(lambda: sv.bitmap_async(lo, hi, b.primes, b.recips, b.nbase, out, res))
    ok = res.cpu().tolist()[0] == 50847534
    sv.debug_set_flags(1)
    wmed, wmn = timed(lambda: sv.bitmap_async(lo, hi, b.primes, b.recips, b.nbase, out, res))
    sv.debug_set_flags(0)
    byts = words * 4
    emit({"config": 2, "mode": "bitmap", "segment_kb": seg_kb, "ok": ok, "kernel_ms": med,
          "integers_per_s": (hi - lo) / (med / 1e3), "bitmap_bytes": byts,
          "hbm_gbs_end_to_end": byts / (med / 1e3) / 1e9,
          "hbm_frac_end_to_end": byts / (med / 1e3) / 1e9 / HBM_PEAK,
          "writeback_only_ms": wmed, "writeback_only_gbs": byts / (wmed / 1e3) / 1e9,
          "writeback_only_frac": byts / (wmed / 1e3) / 1e9 / HBM_PEAK,
          "hbm_peak_gbs": HBM_PEAK, "peak_basis": "MEASURED_PEAKS.json hbm_gbs (copy)"})
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
          "ok": got == [361840208, 13161149016643422504]})
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


def config5():
    lo, hi = inputs.config5_intervals()
    total = int((hi - lo).sum())
    for _ in range(2):
        c, s = sv.batch(lo, hi)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        c, s = sv.batch(lo, hi)
        ts.append(time.perf_counter() - t0)
    med = statistics.median(ts)
    emit({"config": 5, "mode": "batch (sieve_batch, host API incl. item upload)", "ms": med * 1e3,
          "integers_per_s": total / med, "ok": int(c.sum()) == 715907351})


if __name__ == "__main__":
    which = [a for a in sys.argv[1:] if "=" not in a] or ["1", "2", "4", "5"]
    if "1" in which:
        config1()
    if "2" in which:
        specs = [a for a in sys.argv[1:] if "=" in a]
        if specs:
            for spec in specs:
                config2({k: int(v) for k, v in (kv.split("=") for kv in spec.split(","))})
        else:
            for kb in (32, 64, 128, 192, 208):
                config2(kb)
    if "4" in which:
        for kb in (32, 208):
            config4(kb)
        config4_list()
    if "5" in which:
        config5()
    if "f2" in which:
        f2()
