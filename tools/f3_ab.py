"""F3 A/B: the cluster-pair kernel (sieve_debug_set_flags
FLAG_CLUSTER: two CTAs per super-segment, region C over distributed shared
memory) against the product count kernel, same box, same base primes (K1
outside the timed region), CUDA events, L2 flushed; results checked."""
import math, os, statistics, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import oracle
import paper_1205_4883_b200 as sv
from paper_1205_4883_b200 import dist as D
FLAG_CLUSTER = 64
stream = torch.cuda.Stream(); sv.set_stream(stream); torch.cuda.set_stream(stream)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
cases = [("config3", 2, 10**10 + 1, 208, (455052511, 2220822432581729238)),
         ("config4", 10**12, 10**12 + 10**10, 208, (361840208, 13161149016643422504)),
         ("config4@32KiB", 10**12, 10**12 + 10**10, 32, (361840208, 13161149016643422504))]
# small correctness cases (odd and even segment counts, ragged ends)
for lo, hi in [(2, 10**8 + 1), (10**12 + 1, 10**12 + 3 * 10**7 + 7), (999_999_999_989, 1_000_040_000_000)]:
    sv.set_options(segment_kb=16)
    sv.debug_set_flags(FLAG_CLUSTER)
    got = sv.stats(lo, hi)
    sv.debug_set_flags(0)
    assert got == oracle.stats(lo, hi), (lo, hi, got)
sv.set_options()
for name, lo, hi, kb, want in cases:
    sv.set_options(segment_kb=kb)
    r = math.isqrt(hi - 1)
    b = D.alloc_base(sv.base_capacity(r), torch.device("cuda"))
    res = torch.zeros(2, dtype=torch.int64, device="cuda")
    sv.base_primes_async(r, b.primes, b.recips, b.nbase)
    out = {}
    for label, flags in (("product", 0), ("cluster", FLAG_CLUSTER)):
        sv.debug_set_flags(flags)
        ts = []
        for i in range(10):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); sv.stats_async(lo, hi, b.primes, b.recips, b.nbase, res); e1.record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(e0.elapsed_time(e1))
        got = tuple(int(x) & ((1 << 64) - 1) for x in res.cpu().tolist())
        out[label] = {"ms": statistics.median(ts), "ok": got == want}
    sv.debug_set_flags(0)
    print(json.dumps({"case": name, "segment_kb": kb, **out}), flush=True)
sv.set_options()
