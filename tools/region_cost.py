"""Marginal cost of each marking region in context: config 3 sieve-kernel time
with regions dropped by the diagnostic flags (wrong results by design)."""
import math, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1205_4883_b200 as sv
from paper_1205_4883_b200 import dist as D
lo, hi = (int(x) for x in os.environ.get("RANGE", "2,10000000001").split(","))
stream = torch.cuda.Stream(); sv.set_stream(stream); torch.cuda.set_stream(stream)
r = math.isqrt(hi - 1)
b = D.alloc_base(sv.base_capacity(r), torch.device("cuda"))
res = torch.zeros(2, dtype=torch.int64, device="cuda")
sv.base_primes_async(r, b.primes, b.recips, b.nbase)
for name, fl in [("all", 0), ("-A", 2), ("-B", 4), ("-C", 8), ("-A-B", 6), ("-A-C", 10), ("-B-C", 12), ("-ABC", 14), ("no marking", 1)]:
    sv.debug_set_flags(fl)
    ts = []
    for i in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); sv.stats_async(lo, hi, b.primes, b.recips, b.nbase, res); e1.record()
        torch.cuda.synchronize()
        if i >= 3: ts.append(e0.elapsed_time(e1))
    print(f"{name:12s} {statistics.median(ts):.3f} ms", flush=True)
sv.debug_set_flags(0)
