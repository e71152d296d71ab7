"""A/B timing of the count kernel on several ranges for one library build
(SIEVE_LIBRARY); run once per variant, interleaved, by tools/ab.sh."""
import math, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1205_4883_b200 as sv
from paper_1205_4883_b200 import dist as D
stream = torch.cuda.Stream(); sv.set_stream(stream); torch.cuda.set_stream(stream)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
name = os.environ.get("SIEVE_LIBRARY", "default").split("/")[-1]
for spec in sys.argv[1:]:
    lo, hi = (int(x) for x in spec.split(","))
    r = math.isqrt(hi - 1)
    b = D.alloc_base(sv.base_capacity(r), torch.device("cuda"))
    res = torch.zeros(2, dtype=torch.int64, device="cuda")
    sv.base_primes_async(r, b.primes, b.recips, b.nbase)
    ts = []
    for i in range(12):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); sv.stats_async(lo, hi, b.primes, b.recips, b.nbase, res); e1.record()
        torch.cuda.synchronize()
        if i >= 3: ts.append(e0.elapsed_time(e1))
    print(f"{name} {spec} {statistics.median(ts) * 1e3:.1f}us", flush=True)
