"""Time sieve_stats_async (kernel only, CUDA events) on a range with options."""
import math, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1205_4883_b200 as sv
from paper_1205_4883_b200 import dist as D
lo, hi = int(sys.argv[1]), int(sys.argv[2])
stream = torch.cuda.Stream()
sv.set_stream(stream)
torch.cuda.set_stream(stream)
for spec in sys.argv[3:] or [""]:
    opts = dict(kv.split("=") for kv in spec.split(",") if kv)
    sv.set_options(**{k: int(v) for k, v in opts.items()})
    r = math.isqrt(hi - 1)
    b = D.alloc_base(sv.base_capacity(r), torch.device("cuda"))
    res = torch.zeros(2, dtype=torch.int64, device="cuda")
    sv.base_primes_async(r, b.primes, b.recips, b.nbase)
    ts = []
    for i in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); sv.stats_async(lo, hi, b.primes, b.recips, b.nbase, res); e1.record()
        torch.cuda.synchronize()
        if i >= 2: ts.append(e0.elapsed_time(e1))
    print(os.environ.get("SIEVE_LIBRARY", "default").split("/")[-1], spec, "ms=%.3f" % statistics.median(ts),
          [D.i64_to_u64(x) for x in res.cpu().tolist()], flush=True)
