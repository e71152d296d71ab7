"""Run one sieve_stats_async on a config range (for ncu captures)."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1205_4883_b200 as sv
from paper_1205_4883_b200 import dist as D
lo, hi = int(sys.argv[1]), int(sys.argv[2])
opts = dict(kv.split("=") for kv in (sys.argv[3].split(",") if len(sys.argv) > 3 and sys.argv[3] else []))
sv.set_options(**{k: int(v) for k, v in opts.items()})
r = math.isqrt(hi - 1)
b = D.alloc_base(sv.base_capacity(r), torch.device("cuda"))
res = torch.zeros(2, dtype=torch.int64, device="cuda")
for _ in range(int(os.environ.get("REPS", "2"))):
    sv.base_primes_async(r, b.primes, b.recips, b.nbase)
    sv.stats_async(lo, hi, b.primes, b.recips, b.nbase, res)
torch.cuda.synchronize()
print([D.i64_to_u64(x) for x in res.cpu().tolist()])
