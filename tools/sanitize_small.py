"""Small invocations of every kernel path (count, bitmap, list, batch, fused
base launch, F2), each checked against the oracle: a quick all-paths smoke,
and the script to run under compute-sanitizer where the pool allows it."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
import paper_1205_4883_b200 as sv
from paper_1205_4883_b200 import dist as D
sv.set_options(segment_kb=int(os.environ.get("SEG_KB", "16")))
for lo, hi in [(2, 3 * 10**5 + 1), (10**9, 10**9 + 2 * 10**5 + 7), (7, 7), (0, 100)]:
    assert sv.stats(lo, hi) == oracle.stats(lo, hi), (lo, hi)
    bm, c = sv.bitmap(lo, hi)
    obm, oc, _ = oracle.bitmap(lo, hi)
    assert c == oc and np.array_equal(bm[: obm.size], obm)
    lst, c2 = sv.primes(lo, hi)
    assert c2 == oracle.stats(lo, hi)[0] and np.array_equal(lst[:c2], oracle.primes(lo, hi))
lo = np.array([10**6, 10**9, 5 * 10**11], dtype=np.uint64)
hi = lo + np.array([10**5, 3 * 10**5, 2 * 10**5], dtype=np.uint64)
c, s = sv.batch(lo, hi)
oc, os_ = oracle.batch(lo, hi)
assert np.array_equal(c, oc) and np.array_equal(s, os_)
dev = torch.device("cuda", 0)
base = D.alloc_base(sv.base_capacity(10**5), dev)
res = torch.zeros(2, dtype=torch.int64, device=dev)
sv.set_stream(torch.cuda.current_stream())
sv.stats_base_async(10**9, 10**9 + 10**6, base.primes, base.recips, base.nbase, res)
torch.cuda.synchronize()
assert tuple(int(x) & ((1 << 64) - 1) for x in res.cpu().tolist()) == oracle.stats(10**9, 10**9 + 10**6)
sv.set_stream(None)
p = np.array([97, 561, 1105, 2**61 - 1], dtype=np.uint64)
assert sv.is_prime(p).tolist() == [1, 0, 0, 1]
print("sanitize run ok")
