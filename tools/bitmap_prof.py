"""Config 2 bitmap write-back (sieve_bitmap_async into device memory), optionally
with marking skipped (FLAGS=1: the write-back stage in isolation); ncu target."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import inputs
import paper_1205_4883_b200 as sv
from paper_1205_4883_b200 import dist as D
lo, hi = inputs.CONFIG3 if os.environ.get('CFG') == '3' else inputs.CONFIG2
r = math.isqrt(hi - 1)
b = D.alloc_base(sv.base_capacity(r), torch.device("cuda"))
sv.base_primes_async(r, b.primes, b.recips, b.nbase)
out = torch.empty(sv.bitmap_words(lo, hi), dtype=torch.int32, device="cuda")
res = torch.zeros(2, dtype=torch.int64, device="cuda")
sv.debug_set_flags(int(os.environ.get("FLAGS", "0")))
for _ in range(int(os.environ.get('CALLS', '3'))):
    sv.bitmap_async(lo, hi, b.primes, b.recips, b.nbase, out, res)
torch.cuda.synchronize()
print(res.tolist())
