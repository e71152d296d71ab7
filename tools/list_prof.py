"""One config-4 list call (sieve_primes into device memory) for an ncu launch list."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import inputs
import paper_1205_4883_b200 as sv
lo, hi = inputs.CONFIG4
n = 361840208
out = torch.empty(n, dtype=torch.int64, device="cuda")
for _ in range(int(os.environ.get("REPS", "2"))):
    c = sv.primes(lo, hi, cap=n, out=out)[1]
torch.cuda.synchronize()
print("count", c)
