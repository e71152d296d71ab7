"""One list-mode call of config 4 (for ncu): all 361,840,208 primes of
[1e12, 1e12 + 1e10) into device memory."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch, inputs
import paper_1205_4883_b200 as sv
lo, hi = inputs.CONFIG4
n = 361840208
out = torch.empty(n, dtype=torch.int64, device="cuda")
print(sv.primes(lo, hi, cap=n, out=out)[1])
