"""Base-prime kernel alone (K1) for r given on the command line (ncu target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1205_4883_b200 as sv
from paper_1205_4883_b200 import dist as D
r = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
b = D.alloc_base(sv.base_capacity(r), torch.device("cuda"))
for _ in range(3):
    sv.base_primes_async(r, b.primes, b.recips, b.nbase)
torch.cuda.synchronize()
print("nbase", int(b.nbase.item()))
