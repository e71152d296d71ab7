import os, sys, time, statistics
sys.path.insert(0, '.')
import torch, inputs
import paper_1205_4883_b200 as sv
lo, hi = inputs.CONFIG4
n = 361840208
out = torch.empty(n, dtype=torch.int64, device="cuda")
for _ in range(2): sv.primes(lo, hi, cap=n, out=out)
ts=[]
for _ in range(5):
    torch.cuda.synchronize(); t0=time.perf_counter(); c = sv.primes(lo, hi, cap=n, out=out)[1]; ts.append(time.perf_counter()-t0)
print(os.environ.get("SIEVE_LIBRARY","default"), "list ms", round(min(ts)*1e3,3), c)
