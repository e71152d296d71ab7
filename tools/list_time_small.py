"""List-mode timing on ranges served by the non-plain list kernel (r <= S/8):
[2, 1e9+1) and [1e9, 2e9) into device memory; min of 5 synchronous calls."""
import os, sys, time
sys.path.insert(0, '.')
import torch
import paper_1205_4883_b200 as sv
for lo, hi in [(2, 10**9 + 1), (10**9, 2 * 10**9)]:
    n = sv.count(lo, hi)
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    for _ in range(2): sv.primes(lo, hi, cap=n, out=out)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize(); t0 = time.perf_counter(); c = sv.primes(lo, hi, cap=n, out=out)[1]; ts.append(time.perf_counter() - t0)
    print(os.environ.get("SIEVE_LIBRARY", "default"), f"[{lo},{hi}) list ms", round(min(ts) * 1e3, 4), c, flush=True)
