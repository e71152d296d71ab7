"""Launch overhead of the fused count launch (the N>1 production step) on
one B200: the G=8 top block of config 3 timed with CUDA events (a) after an
L2-flush kernel (torch fill, as bench.py), (b) back to back, (c) after a
small kernel that uses no shared memory.  The difference between (a)/(c)
and (b) is what the switch of the SM's shared-memory carve-out between the
flush kernel and the 208 KiB sieve kernel costs inside the events."""
import math, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1205_4883_b200 as sv
from paper_1205_4883_b200 import dist as D

stream = torch.cuda.Stream(); sv.set_stream(stream); torch.cuda.set_stream(stream)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
small = torch.empty(1024, dtype=torch.uint8, device="cuda")
lo, hi = 2, 10**10 + 1
G = int(os.environ.get("G", "8"))
for g in (0, G - 1):
    a, b = D.block_of(lo, hi, g, G)
    base = D.alloc_base(sv.base_capacity(math.isqrt(b - 1)), torch.device("cuda"))
    res = torch.zeros(2, dtype=torch.int64, device="cuda")
    out = {}
    for mode in ("flush", "b2b", "small"):
        ts = []
        for i in range(15):
            if mode == "flush":
                flush.zero_()
            elif mode == "small":
                small.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); sv.stats_base_async(a, b, base.primes, base.recips, base.nbase, res); e1.record()
            if mode != "b2b":
                torch.cuda.synchronize()
            ts.append((e0, e1))
        torch.cuda.synchronize()
        out[mode] = statistics.median(x.elapsed_time(y) * 1e3 for x, y in ts[3:])
    print(f"G={G} block {g} [{a},{b}): " + " ".join(f"{k}={v:.1f}us" for k, v in out.items()), flush=True)
