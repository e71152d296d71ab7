"""Phase timeline of the base-prime kernel K1 (diagnostics counters,
globaltimer ns): small primes, slice marked, list offset known, end."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1205_4883_b200 as sv
from paper_1205_4883_b200 import dist as D
M = (1 << 64) - 1
stream = torch.cuda.Stream(); sv.set_stream(stream); torch.cuda.set_stream(stream)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for r in [int(x) for x in sys.argv[1:]]:
    b = D.alloc_base(sv.base_capacity(r), torch.device("cuda"))
    rows = []
    for i in range(10):
        flush.zero_()
        c = torch.zeros(120, dtype=torch.int64, device="cuda")
        sv.debug_set_profile(c)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); sv.base_primes_async(r, b.primes, b.recips, b.nbase); e1.record()
        torch.cuda.synchronize()
        sv.debug_set_profile(None)
        v = [x & M for x in c.cpu().tolist()]
        t0 = M ^ v[112]
        rows.append([e0.elapsed_time(e1) * 1e3] + [(v[k] - t0) / 1e3 for k in (113, 114, 115, 116)])
    m = [statistics.median(x) for x in zip(*rows[3:])]
    print(f"r={r} nbase={int(b.nbase.item())} event {m[0]:.1f}us | small primes {m[1]:.1f} | "
          f"marked {m[2]:.1f} | offset {m[3]:.1f} | end {m[4]:.1f}", flush=True)
