"""Launch timeline of the count kernel (diagnostics counters, globaltimer ns):
CTA entry spread, prologue, sieving, final reduction, and the event-timed
total (the rest is launch and drain)."""
import math, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1205_4883_b200 as sv
from paper_1205_4883_b200 import dist as D
M = (1 << 64) - 1
stream = torch.cuda.Stream(); sv.set_stream(stream); torch.cuda.set_stream(stream)
for spec in sys.argv[1:]:
    lo, hi = (int(x) for x in spec.split(","))
    r = math.isqrt(hi - 1)
    b = D.alloc_base(sv.base_capacity(r), torch.device("cuda"))
    res = torch.zeros(2, dtype=torch.int64, device="cuda")
    sv.base_primes_async(r, b.primes, b.recips, b.nbase)
    rows = []
    for i in range(8):
        c = torch.zeros(120, dtype=torch.int64, device="cuda")
        sv.debug_set_profile(c)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if os.environ.get("FUSED"):
            sv.stats_base_async(lo, hi, b.primes, b.recips, b.nbase, res)
        else:
            sv.stats_async(lo, hi, b.primes, b.recips, b.nbase, res)
        e1.record()
        torch.cuda.synchronize()
        sv.debug_set_profile(None)
        v = [x & M for x in c.cpu().tolist()]
        t0 = M ^ v[104]
        rows.append((e0.elapsed_time(e1) * 1e3, (v[105] - t0) / 1e3, (v[106] - t0) / 1e3,
                     ((M ^ v[109]) - t0) / 1e3, (v[107] - t0) / 1e3, (v[108] - t0) / 1e3,
                     max(0, v[110] - t0) / 1e3, max(0, v[111] - t0) / 1e3,
                     max(0, v[117] - t0) / 1e3, max(0, v[118] - t0) / 1e3))
    med = [statistics.median(x) for x in zip(*rows[3:])]
    fa = (f" | fused A2: counted {med[6]:.1f}, barrier1 {med[7]:.1f}, emitted {med[8]:.1f}, "
          f"barrier2 {med[9]:.1f}" if os.environ.get("FUSED") else "")
    print(f"[{lo},{hi}) event {med[0]:.1f}us | entry spread {med[1]:.1f} | prologue done {med[2]:.1f} | "
          f"first CTA done {med[3]:.1f} | last CTA done {med[4]:.1f} | result {med[5]:.1f} | "
          f"launch+drain {med[0] - med[5]:.1f}{fa}", flush=True)
