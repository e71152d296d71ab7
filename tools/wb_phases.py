"""Write-back stage of config 2 in isolation (marking skipped): kernel time
and per-segment CTA phase cycles (wheel init / epilogue incl. transpose and
stores) in bitmap mode against count mode (no transpose, no stores)."""
import math, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import inputs
import paper_1205_4883_b200 as sv
from paper_1205_4883_b200 import dist as D
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(); sv.set_stream(stream); torch.cuda.set_stream(stream)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
lo, hi = inputs.CONFIG3 if 'c3' in sys.argv[1:] else inputs.CONFIG2
r = math.isqrt(hi - 1)
b = D.alloc_base(sv.base_capacity(r), dev)
sv.base_primes_async(r, b.primes, b.recips, b.nbase)
words = sv.bitmap_words(lo, hi)
out = torch.empty(words, dtype=torch.int32, device=dev)
res = torch.zeros(2, dtype=torch.int64, device=dev)
calls = {"bitmap": lambda: sv.bitmap_async(lo, hi, b.primes, b.recips, b.nbase, out, res),
         "count": lambda: sv.stats_async(lo, hi, b.primes, b.recips, b.nbase, res)}
for skip in (1, 0):
    sv.debug_set_flags(skip)
    for name, fn in calls.items():
        ts = []
        for i in range(13):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(e0.elapsed_time(e1))
        c = torch.zeros(120, dtype=torch.int64, device=dev)
        sv.debug_set_profile(c)
        fn()
        torch.cuda.synchronize()
        sv.debug_set_profile(None)
        v = c.cpu().tolist()
        segs = max(v[6], 1)
        first = (1 << 64) - 1 - (v[104] & ((1 << 64) - 1)) if v[104] else 0
        span = lambda k: (v[k] - first) / 1e3 if v[k] else float("nan")
        print(f"skip={skip} {name:6s} {statistics.median(ts)*1e3:7.1f}us  GB/s {words*4/statistics.median(ts)/1e6:7.0f}"
              f"  segs {segs}  per seg: wheel {v[0]/segs:.0f} mark {v[1]/segs:.0f} epi {v[2]/segs:.0f} cyc"
              f"  | regions done {span(106):.1f} first CTA end {(((1<<64)-1-(v[109]&((1<<64)-1))) - first)/1e3:.1f}"
              f" last {span(107):.1f} result {span(108):.1f} us", flush=True)
sv.debug_set_flags(0)
