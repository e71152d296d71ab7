"""Per-CTA phase cycles (wheel init / marking / epilogue incl. list emission)
of config 4 in count mode and list mode (diagnostics counters)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import inputs
import paper_1205_4883_b200 as sv
lo, hi = inputs.CONFIG4
n = 361840208
out = torch.empty(n, dtype=torch.int64, device="cuda")
for mode in ("count", "list"):
    for rep in range(2):
        c = torch.zeros(120, dtype=torch.int64, device="cuda")
        sv.debug_set_profile(c)
        if mode == "count":
            sv.stats(lo, hi)
        else:
            sv.primes(lo, hi, cap=n, out=out)
        torch.cuda.synchronize()
        sv.debug_set_profile(None)
    v = c.cpu().tolist()
    segs = v[6]
    print(f"{mode}: segments {segs}  per segment (CTA cycles): wheel {v[0]/segs:.0f}  marking {v[1]/segs:.0f}  "
          f"epilogue/emission {v[2]/segs:.0f}", flush=True)
