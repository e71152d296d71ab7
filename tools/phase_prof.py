"""Phase breakdown of the sieve kernel (diagnostics counters, not a bench number)."""
import sys, json
sys.path.insert(0, ".")
import torch
import paper_1205_4883_b200 as sv
import os
lo, hi = (int(x) for x in os.environ.get("RANGE", "2,10000000001").split(","))
for spec in sys.argv[1:] or [""]:
    kw = dict(kv.split("=") for kv in spec.split(",") if kv)
    kw = {k: int(v) for k, v in kw.items()}
    sv.set_options(**kw)
    sv.stats(lo, hi)
    c = torch.zeros(120, dtype=torch.int64, device="cuda")
    sv.debug_set_profile(c)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); ev0.record(); r = sv.stats(lo, hi); ev1.record(); torch.cuda.synchronize()
    sv.debug_set_profile(None)
    v = c.cpu().tolist()
    cta = v[0] + v[1] + v[2]
    o = sv.get_options()
    nw = o["threads"] // 32
    print(json.dumps({"opts": o, "ms_with_prof": ev0.elapsed_time(ev1), "result": r,
          "segments": v[6], "cta_cycles_per_seg": cta / v[6],
          "init%": 100 * v[0] / cta, "mark%": 100 * v[1] / cta, "epi%": 100 * v[2] / cta,
          "warp_A1_per_seg": v[3] / v[6] / nw, "warp_A2_per_seg": v[4] / v[6] / nw,
          "warp_B_per_seg": v[5] / v[6] / nw, "warp_C_per_seg": v[7] / v[6] / nw,
          "per_warp_A_per_seg": [round(x / v[6]) for x in v[8:8 + nw]],
          "per_warp_B_per_seg": [round(x / v[6]) for x in v[40:40 + nw]],
          "per_warp_C_per_seg": [round(x / v[6]) for x in v[72:72 + nw]], "mark_cta_per_seg": v[1] / v[6]}))
