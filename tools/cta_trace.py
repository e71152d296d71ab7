import os, sys, statistics
sys.path.insert(0, '.')
import torch, numpy as np
import paper_1205_4883_b200 as sv
M = (1 << 64) - 1
for spec in sys.argv[1:]:
    lo, hi = (int(x) for x in spec.split(","))
    sv.stats(lo, hi)
    rows = []
    for rep in range(3):
        c = torch.zeros(120 + 2 * 148, dtype=torch.int64, device="cuda")
        sv.debug_set_profile(c)
        sv.stats(lo, hi)
        torch.cuda.synchronize()
        sv.debug_set_profile(None)
        v = [x & M for x in c.cpu().tolist()]
        t0 = M ^ v[104]
        sm = np.array(v[120::2][:148]); t = (np.array(v[121::2][:148]) - t0) / 1e3
        rows.append((sm, t))
    sm, t = rows[-1]
    order = np.argsort(sm)
    print(spec, "end of sieving per SM (us), min/median/max:", t.min().round(1), np.median(t).round(1), t.max().round(1))
    half = sm < 74
    print("  SM < 74:", t[half].mean().round(1), " SM >= 74:", t[~half].mean().round(1))
    # correlation between reps per SM
    a = np.zeros(148); b = np.zeros(148)
    for s_, tt in zip(rows[0][0], rows[0][1]): a[s_] = tt
    for s_, tt in zip(rows[1][0], rows[1][1]): b[s_] = tt
    print("  rep-to-rep correlation of per-SM end times:", np.corrcoef(a, b)[0, 1].round(2))
    print("  slowest SMs:", sm[np.argsort(-t)[:10]].tolist())
    print("  per-GPC-ish blocks of 16 SM mean:", [round(float(t[(sm >= g) & (sm < g + 16)].mean()), 1) for g in range(0, 148, 16)])
