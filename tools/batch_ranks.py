"""Config 5 split over G ranks by dist.batch's LPT assignment (A10 multi-GPU):
each rank's share of the 4096 intervals timed alone on one B200 with
sieve_batch_async (device-resident intervals; K1 + plan + batch sieve, CUDA
events, L2 flushed).  The N-GPU batch step is max over ranks of these plus an
all_gather of 64 KB; prints per-rank ms and the max/mean balance."""
import os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import inputs
import paper_1205_4883_b200 as sv
from paper_1205_4883_b200 import dist as D

lo, hi = inputs.config5_intervals()
st = torch.cuda.Stream(); sv.set_stream(st); torch.cuda.set_stream(st)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
total = int((hi - lo).sum())


def t_share(idx):
    l, h = lo[idx], hi[idx]
    dl = torch.from_numpy(l.view(np.int64)).cuda()
    dh = torch.from_numpy(h.view(np.int64)).cuda()
    res = torch.zeros(2 * idx.size, dtype=torch.int64, device="cuda")
    ts = []
    for i in range(7):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); sv.batch_async(dl, dh, int(h.max()), int((h - l).max()), res); e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


for G in [int(x) for x in os.environ.get("GS", "1,2,4,8").split(",")]:
    parts = D.lpt_assign(D.batch_cost(lo, hi), G)
    ms = [t_share(p) for p in parts]
    mx = max(ms)
    print(f"G={G} per-rank ms {[round(x, 3) for x in ms]} max {mx:.3f} mean {statistics.mean(ms):.3f} "
          f"max/mean {mx / statistics.mean(ms):.3f} -> projected {total / (mx / 1e3):.3e} integers/s", flush=True)
