"""Per-rank sieve-kernel time and roofline fraction of config 3 split over G
GPUs, measured one block at a time on one GPU (each rank's block is an
independent range: the N>1 kernels do not interact until the all-reduce).
Env: GS (default 1,2,4,8), SPLIT=equal|cost (dist.block_of), RANKS=ends|all."""
import math, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1205_4883_b200 as sv
from paper_1205_4883_b200 import dist as D

stream = torch.cuda.Stream(); sv.set_stream(stream); torch.cuda.set_stream(stream)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
lo, hi = bench.CONFIG3
r_atom, _ = sv.debug_k0()  # K0 on this GPU (lanes/clk/SM)
peak = 148 * r_atom * 1965e6 / 1e9
W = sv.get_options()["wheel"]
SPLIT = os.environ.get("SPLIT", "equal")
for G in [int(x) for x in os.environ.get("GS", "1,2,4,8").split(",")]:
    for g in (range(G) if os.environ.get("RANKS", "ends") == "all" else sorted({0, G - 1})):
        a, b = D.block_of(lo, hi, g, G, SPLIT)
        r = math.isqrt(b - 1)
        base = D.alloc_base(sv.base_capacity(r), torch.device("cuda"))
        res = torch.zeros(2, dtype=torch.int64, device="cuda")
        ks, bs = [], []
        for i in range(13):
            flush.zero_()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record(); sv.base_primes_async(r, base.primes, base.recips, base.nbase)
            e[1].record(); sv.stats_async(a, b, base.primes, base.recips, base.nbase, res); e[2].record()
            torch.cuda.synchronize()
            if i >= 3:
                bs.append(e[0].elapsed_time(e[1])); ks.append(e[1].elapsed_time(e[2]))
        fs = []
        for i in range(13):  # A2 fused into the sieve launch
            flush.zero_()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            e[0].record(); sv.stats_base_async(a, b, base.primes, base.recips, base.nbase, res); e[1].record()
            torch.cuda.synchronize()
            if i >= 3:
                fs.append(e[0].elapsed_time(e[1]))
        k = statistics.median(ks)
        m = bench.algorithmic_marks(a, b, W)
        print(f"split={SPLIT} G={G} rank={g} [{a},{b}) K1={statistics.median(bs)*1e3:.1f}us sieve={k*1e3:.1f}us "
              f"frac={m / (k / 1e3) / 1e9 / peak:.3f} | K1+sieve={(statistics.median(bs) + k)*1e3:.1f}us "
              f"fused={statistics.median(fs)*1e3:.1f}us", flush=True)
