"""Config 5 kernel time (sieve_batch_async, device-resident intervals, CUDA
events, L2 flushed) for one library build (SIEVE_LIBRARY); checks the
per-interval results against tests/golden/config5_oracle.txt."""
import os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch
import inputs
import paper_1205_4883_b200 as sv
from golden_io import config5_oracle
lo, hi = inputs.config5_intervals()
dlo = torch.from_numpy(lo.view(np.int64)).cuda()
dhi = torch.from_numpy(hi.view(np.int64)).cuda()
res = torch.zeros(2 * lo.size, dtype=torch.int64, device="cuda")
st = torch.cuda.Stream(); sv.set_stream(st); torch.cuda.set_stream(st)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
ts = []
for i in range(8):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); sv.batch_async(dlo, dhi, int(hi.max()), int((hi - lo).max()), res); e1.record()
    torch.cuda.synchronize()
    if i >= 2:
        ts.append(e0.elapsed_time(e1))
got = res.cpu().numpy().view(np.uint64)
_, _, fc, fs = config5_oracle()
ok = np.array_equal(got[0::2], fc) and np.array_equal(got[1::2], fs)
print(os.path.basename(os.environ.get("SIEVE_LIBRARY", "default")), "config5",
      f"{statistics.median(ts) * 1e3:.1f}us", "ok" if ok else "MISMATCH", flush=True)
