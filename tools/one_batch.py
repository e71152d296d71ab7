"""Config 5 through sieve_batch_async once (an ncu capture target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import inputs
import paper_1205_4883_b200 as sv
lo, hi = inputs.config5_intervals()
dlo = torch.from_numpy(lo.view(np.int64)).cuda()
dhi = torch.from_numpy(hi.view(np.int64)).cuda()
res = torch.zeros(2 * lo.size, dtype=torch.int64, device="cuda")
sv.set_stream(torch.cuda.current_stream())
for _ in range(int(os.environ.get("REPS", "1"))):
    sv.batch_async(dlo, dhi, int(hi.max()), int((hi - lo).max()), res)
torch.cuda.synchronize()
print(int(res.cpu().numpy().view(np.uint64)[0::2].sum()))
