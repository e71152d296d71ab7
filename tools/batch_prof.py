"""Config 5 batch (sieve_batch through the host API), for an ncu launch list."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs
import paper_1205_4883_b200 as sv
lo, hi = inputs.config5_intervals()
for _ in range(int(os.environ.get("REPS", "2"))):
    t0 = time.perf_counter()
    c, s = sv.batch(lo, hi)
    print("batch ms", (time.perf_counter() - t0) * 1e3, int(c.sum()))
