"""Quick timings for regression checks: config 4 count at 32 KiB segments and
config 5 batch (host API), with library/options from the environment
(SIEVE_LIBRARY, WHEEL)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs
import paper_1205_4883_b200 as sv
w = int(os.environ.get("WHEEL", "0"))
name = os.environ.get("SIEVE_LIBRARY", "default").split("/")[-1] + f" wheel={w or 'default'}"
lo, hi = inputs.CONFIG4
sv.set_options(segment_kb=32, wheel=w)
sv.stats(lo, hi)
ts = []
for _ in range(3):
    t0 = time.perf_counter(); sv.stats(lo, hi); ts.append(time.perf_counter() - t0)
c4 = min(ts) * 1e3
sv.set_options(wheel=w)
l5, h5 = inputs.config5_intervals(4096)
sv.batch(l5, h5)
ts = []
for _ in range(3):
    t0 = time.perf_counter(); sv.batch(l5, h5); ts.append(time.perf_counter() - t0)
print(f"{name}: config4@32KiB {c4:.2f} ms  config5 {min(ts)*1e3:.2f} ms", flush=True)
