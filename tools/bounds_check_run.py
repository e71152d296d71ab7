"""Every kernel path against the oracle, run with the BOUNDS-CHECK build
(libsieve_check.so, -DSIEVE_CHECK_BOUNDS=1; include/sieve.h
sieve_debug_violations): count, bitmap (bulk copy, unaligned and ragged
outputs), list, batch, fused base launch, the K1 + ordinary-launch path,
reversed segment order, bucket rings, small and maximum segments, every
wheel, hi = 2^48.  Prints one JSON line {"check_build": ..., "violations":
[smem marks, bitmap stores, list stores, scratch], "cases": n}; exits 1 on
a parity failure.  tests/test_gpu_bounds.py runs it in a subprocess with
SIEVE_LIBRARY pointing at the check build."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import oracle  # noqa: E402
import paper_1205_4883_b200 as sv  # noqa: E402
from paper_1205_4883_b200 import dist as D  # noqa: E402

sv.set_device(0)
is_check, v0 = sv.debug_violations(reset=True)
cases = 0


def three_modes(lo, hi):
    global cases
    want = oracle.stats(lo, hi)
    assert sv.stats(lo, hi) == want, (lo, hi)
    bm, c = sv.bitmap(lo, hi)
    obm, oc, _ = oracle.bitmap(lo, hi)
    assert c == oc and np.array_equal(bm[: obm.size], obm), (lo, hi)
    lst, n = sv.primes(lo, hi)
    assert n == want[0] and np.array_equal(lst[:n], oracle.primes(lo, hi)), (lo, hi)
    cases += 1


opts = [dict(), dict(segment_kb=4), dict(segment_kb=16, buckets=1), dict(segment_kb=32, buckets=1),
        dict(segment_kb=216, wheel=11), dict(segment_kb=64, wheel=47), dict(segment_kb=104, wheel=17),
        dict(threads=256, segment_kb=40), dict(ctas_per_sm=2, segment_kb=96)]
ranges = [(2, 3 * 10**6 + 1), (0, 100), (7, 7), (10**9 + 1, 10**9 + 4 * 10**6 + 3),
          (10**12 - 7, 10**12 + 2 * 10**6 + 5), ((1 << 48) - 10**6 - 17, 1 << 48)]
for o in opts:
    sv.set_options(**o)
    for lo, hi in ranges:
        three_modes(lo, hi)
sv.set_options()
# diagnostic paths: reversed segment order, the non-cooperative fallback
for flags in (sv.FLAG_REVERSE, sv.FLAG_NO_COOP, sv.FLAG_REVERSE | sv.FLAG_NO_COOP, sv.FLAG_CLUSTER):
    sv.debug_set_flags(flags)
    for lo, hi in ranges[:5]:
        three_modes(lo, hi)
sv.debug_set_flags(0)
# device outputs at every 4-byte offset (bulk copy vs plain stores) and a
# list output 8 bytes past a 16-byte boundary
for shift in range(4):
    lo, hi = 10**9 + 1, 10**9 + 64 * (4 * 4096 + 3) - 5
    w = sv.bitmap_words(lo, hi)
    buf = torch.zeros(w + 8, dtype=torch.int32, device="cuda")
    _, c = sv.bitmap(lo, hi, out=buf[shift: shift + w])
    obm, oc, _ = oracle.bitmap(lo, hi)
    assert c == oc and np.array_equal(buf[shift: shift + w].cpu().numpy().view(np.uint32), obm)
    cases += 1
full = oracle.primes(10**9, 10**9 + 10**6)
d2 = torch.zeros(full.size + 1, dtype=torch.int64, device="cuda")
_, c = sv.primes(10**9, 10**9 + 10**6, cap=full.size, out=d2[1:])
assert c == full.size and np.array_equal(d2[1:].cpu().numpy().view(np.uint64), full)
_, c = sv.primes(10**9, 10**9 + 10**6, cap=100, out=d2[1:])  # truncated
assert c == full.size and np.array_equal(d2[1:101].cpu().numpy().view(np.uint64), full[:100])
# batch: config-5 style intervals and edge intervals
lo5, hi5 = inputs.config5_intervals(64)
c, s = sv.batch(lo5, hi5)
oc, os_ = oracle.batch(lo5, hi5)
assert np.array_equal(c, oc) and np.array_equal(s, os_)
iv = inputs.random_intervals(200, seed=99, lo_max=10**13, width_max=10**6) + [(0, 0), (2, 3), (0, 300)]
lo = np.array([a for a, _ in iv], dtype=np.uint64)
hi = np.array([b for _, b in iv], dtype=np.uint64)
c, s = sv.batch(lo, hi)
oc, os_ = oracle.batch(lo, hi)
assert np.array_equal(c, oc) and np.array_equal(s, os_)
cases += 2
# config 2's bitmap at the four swept segment sizes (hash only: 62.5 MB)
for kb in (32, 64, 128, 192):
    sv.set_options(segment_kb=kb)
    bm, c = sv.bitmap(*inputs.CONFIG2)
    assert c == 50847534 and oracle.fnv1a64(bm) == 0xe4b98535dc2fea3d
    cases += 1
sv.set_options()
# the device-resident fused-base launch
dev = torch.device("cuda", 0)
base = D.alloc_base(sv.base_capacity(10**5), dev)
res = torch.zeros(2, dtype=torch.int64, device=dev)
sv.set_stream(torch.cuda.current_stream())
sv.stats_base_async(2, 10**10 + 1, base.primes, base.recips, base.nbase, res)
torch.cuda.synchronize()
assert [int(x) & ((1 << 64) - 1) for x in res.cpu().tolist()] == [455052511, 2220822432581729238]
sv.set_stream(None)
cases += 1
is_check, v = sv.debug_violations()
print(json.dumps({"check_build": is_check, "violations": v, "cases": cases,
                  "library": sv.library_path}))
