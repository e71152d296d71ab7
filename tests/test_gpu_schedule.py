"""Schedule invariance and the launch fallbacks (the result
must not depend on the order or the assignment of the work).

* reversed segment order (FLAG_REVERSE: every CTA of the bitmap kernel walks
  its segments backwards) gives bit-identical bitmaps and identical counts;
* the K1 + ordinary-launch path (FLAG_NO_COOP, the runtime's fallback when a
  cooperative fused-A2 launch is refused) gives identical results;
* an explicit ctas_per_sm above the occupancy is clamped (the fused A2 grid
  barriers and the list look-back need every CTA resident);
* switching the library stream orders the new stream after the old one;
* K0 measures the conflict-free shared atomicOr rate (~32 lanes/clk/SM).
"""
import numpy as np
import pytest

import inputs
import oracle
import paper_1205_4883_b200 as sv

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _reset():
    sv.set_options()
    sv.debug_set_flags(0)
    yield
    sv.debug_set_flags(0)
    sv.set_options()


RANGES = [(2, 4 * 10**7 + 1), (10**12 + 3, 10**12 + 3 * 10**7), (999_999_999_989, 1_000_100_000_000),
          (0, 5000), (41, 47)]


@pytest.mark.parametrize("seg_kb", [16, 64, 208])
def test_reverse_segment_order_invariance(seg_kb):
    sv.set_options(segment_kb=seg_kb)
    fwd = [(sv.stats(lo, hi), sv.bitmap(lo, hi)[0].copy()) for lo, hi in RANGES]
    sv.debug_set_flags(sv.FLAG_REVERSE)  # bitmap mode walks its segments backwards
    for (lo, hi), (st, bm) in zip(RANGES, fwd):
        assert st == oracle.stats(lo, hi), (lo, hi)
        bm2, c2 = sv.bitmap(lo, hi)
        assert np.array_equal(bm2, bm) and c2 == st[0], (lo, hi)
    bm, c = sv.bitmap(*inputs.CONFIG2)
    assert c == 50847534 and oracle.fnv1a64(bm) == 0xe4b98535dc2fea3d


def test_non_cooperative_fallback_path():
    sv.debug_set_flags(sv.FLAG_NO_COOP)
    n0 = sv.kernel_launches()
    for lo, hi in RANGES:
        want = oracle.stats(lo, hi)
        assert sv.stats(lo, hi) == want
        bm, c = sv.bitmap(lo, hi)
        obm, oc, _ = oracle.bitmap(lo, hi)
        assert c == oc and np.array_equal(bm[: obm.size], obm)
        lst, n = sv.primes(lo, hi)
        assert np.array_equal(lst[:n], oracle.primes(lo, hi))
    # K1 runs before each sieve launch on this path: more launches than calls
    assert sv.kernel_launches() - n0 > 3 * len(RANGES)
    assert sv.stats(*inputs.CONFIG3) == (455052511, 2220822432581729238)


@pytest.mark.parametrize("per", [2, 4, 8])
def test_ctas_per_sm_clamped_to_occupancy(per):
    # 1024 threads x 64 registers: one CTA per SM; asking for more must not
    # launch non-resident CTAs (the list look-back would wait on them)
    sv.set_options(ctas_per_sm=per)
    for lo, hi in [(2, 10**7 + 1), (10**11, 10**11 + 3 * 10**7)]:
        lst, n = sv.primes(lo, hi)
        assert np.array_equal(lst[:n], oracle.primes(lo, hi))
        assert sv.stats(lo, hi) == oracle.stats(lo, hi)


def test_stream_switch_orders_work():
    torch = pytest.importorskip("torch")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    dev = torch.device("cuda", 0)
    from paper_1205_4883_b200 import dist as D
    lo, hi = 2, 10**10 + 1
    base = D.alloc_base(sv.base_capacity(10**5), dev)
    torch.cuda.synchronize()
    res = [torch.zeros(2, dtype=torch.int64, device=dev) for _ in range(6)]
    try:
        for k in range(6):  # back-to-back async launches, alternating streams
            sv.set_stream(s1 if k % 2 == 0 else s2)
            sv.stats_base_async(lo, hi, base.primes, base.recips, base.nbase, res[k])
        torch.cuda.synchronize()
    finally:
        sv.set_stream(None)
    for r in res:
        assert [int(x) & ((1 << 64) - 1) for x in r.tolist()] == [455052511, 2220822432581729238]


def test_k0_conflict_free_atomic_rate():
    lanes, ghz = sv.debug_k0()
    assert 28.0 < lanes <= 32.5, lanes
    assert 0.5 < ghz < 2.2, ghz


@pytest.mark.parametrize("seg_kb", [16, 32, 208])
def test_f3_cluster_pair_kernel_parity(seg_kb):
    """F3 (PAPER.md:137-161 re-expressed): the cluster-pair
    kernel -- two CTAs per super-segment, the large primes walked once over
    both halves, the partner half marked through distributed shared memory --
    gives the oracle's results (odd and even segment counts, ragged ends,
    first segments below p^2).  It is a measured A/B variant (3-6x slower,
    profiles/r02_f3_cluster_ab.jsonl), not the product path."""
    sv.set_options(segment_kb=seg_kb)
    sv.debug_set_flags(64)  # FLAG_CLUSTER
    for lo, hi in [(2, 10**8 + 1), (10**12 + 1, 10**12 + 3 * 10**7 + 7), (999_999_999_989, 1_000_040_000_000),
                   (0, 5000), (3, 10**6)]:
        assert sv.stats(lo, hi) == oracle.stats(lo, hi), (lo, hi, seg_kb)
    if seg_kb == 208:
        assert sv.stats(*inputs.CONFIG3) == (455052511, 2220822432581729238)
