"""F4: the all-reduce of (count, sum) fused into the sieve
kernel over peer memory (csrc/peer.cuh), on one B200.  A second GPU is not
available, so the peer side of world = 2 is played by the test: it writes the
other rank's slot (its (count, sum) from the oracle and the launch's epoch)
into this rank's slab before the launch, and checks the slot this rank
published into the "peer" slab after it.  The protocol across real processes
is exercised on CPU in test_dist_gloo.py (same slot/epoch/parity logic on
shared memory)."""
import pytest
import torch

import oracle
import paper_1205_4883_b200 as sv
from paper_1205_4883_b200 import dist as D

pytestmark = pytest.mark.gpu
MASK64 = (1 << 64) - 1
SLOT = 4  # u64 per slot


def _i64(x):
    x &= MASK64
    return x - (1 << 64) if x >= (1 << 63) else x


def _u64(x):
    return int(x) & MASK64


@pytest.fixture
def dev():
    sv.set_device(0)
    yield torch.device("cuda", 0)
    D.detach_peers()
    sv.set_stream(None)


def _same_stream():
    """The test writes slabs on torch's stream: launch the library there too."""
    sv.set_stream(torch.cuda.current_stream())


def _base(hi, dev):
    r = D.isqrt(hi - 1)
    base = D.alloc_base(sv.base_capacity(r), dev)
    sv.base_primes_async(r, base.primes, base.recips, base.nbase)
    return base


def test_world1_self_attach(dev):
    """world = 1 through the IPC-handle path: the kernel publishes into its
    own slab and reads it back; both parities, several ranges.  The library
    keeps its own stream here: dist.stats orders it against torch's."""
    D.attach_peers()
    for k, (lo, hi) in enumerate([(2, 10**7 + 1), (10**12, 10**12 + 10**6), (5, 6), (0, 0),
                                  (2, 3), (10**10, 10**10 + 3 * 10**6 + 17)]):
        e0 = sv.peer_epoch()
        got = D.stats(lo, hi)
        assert sv.peer_epoch() == e0 + 1
        assert got == oracle.stats(lo, hi), (lo, hi)


@pytest.mark.parametrize("rank", [0, 1])
@pytest.mark.parametrize("lo,hi", [(2, 2 * 10**7 + 1), (10**11, 10**11 + 4 * 10**6 + 3),
                                   (2, 40), (7, 7)])
def test_world2_simulated_peer(dev, rank, lo, hi):
    _same_stream()
    own = torch.zeros(sv.PEER_SLAB_BYTES // 8, dtype=torch.int64, device=dev)
    other = torch.zeros_like(own)
    slabs = [own, other] if rank == 0 else [other, own]
    sv.peer_attach_ptrs(slabs, rank, timeout_ms=5000)
    base = _base(max(hi, 3), dev)
    res = torch.zeros(2, dtype=torch.int64, device=dev)
    want = oracle.stats(lo, hi)
    for it in range(3):  # epochs 1, 2, 3: both parities, slot reuse
        a, b = D.block_of(lo, hi, rank, 2)
        pa, pb = D.block_of(lo, hi, 1 - rank, 2)
        pc, ps = oracle.stats(pa, pb)
        e = sv.peer_epoch() + 1
        slot = SLOT * ((e & 1) * sv.MAX_PEERS + (1 - rank))
        own[slot: slot + 3] = torch.tensor([_i64(pc), _i64(ps), e], dtype=torch.int64)
        sv.stats_allreduce_async(a, b, base.primes, base.recips, base.nbase, res)
        torch.cuda.synchronize()
        assert (_u64(res[0]), _u64(res[1])) == want, (it, a, b)
        mc, ms = oracle.stats(a, b)
        mine = SLOT * ((e & 1) * sv.MAX_PEERS + rank)
        assert [_u64(v) for v in other[mine: mine + 3].tolist()] == [mc, ms, e]


def test_timeout_sentinel_then_recovery(dev):
    """A peer that never publishes: the kernel gives up after timeout_ms and
    writes the sentinel; the library (done ticket, stream) stays usable."""
    _same_stream()
    own = torch.zeros(sv.PEER_SLAB_BYTES // 8, dtype=torch.int64, device=dev)
    other = torch.zeros_like(own)
    sv.peer_attach_ptrs([own, other], 0, timeout_ms=100)
    base = _base(10**8, dev)
    res = torch.zeros(2, dtype=torch.int64, device=dev)
    sv.stats_allreduce_async(10**7, 10**8, base.primes, base.recips, base.nbase, res)
    torch.cuda.synchronize()
    assert [_u64(v) for v in res.tolist()] == [MASK64, MASK64]
    sv.peer_detach()
    with pytest.raises(sv.SieveError):
        sv.stats_allreduce_async(10**7, 10**8, base.primes, base.recips, base.nbase, res)
    assert sv.stats(10**7, 10**8) == oracle.stats(10**7, 10**8)
    D.attach_peers()
    assert D.stats(10**7, 10**8) == oracle.stats(10**7, 10**8)


def test_attach_validation(dev):
    own = torch.zeros(sv.PEER_SLAB_BYTES // 8, dtype=torch.int64, device=dev)
    for world, rank in [(0, 0), (2, 2), (65, 0), (1, -1)]:
        with pytest.raises(sv.SieveError):
            sv.peer_attach_ptrs([own] * world, rank)
    with pytest.raises(sv.SieveError):  # nothing attached
        res = torch.zeros(2, dtype=torch.int64, device=dev)
        sv.stats_allreduce_async(10, 100, own, own, own, res)


@pytest.mark.parametrize("rank", [0, 1])
@pytest.mark.parametrize("lo,hi", [(2, 10**9 + 1), (10**12, 10**12 + 6 * 10**6 + 1), (2, 30)])
def test_world2_simulated_peer_fused_base(dev, rank, lo, hi):
    """The N > 1 production step: base primes, sieve and all-reduce in one
    cooperative launch (sieve_stats_base_async with allreduce), the peer's
    slot written by the test as in test_world2_simulated_peer."""
    _same_stream()
    own = torch.zeros(sv.PEER_SLAB_BYTES // 8, dtype=torch.int64, device=dev)
    other = torch.zeros_like(own)
    slabs = [own, other] if rank == 0 else [other, own]
    sv.peer_attach_ptrs(slabs, rank, timeout_ms=5000)
    a, b = D.block_of(lo, hi, rank, 2)
    pa, pb = D.block_of(lo, hi, 1 - rank, 2)
    r = D.isqrt(hi - 1) if hi >= 2 else 0
    base = D.alloc_base(sv.base_capacity(r), dev)
    res = torch.zeros(2, dtype=torch.int64, device=dev)
    want = oracle.stats(lo, hi)
    pc, ps = oracle.stats(pa, pb)
    for it in range(2):
        e = sv.peer_epoch() + 1
        slot = SLOT * ((e & 1) * sv.MAX_PEERS + (1 - rank))
        own[slot: slot + 3] = torch.tensor([_i64(pc), _i64(ps), e], dtype=torch.int64)
        sv.stats_base_async(a, b, base.primes, base.recips, base.nbase, res, allreduce=True)
        torch.cuda.synchronize()
        assert (_u64(res[0]), _u64(res[1])) == want, (it, a, b)
