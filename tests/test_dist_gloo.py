"""Multi-process (world_size 2, gloo, CPU) tests of the multi-GPU host logic
in paper_1205_4883_b200/dist.py: block partition, the packed base-prime
broadcast, the u64-as-int64 all-reduce, the LPT batch assignment with its
all_gather reassembly, the F1 gather of per-rank bitmaps and lists with
the decomposable bitmap checksum, and the F4 fused all-reduce's protocol
(csrc/peer.cuh: slab slots, epochs, parity double buffering) between real
processes on shared memory.  The per-rank compute is injected (a CPU stand-in
built on the oracle) because this container has no GPU; the CUDA backend is
the default in the product path and is exercised by the -m gpu tests."""
import os
import socket
import tempfile
import time

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import inputs
import oracle
from paper_1205_4883_b200 import dist as D

MASK64 = (1 << 64) - 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleBackend:
    """CPU stand-in for CudaBackend (test only): base primes from the
    oracle, packed the same way; stats from the oracle, written into the
    int64[2] result tensor as two's-complement u64."""

    def base_capacity(self, r):
        return max(32, len(oracle.base_primes(r)) + 8)

    def base_primes(self, r, base):
        pr = oracle.base_primes(r)
        odd = pr[pr > 2].astype(np.int64)
        base.primes[: odd.size] = torch.from_numpy(odd.astype(np.int32))
        base.nbase[0] = int(odd.size)

    def stats(self, a, b, base, result):
        # the rank must see the broadcast primes: check them against its own copy
        n = int(base.nbase[0])
        got = base.primes[:n].numpy().astype(np.int64)
        r = D.isqrt(b - 1) if b >= 2 else 0
        mine = oracle.base_primes(r)
        mine = mine[mine > 2]
        assert np.array_equal(got[: mine.size], mine), "broadcast base primes differ"
        c, s = oracle.stats(a, b, 1)
        result[0] = D.u64_to_i64(c)
        result[1] = D.u64_to_i64(s)

    def stats_base(self, a, b, base, result, allreduce=False):
        # the fused launch: this block's own base primes, then its stats
        self.base_primes(D.isqrt(b - 1) if b >= 2 else 0, base)
        (self.stats_allreduce if allreduce else self.stats)(a, b, base, result)


class OracleGatherBackend:
    """CPU stand-in for CudaGatherBackend (test only)."""

    def bitmap(self, a, b, device):
        bm, _, _ = oracle.bitmap(a, b)
        return torch.from_numpy(bm.view(np.int32).copy())

    def primes(self, a, b, device):
        return torch.from_numpy(oracle.primes(a, b).view(np.int64).copy())


class SlabSimBackend(OracleBackend):
    """CPU stand-in for the F4 fused all-reduce (test only): each rank's slab
    is a shared file mapping (its path is the "IPC handle"), and
    stats_allreduce follows csrc/peer.cuh step by step -- publish (count,
    sum) then the epoch into slot [e & 1][rank] of every slab, then wait for
    epoch e in every slot [e & 1][*] of its own slab and sum.  x86 stores are
    ordered, standing in for the kernel's release/acquire pair."""

    def __init__(self, tmpdir, rank):
        self.path = os.path.join(tmpdir, f"slab{rank}")
        np.zeros(512, dtype=np.uint64).tofile(self.path)
        self.views = None

    def peer_handle(self):
        return self.path.encode().ljust(64, b"\0")

    def peer_attach(self, handles, rank, timeout_ms):
        self.handles = handles
        self.rank, self.world, self.epoch = rank, len(handles), 0
        self.views = [np.memmap(h.rstrip(b"\0").decode(), dtype=np.uint64, mode="r+", shape=(512,))
                      for h in handles]

    def peer_detach(self):
        self.views = None

    def stats_allreduce(self, a, b, base, result):
        self.epoch += 1
        e = self.epoch
        c, s = oracle.stats(a, b, 1)
        par = (e & 1) * 64
        for v in self.views:
            i = 4 * (par + self.rank)
            v[i], v[i + 1] = c, s
            v[i + 2] = e
        mine = self.views[self.rank]
        tc = ts = 0
        for q in range(self.world):
            i = 4 * (par + q)
            t0 = time.time()
            while int(mine[i + 2]) != e:
                assert time.time() - t0 < 60, "peer never published"
                time.sleep(0)
            tc += int(mine[i])
            ts += int(mine[i + 1])
        result[0] = D.u64_to_i64(tc & MASK64)
        result[1] = D.u64_to_i64(ts & MASK64)


def _worker(rank, world, port, q, tmpdir=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        be = OracleBackend()
        cpu = torch.device("cpu")
        for lo, hi in [(2, 10**6 + 1), (10**12, 10**12 + 3 * 10**5), (0, 0), (5, 6),
                       (2**63 // 2**16, 2**63 // 2**16 + 10**5)]:
            out[(lo, hi)] = D.stats(lo, hi, backend=be, device=cpu)
            out[("per-rank base", lo, hi)] = D.stats(lo, hi, broadcast=False, backend=be, device=cpu)
            out[("cost split", lo, hi)] = D.stats(lo, hi, broadcast=False, backend=be, device=cpu, split="cost")
        lo5, hi5 = inputs.config5_intervals(64)
        c, s = D.batch(lo5, hi5, batch_fn=lambda a, b: oracle.batch(a, b, 1), device=cpu)
        out["batch"] = (c.tolist(), s.tolist())
        # u64 wrap across the all-reduce: two values whose sum wraps mod 2^64
        t = torch.tensor([D.u64_to_i64((1 << 64) - 5 if rank == 0 else 9)], dtype=torch.int64)
        dist.all_reduce(t)
        out["wrap"] = D.i64_to_u64(int(t.item()))
        gb = OracleGatherBackend()
        for lo, hi in [(2, 2 * 10**5 + 1), (10**9 + 7, 10**9 + 3 * 10**5), (3, 3), (10, 12)]:
            words, cs = D.gather_bitmap(lo, hi, backend=gb, device=cpu)
            lst = D.gather_primes(lo, hi, backend=gb, device=cpu)
            out[("F1", lo, hi)] = (words.numpy().view(np.uint32).tolist(), cs, lst.numpy().tolist())
        # F4: the fused all-reduce protocol between the two processes; random
        # per-rank delays let one rank run ahead into the other parity
        sim = SlabSimBackend(tmpdir, rank)
        D.attach_peers(backend=sim)
        out["handles"] = [h.rstrip(b"\0").decode() for h in sim.handles]
        rng = np.random.default_rng(rank + 7)
        for k in range(40):
            lo, hi = 10**6 * k + k, 10**6 * k + 6 * 10**4 + 3 * k
            if rng.random() < 0.5:
                time.sleep(rng.random() * 0.02)
            # odd k: the per-rank fused base-prime launch with the fused all-reduce
            out[("F4", lo, hi)] = D.stats(lo, hi, broadcast=k % 2 == 0, backend=sim, device=cpu)
        out[("F4", 9, 9)] = D.stats(9, 9, backend=sim, device=cpu)
        out["epochs"] = sim.epoch
        D.detach_peers(backend=sim)
        # a rank whose attach fails still completes the collectives; the
        # ranks agree (MIN) and fall back to the NCCL/gloo all-reduce
        class FailingSim(SlabSimBackend):
            def peer_attach(self, handles, rank, timeout_ms):
                raise RuntimeError("simulated IPC failure")
        fb = FailingSim(tmpdir, rank) if rank == 1 else SlabSimBackend(tmpdir, rank)
        ok = D.attach_peers(backend=fb)
        t = torch.tensor([1 if ok else 0], dtype=torch.int32)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        # attach_peers itself agrees: every rank reports the failure and the
        # default of stats(fused=None) is NCCL/gloo everywhere
        out["attach_ok"] = (bool(ok), bool(t.item()), id(None) in D._ATTACHED, fb.views is None)
        D.detach_peers(backend=fb)
        out["after_fail"] = D.stats(2, 10**5 + 1, backend=be, device=cpu)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_stats_batch_and_wrap():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    tmpdir = tempfile.mkdtemp(prefix="slabs")
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q, tmpdir)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0]["attach_ok"] == (False, False, False, True)
    assert res[1]["attach_ok"] == (False, False, False, True)
    assert res[0]["after_fail"] == res[1]["after_fail"] == oracle.stats(2, 10**5 + 1)
    for rr in res.values():
        del rr["attach_ok"]
    assert res[0] == res[1]
    r = res[0]
    for key, val in r.items():
        if isinstance(key, tuple) and key[0] == "F1":
            _, lo, hi = key
            words, cs, lst = val
            obm, _, _ = oracle.bitmap(lo, hi)
            assert words == obm.tolist(), key                     # gathered bitmap == whole bitmap
            assert cs == D.bitmap_checksum(obm), key              # all-reduced decomposable checksum
            assert lst == oracle.primes(lo, hi).tolist(), key     # gathered list == whole list
        elif isinstance(key, tuple) and key[0] in ("F4", "per-rank base", "cost split"):
            assert val == oracle.stats(*key[1:]), key          # one reduction, whole range
        elif isinstance(key, tuple):
            assert val == oracle.stats(*key), key
    assert r["handles"] == [os.path.join(tmpdir, "slab0"), os.path.join(tmpdir, "slab1")]
    assert r["epochs"] == 41
    lo5, hi5 = inputs.config5_intervals(64)
    oc, os_ = oracle.batch(lo5, hi5)
    assert r["batch"] == (oc.tolist(), os_.tolist())
    assert r["wrap"] == 4


@pytest.mark.parametrize("split", ["equal", "cost"])
@pytest.mark.parametrize("G", [1, 2, 3, 4, 8, 13])
def test_block_partition_tiles_range(G, split):
    for lo, hi in [(2, 10**10 + 1), (0, 1), (0, 0), (7, 7 + 64 * 5 + 3), (10**12, 10**12 + 10**10),
                   (123, 124), (1, 64 * 3)]:
        blocks = [D.block_of(lo, hi, g, G, split) for g in range(G)]
        assert blocks[0][0] == lo and blocks[-1][1] == hi
        for (a0, b0), (a1, b1) in zip(blocks, blocks[1:]):
            assert b0 == a1 and a0 <= b0
        o0 = lo | 1
        for a, _ in blocks[1:]:
            if lo < a < hi:
                assert (a - o0) % 64 == 0 and a % 2 == 1  # word-aligned odd boundary


def test_block_partition_matches_survey_g2():
    # config 3 at G=2 splits at 5000000003
    assert D.block_of(2, 10**10 + 1, 0, 2) == (2, 5000000003)
    assert D.block_of(2, 10**10 + 1, 1, 2) == (5000000003, 10**10 + 1)


def test_cost_split_shape():
    """split="cost": the low blocks of [2, 10^10] are longer than the high
    ones (work per integer grows like ln ln x), monotonically; far from 0
    (config 4) the blocks are equal to within 0.1 %; an unknown split raises."""
    lo, hi = 2, 10**10 + 1
    for G in (2, 4, 8):
        w = [b - a for a, b in (D.block_of(lo, hi, g, G, "cost") for g in range(G))]
        assert all(x > y for x, y in zip(w, w[1:])) and sum(w) == hi - lo
        assert 1.0 < w[0] / w[-1] < 1.35
    lo, hi = 10**12, 10**12 + 10**10
    w = [b - a for a, b in (D.block_of(lo, hi, g, 8, "cost") for g in range(8))]
    assert max(w) / min(w) < 1.001
    with pytest.raises(ValueError):
        D.block_of(2, 100, 0, 2, "lpt")


@pytest.mark.parametrize("split", ["equal", "cost"])
def test_block_additivity_small(split):
    lo, hi = (10**9, 10**9 + 4 * 10**6 + 7) if split == "equal" else (2, 4 * 10**6 + 7)
    tot_c, tot_s = 0, 0
    for g in range(5):
        a, b = D.block_of(lo, hi, g, 5, split)
        c, s = oracle.stats(a, b, 1)
        tot_c += c
        tot_s = (tot_s + s) & MASK64
    assert (tot_c, tot_s) == oracle.stats(lo, hi)


def test_lpt_assignment_properties():
    lo, hi = inputs.config5_intervals()
    cost = D.batch_cost(lo, hi)
    for world in (1, 2, 8):
        parts = D.lpt_assign(cost, world)
        allidx = np.sort(np.concatenate(parts))
        assert np.array_equal(allidx, np.arange(lo.size))
        loads = np.array([cost[p].sum() for p in parts])
        # LPT is within 4/3 of optimal; here the spread is tiny
        assert loads.max() <= loads.mean() * 1.05 + cost.max()


def test_prime_count_bound_and_device_checksum():
    """F1 helpers: the list-capacity bound holds (it sizes gather_primes'
    single list-mode pass), and the on-device decomposable checksum equals
    the host one, wrap-around included."""
    for lo, hi in [(0, 0), (0, 3), (2, 3), (0, 100), (2, 10**6), (10**12, 10**12 + 10**6),
                   (10**9, 10**9 + 7), (999_999_999_989, 1_000_000_000_039)]:
        assert D.prime_count_bound(lo, hi) >= oracle.stats(lo, hi)[0], (lo, hi)
    for x in (10**7, 10**8, 10**9):  # pi(x) from known_pi.txt
        pi = {10**7: 664579, 10**8: 5761455, 10**9: 50847534}[x]
        assert D.prime_count_bound(0, x + 1) >= pi
    rng = np.random.default_rng(5)
    w = rng.integers(0, 2**32, size=100003, dtype=np.uint64).astype(np.uint32)
    t = torch.from_numpy(w.view(np.int32).copy())
    for first in (0, 7, 2**40):
        assert D.bitmap_checksum_tensor(t, first) == D.bitmap_checksum(w, first)
