"""Multi-GPU orchestration (step A9 and the multi-GPU half of A10).

One process per GPU (torchrun), torch.distributed process groups over NCCL
for the plumbing -- the paper's Fig. 6 flow (partition ->
distribute -> sieve -> gather, read as SPEC.md:10/271/296) re-expressed for
one NVSwitch box:

  partition : equal contiguous blocks of the odd-only word grid
              (reading R10; "average divide data into nodes")
  distribute: rank 0 computes the base primes (K1) and broadcasts ONE packed
              buffer [recips | primes | nbase] (PAPER.md:19's FIFO buffer of
              data from other nodes becomes a single NCCL broadcast); or
              (broadcast=False) every rank computes its own block's base
              primes inside its sieve launch (fused A2, no collective)
  sieve     : every rank runs the segmented sieve on its block (CUDA, C ABI)
  gather    : one all-reduce of u64[2] = {count, sum}; two's-complement int64
              addition is bit-identical to u64 addition mod 2^64.  With
              attach_peers() done (F4) that all-reduce happens INSIDE the
              sieve kernel: its last CTA writes the rank's result into every
              peer's slab over NVLink and sums its own (csrc/peer.cuh) --
              no NCCL launch on the count path.

The compute callables default to the CUDA library; tests may inject others
to exercise this host logic with the gloo backend on CPU.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

MASK64 = (1 << 64) - 1


def isqrt(x: int) -> int:
    return math.isqrt(x) if x > 0 else 0


# Cost-weighted split (split="cost"): marking work per integer near x grows
# like sum_{w < p <= sqrt(x)} 1/p ~ ln ln x + const (Mertens), so equal blocks
# of [2, 10^10] leave the top rank ~19 % more kernel time than rank 0 at G = 8
# (profiles/r02_rank_blocks.txt).  COST_KAPPA is the constant of the density
# ln ln x - kappa fitted to those block times on B200 (default segment size,
# wheel 31); only the ratio of the densities at the two ends matters.
COST_KAPPA = 2.35
_COST_FLOOR = 0.05
_COST_PANELS = 4096


def _cost_edges(lo: int, hi: int, world: int, words: int) -> list[int]:
    """Word indices k_1 <= ... <= k_{world-1} cutting [lo, hi) into `world`
    pieces of equal modelled cost (midpoint rule on _COST_PANELS panels,
    inverted by linear interpolation; the same on every rank)."""
    n = _COST_PANELS
    x = lo + (np.arange(n, dtype=np.float64) + 0.5) * ((hi - lo) / n)
    dens = np.maximum(np.log(np.log(np.maximum(x, 16.0))) - COST_KAPPA, _COST_FLOOR)
    cum = np.concatenate([[0.0], np.cumsum(dens)])
    cum /= cum[-1]
    pos = np.interp(np.arange(1, world) / world, cum, np.arange(n + 1) / n)
    ks = [min(words, max(0, int(round(float(f) * words)))) for f in pos]
    for i in range(1, len(ks)):
        ks[i] = max(ks[i], ks[i - 1])
    return ks


def block_of(lo: int, hi: int, rank: int, world: int, split: str = "equal") -> tuple[int, int]:
    """Step A1 across GPUs (reading R10): block `rank` of `world` contiguous
    blocks of [lo, hi) on the odd-only word grid.  split="equal" (default,
    PAPER.md:19 "average divide data into nodes", config 3): boundaries at
    o0 + 64*floor(k*words/world) (o0 = lo|1), clipped to [lo, hi].
    split="cost": boundaries at words of equal modelled marking cost
    (_cost_edges; the load balance PAPER.md:105-110 asks for, applied across
    GPUs).  Either way every block's bitmap starts on a 32-bit word of the
    whole range's bitmap and the blocks tile [lo, hi) exactly."""
    if split not in ("equal", "cost"):
        raise ValueError(f"split must be 'equal' or 'cost', not {split!r}")
    if hi <= lo:
        return lo, hi
    o0 = lo | 1
    words = (hi // 2 - lo // 2 + 31) // 32
    cost = _cost_edges(lo, hi, world, words) if split == "cost" and world > 1 else None

    def edge(k: int) -> int:
        if k <= 0:
            return lo
        if k >= world:
            return hi
        kw = cost[k - 1] if cost is not None else (k * words) // world
        return min(hi, o0 + 64 * kw) if kw > 0 else lo

    return edge(rank), edge(rank + 1)


class _LibraryStreamOrder:
    """Orders the library's stream (sieve_set_stream, or its own) after
    torch's current stream on entry -- the buffers were allocated/filled
    there -- and torch's current stream after the library's on exit, so the
    caller can read the result on its stream.  A no-op when they coincide."""

    def __enter__(self):
        import torch
        import paper_1205_4883_b200 as sv
        self.cur = torch.cuda.current_stream()
        h = sv.get_stream()
        self.lib = None if h in (0, self.cur.cuda_stream) else torch.cuda.ExternalStream(h)
        if self.lib is not None:
            self.lib.wait_stream(self.cur)
        return self

    def __exit__(self, *exc):
        if self.lib is not None:
            self.cur.wait_stream(self.lib)
        return False


class CudaBackend:
    """The product compute path: the C-ABI library on the current device."""

    def base_capacity(self, r):
        import paper_1205_4883_b200 as sv
        return sv.base_capacity(r)

    def base_primes(self, r, base):
        import paper_1205_4883_b200 as sv
        with _LibraryStreamOrder():
            sv.base_primes_async(r, base.primes, base.recips, base.nbase)

    def stats(self, a, b, base, result):
        import paper_1205_4883_b200 as sv
        with _LibraryStreamOrder():
            sv.stats_async(a, b, base.primes, base.recips, base.nbase, result)

    def stats_allreduce(self, a, b, base, result):
        import paper_1205_4883_b200 as sv
        with _LibraryStreamOrder():
            sv.stats_allreduce_async(a, b, base.primes, base.recips, base.nbase, result)

    def stats_base(self, a, b, base, result, allreduce=False):
        """A2 (base primes <= isqrt(b-1), into base) and the block's count/sum
        in one kernel launch; allreduce: the fused peer all-reduce too."""
        import paper_1205_4883_b200 as sv
        with _LibraryStreamOrder():
            sv.stats_base_async(a, b, base.primes, base.recips, base.nbase, result, allreduce)

    def peer_handle(self) -> bytes:
        import paper_1205_4883_b200 as sv
        return sv.peer_slab_handle()

    def peer_attach(self, handles, rank, timeout_ms):
        import paper_1205_4883_b200 as sv
        sv.peer_attach(handles, rank, timeout_ms)

    def peer_detach(self):
        import paper_1205_4883_b200 as sv
        sv.peer_detach()


# groups attached for the fused all-reduce (F4): id(group) -> world
_ATTACHED: dict = {}
SENTINEL = (1 << 64) - 1


def attach_peers(group=None, timeout_ms: int = 10000, backend=None) -> bool:
    """F4 setup, collective over `group`: every rank exports its slab's CUDA
    IPC handle, the handles are all-gathered over the host in rank order and
    every rank opens its peers' slabs; a barrier makes every slab zeroed
    before anyone's first fused launch.  Later stats(..., fused=True) calls
    on this group all-reduce inside the sieve kernel.  Every rank takes part
    in every collective even when its own export or attach fails, so a local
    failure cannot leave the others waiting, and the ranks then agree: the
    per-rank outcomes are combined with a MIN all-reduce, and if any rank
    failed every rank detaches -- so the default of stats(fused=None) is the
    same on every rank (all fused or all NCCL).  Returns the agreed outcome."""
    import torch.distributed as dist
    be = backend if backend is not None else CudaBackend()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    ok = True
    try:
        mine = be.peer_handle()
    except Exception:  # noqa: BLE001 -- reported through the return value
        mine, ok = b"", False
    if world > 1:
        handles = [None] * world
        dist.all_gather_object(handles, mine, group=group)
    else:
        handles = [mine]
    if ok and all(isinstance(h, bytes) and len(h) > 0 for h in handles):
        try:
            be.peer_attach(handles, rank, timeout_ms)
        except Exception:  # noqa: BLE001
            ok = False
    else:
        ok = False
    if world > 1:
        dist.barrier(group=group)
        ok = _agree_all(ok, group)
    if ok:
        _ATTACHED[id(group)] = world
    else:
        try:
            be.peer_detach()
        except Exception:  # noqa: BLE001 -- nothing attached on this rank
            pass
    return ok


def _agree_all(ok: bool, group=None) -> bool:
    """True iff every rank of `group` passed ok=True (MIN all-reduce over the
    group's backend: a CPU tensor for gloo, a CUDA tensor for NCCL)."""
    import torch
    import torch.distributed as dist
    dev = torch.device("cpu")
    if dist.get_backend(group) == "nccl":
        dev = torch.device("cuda", torch.cuda.current_device())
    t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return bool(t.item())


def u64_to_i64(x: int) -> int:
    x &= MASK64
    return x - (1 << 64) if x >= (1 << 63) else x


def i64_to_u64(x: int) -> int:
    return x & MASK64


@dataclass
class BaseBuffers:
    """Views into one packed device buffer: recips (u64) | primes (u32) | nbase."""
    packed: "object"
    recips: "object"
    primes: "object"
    nbase: "object"
    cap: int


def alloc_base(cap: int, device) -> BaseBuffers:
    import torch
    n32 = 2 * cap + cap + 1
    packed = torch.zeros(n32, dtype=torch.int32, device=device)
    recips = packed[: 2 * cap].view(torch.int64)
    primes = packed[2 * cap: 3 * cap]
    nbase = packed[3 * cap: 3 * cap + 1]
    return BaseBuffers(packed, recips, primes, nbase, cap)


def detach_peers(group=None, backend=None) -> None:
    """Undo attach_peers: later stats() calls on `group` use NCCL again."""
    _ATTACHED.pop(id(group), None)
    be = backend if backend is not None else CudaBackend()
    be.peer_detach()


def stats(lo: int, hi: int, group=None, broadcast: bool = True, base: BaseBuffers | None = None,
          result=None, sync: bool = True, backend=None, device=None, fused: bool | None = None,
          split: str = "equal"):
    """pi-count and prime sum of [lo, hi) over all ranks of `group` (public
    multi-GPU API).  Returns (count, sum mod 2^64) on every rank when sync,
    else the device result tensor (int64[2], already all-reduced).
    fused (default: whether attach_peers(group) was done): the all-reduce
    runs inside the sieve kernel over peer memory (F4) instead of NCCL.
    split: "equal" blocks (config 3) or "cost"-weighted blocks (block_of)."""
    import torch
    import torch.distributed as dist

    be = backend if backend is not None else CudaBackend()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    r = isqrt(hi - 1) if hi >= 2 else 0
    if base is None:
        base = alloc_base(be.base_capacity(r), dev)
    if result is None:
        result = torch.zeros(2, dtype=torch.int64, device=dev)
    a, b = block_of(lo, hi, rank, world, split)
    if fused is None:
        fused = _ATTACHED.get(id(group)) == world
    if world > 1 and broadcast:
        # A9 distribute: rank 0 computes the base primes, one NCCL broadcast
        if rank == 0:
            be.base_primes(r, base)
        dist.broadcast(base.packed, src=0, group=group)
        (be.stats_allreduce if fused else be.stats)(a, b, base, result)
    else:
        # every rank computes its block's base primes inside its sieve launch
        be.stats_base(a, b, base, result, fused)
    if world > 1 and not fused:
        dist.all_reduce(result, op=dist.ReduceOp.SUM, group=group)
    if not sync:
        return result
    h = result.cpu().tolist()
    c, s = i64_to_u64(h[0]), i64_to_u64(h[1])
    if fused and c == SENTINEL:
        raise RuntimeError("fused all-reduce timed out waiting for a peer (sieve_peer_attach)")
    return c, s


# ---------------------------------------------------------------- batch / LPT
def batch_cost(lo: np.ndarray, hi: np.ndarray, seg_bits: int = 192 * 8192) -> np.ndarray:
    """Cost model of one interval (A10): odd slots to sieve plus one
    first-hit reduction per (segment, base prime).  pi(sqrt(hi)) is
    approximated by sqrt(hi)/ln(sqrt(hi)) -- only the ranking matters."""
    lo = lo.astype(np.float64)
    hi = hi.astype(np.float64)
    width = np.maximum(hi - lo, 0.0)
    rt = np.sqrt(np.maximum(hi, 4.0))
    nprimes = rt / np.log(rt)
    nseg = np.ceil(width / 2.0 / seg_bits)
    return 0.6 * width / 2.0 + 20.0 * nseg * nprimes


def lpt_assign(cost: np.ndarray, world: int) -> list[np.ndarray]:
    """Longest-processing-time-first: intervals in decreasing cost, each to
    the currently least-loaded rank.  Deterministic (stable sort, ties to the
    lowest rank)."""
    order = np.argsort(-cost, kind="stable")
    load = np.zeros(world)
    parts: list[list[int]] = [[] for _ in range(world)]
    for i in order:
        k = int(np.argmin(load))
        parts[k].append(int(i))
        load[k] += cost[i]
    return [np.array(sorted(p), dtype=np.int64) for p in parts]


def batch(lo, hi, group=None, batch_fn=None, device=None):
    """Per-interval (count, sum) over all ranks: LPT assignment, local batch
    on each rank, all_gather of the padded per-rank results, reassembly in
    input order.  Every rank returns the full arrays."""
    import torch
    import torch.distributed as dist

    lo = np.ascontiguousarray(lo, dtype=np.uint64)
    hi = np.ascontiguousarray(hi, dtype=np.uint64)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if batch_fn is None:
        import paper_1205_4883_b200 as sv
        batch_fn = sv.batch
    parts = lpt_assign(batch_cost(lo, hi), world)
    mine = parts[rank]
    c, s = batch_fn(lo[mine], hi[mine])
    if world == 1:
        return np.asarray(c, dtype=np.uint64), np.asarray(s, dtype=np.uint64)
    width = max(len(p) for p in parts)
    dev = device if device is not None else (torch.device("cuda", torch.cuda.current_device())
                                             if torch.cuda.is_available() else torch.device("cpu"))
    loc = np.zeros((width, 2), dtype=np.uint64)
    loc[: len(mine), 0] = c
    loc[: len(mine), 1] = s
    t = torch.from_numpy(loc.view(np.int64)).to(dev)
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t, group=group)
    count = np.zeros(lo.size, dtype=np.uint64)
    ssum = np.zeros(lo.size, dtype=np.uint64)
    for k in range(world):
        arr = outs[k].cpu().numpy().view(np.uint64)
        idx = parts[k]
        count[idx] = arr[: len(idx), 0]
        ssum[idx] = arr[: len(idx), 1]
    return count, ssum


# ---------------------------------------------------------------- F1: gather
# SURVEY.md 8(f) F1, the "gather" step of the paper's flow (PAPER.md:163-169
# via SPEC.md:296: results gathered in node order): the per-GPU bitmap and
# list slices assembled on every rank.  The blocks of block_of() start on
# 32-bit words of the whole range's odd-only grid, so block g's bitmap is
# exactly words [w_g, w_{g+1}) of the whole bitmap, and block g's primes
# follow block g-1's.  NCCL all_gather wants equal sizes: slices are padded
# to the largest and trimmed after.  A decomposable checksum of the bitmap,
# sum_w (w+1) word_w mod 2^64 over global word indices, is all-reduced so
# every rank can check the gathered copy without a sequential FNV.

def _block_words(lo: int, hi: int, world: int) -> list[tuple[int, int]]:
    """(first global word, word count) of every block's bitmap."""
    o0 = lo | 1
    out = []
    for g in range(world):
        a, b = block_of(lo, hi, g, world)
        w0 = ((a | 1) - o0) // 64 if b > a else 0
        nbits = b // 2 - a // 2 if b > a else 0
        out.append((w0, (nbits + 31) // 32))
    return out


def bitmap_checksum(words: np.ndarray, first_word: int = 0) -> int:
    """sum_w (first_word + w + 1) * words[w] mod 2^64 (host, exact)."""
    w = np.asarray(words).astype(np.uint64)
    idx = np.arange(first_word + 1, first_word + 1 + w.size, dtype=np.uint64)
    return int(np.sum(idx * w, dtype=np.uint64))


def bitmap_checksum_tensor(words, first_word: int = 0) -> int:
    """bitmap_checksum on the tensor's own device (no host copy of the
    bitmap): int64 products and sums wrap mod 2^64 like u64 arithmetic; the
    uint32 words are zero-extended from their int32 view."""
    import torch
    w = words.to(torch.int64) & 0xFFFFFFFF
    idx = torch.arange(first_word + 1, first_word + 1 + w.numel(), dtype=torch.int64, device=w.device)
    return i64_to_u64(int((idx * w).sum().item()))


class CudaGatherBackend:
    """The product compute path for F1: per-rank bitmap / list of a block on
    the current device (C ABI), returned as CUDA tensors."""

    def bitmap(self, a, b, device):
        import torch
        import paper_1205_4883_b200 as sv
        n = sv.bitmap_words(a, b)
        out = torch.zeros(max(n, 1), dtype=torch.int32, device=device)
        if n:
            with _LibraryStreamOrder():
                sv.bitmap(a, b, out=out)
        return out[:n]

    def primes(self, a, b, device):
        """ONE list-mode sieve of [a, b): the output is sized by an upper
        bound on the count instead of a count pass, then trimmed."""
        import torch
        import paper_1205_4883_b200 as sv
        cap = prime_count_bound(a, b)
        out = torch.zeros(max(cap, 1), dtype=torch.int64, device=device)
        n = 0
        if cap:
            with _LibraryStreamOrder():
                _, n = sv.primes(a, b, cap=cap, out=out)
        if n > cap:  # cannot happen (the bound holds for every interval)
            raise RuntimeError(f"prime_count_bound({a}, {b}) = {cap} < {n}")
        return out[:n]


def prime_count_bound(a: int, b: int) -> int:
    """An upper bound on the number of primes in [a, b), for sizing a list
    output without a count pass.  Candidates are 2 and 3 plus the integers
    coprime to 6, at most (b - a) / 3 + 2 of them; for long intervals the
    Brun-Titchmarsh inequality pi(x + y) - pi(x) <= 2 y / ln y (Montgomery
    and Vaughan, y > 1) is much tighter.  The smaller of the two, plus 2."""
    y = max(b - a, 0)
    cand = y // 3 + 2
    if y > 1:
        cand = min(cand, int(2 * y / math.log(y)) + 2)
    return cand


def _gather_padded(t, group, world):
    """all_gather of 1-D tensors of different lengths (padded to the max)."""
    import torch
    import torch.distributed as dist
    n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    ns = [int(x.item()) for x in ns]
    m = max(ns) if ns else 0
    pad = torch.zeros(max(m, 1), dtype=t.dtype, device=t.device)
    pad[: t.numel()] = t
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return torch.cat([o[:k] for o, k in zip(outs, ns)]) if world else t


def gather_bitmap(lo: int, hi: int, group=None, backend=None, device=None):
    """The whole odd-only bitmap of [lo, hi) (reading R5) on every rank:
    each rank sieves its block, the slices are all-gathered in block order.
    Returns (words as int32 tensor, checksum) where checksum is the
    all-reduced decomposable checksum of the slices (== bitmap_checksum of
    the gathered words)."""
    import torch
    import torch.distributed as dist
    be = backend if backend is not None else CudaGatherBackend()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    a, b = block_of(lo, hi, rank, world)
    mine = be.bitmap(a, b, dev)
    w0 = _block_words(lo, hi, world)[rank][0]
    part = bitmap_checksum_tensor(mine, w0)
    cs = torch.tensor([u64_to_i64(part)], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(cs, op=dist.ReduceOp.SUM, group=group)
        full = _gather_padded(mine, group, world)
    else:
        full = mine
    return full, i64_to_u64(int(cs.item()))


def gather_primes(lo: int, hi: int, group=None, backend=None, device=None):
    """The whole ascending prime list of [lo, hi) on every rank: per-rank
    block lists all-gathered in block order (block g's primes follow block
    g-1's).  Returns an int64 tensor."""
    import torch
    import torch.distributed as dist
    be = backend if backend is not None else CudaGatherBackend()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    a, b = block_of(lo, hi, rank, world)
    mine = be.primes(a, b, dev)
    return _gather_padded(mine, group, world) if world > 1 else mine
