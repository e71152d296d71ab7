"""F4 across a real process boundary on one B200: two processes (ranks 0 and
1 of a gloo group), each with its own CUDA context on device 0, exchange
their slabs' CUDA IPC handles (dist.attach_peers: all_gather + MIN
agreement) and run the fused all-reduce of the production step
(sieve_stats_base_async with allreduce: base primes, sieve and the peer
all-reduce in ONE cooperative launch) on their config-3 blocks.

The kernels never wait on one another (B200_PROFILING.md: kernels of
different processes on one GPU are not guaranteed to run concurrently): in
each epoch one rank first PUBLISHES its share (sieve_peer_publish_async, no
wait), the ranks meet at a host barrier, then the other rank's fused launch
finds that share already in its slab.  The roles alternate, so both ranks
run the fused kernel, both slab parities are used, and every P2P store and
acquire load crosses the process boundary through the IPC mapping."""
import os
import socket

import pytest

pytestmark = pytest.mark.gpu
MASK64 = (1 << 64) - 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    import oracle
    import paper_1205_4883_b200 as sv
    from paper_1205_4883_b200 import dist as D

    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {"rank": rank, "results": [], "epochs": []}
    try:
        torch.cuda.set_device(0)
        sv.set_device(0)
        dev = torch.device("cuda", 0)
        st = torch.cuda.current_stream()
        sv.set_stream(st)
        ok = D.attach_peers(timeout_ms=3000)
        out["attached"] = ok
        if ok:
            cases = [(2, 10**10 + 1), (10**12, 10**12 + 10**9), (2, 10**8 + 1), (10**9, 10**9 + 7)]
            for k, (lo, hi) in enumerate(cases * 2):
                a, b = D.block_of(lo, hi, rank, world)
                runner = k % world  # this epoch's fused rank; the others publish first
                r = D.isqrt(b - 1) if b >= 2 else 0
                base = D.alloc_base(sv.base_capacity(max(r, 3)), dev)
                res = torch.zeros(2, dtype=torch.int64, device=dev)
                if rank != runner:
                    c, s = oracle.stats(a, b)
                    sv.peer_publish_async(c, s)
                    torch.cuda.synchronize()
                dist.barrier()
                if rank == runner:
                    sv.stats_base_async(a, b, base.primes, base.recips, base.nbase, res, allreduce=True)
                    torch.cuda.synchronize()
                    got = tuple(int(x) & MASK64 for x in res.cpu().tolist())
                    out["results"].append(((lo, hi), got, oracle.stats(lo, hi)))
                out["epochs"].append(sv.peer_epoch())
                dist.barrier()
            D.detach_peers()
    except Exception as e:  # noqa: BLE001
        out["error"] = repr(e)
    finally:
        q.put(out)
        dist.destroy_process_group()


def test_two_processes_one_gpu_fused_allreduce():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    outs = {}
    for _ in ps:
        o = q.get(timeout=600)
        outs[o["rank"]] = o
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    for r in (0, 1):
        assert "error" not in outs[r], outs[r]["error"]
        assert outs[r]["attached"] is True
        assert outs[r]["epochs"] == list(range(1, 9))
        assert len(outs[r]["results"]) == 4  # 8 epochs, the fused launch alternating
        for rng, got, want in outs[r]["results"]:
            assert got == want, (r, rng)
