"""The NCCL side of A9/F1 on a real GPU: a one-rank NCCL process group on
device 0 (the box has one GPU) runs the production orchestration of
dist.py through real NCCL collectives -- the base-prime broadcast, the
(count, sum) all-reduce, the batch all_gather and the F1 gathers -- and the
fused peer path with its fallback agreement.  The N-rank logic itself is
covered on CPU (test_dist_gloo.py) and across processes on one GPU
(test_gpu_peer_xproc.py)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_single_rank_nccl_group_paths():
    import torch
    import torch.distributed as dist

    import inputs
    import oracle
    import paper_1205_4883_b200 as sv
    from paper_1205_4883_b200 import dist as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        assert dist.get_backend() == "nccl"
        for lo, hi in [inputs.CONFIG3, (10**12, 10**12 + 10**8), (5, 6), (2, 3)]:
            want = oracle.stats(lo, hi) if hi - lo < 10**9 else (455052511, 2220822432581729238)
            assert D.stats(lo, hi, broadcast=True, fused=False) == want, (lo, hi)   # NCCL broadcast + all_reduce
            assert D.stats(lo, hi, broadcast=False, fused=False) == want, (lo, hi)  # fused A2 + NCCL all_reduce
        lo5, hi5 = inputs.config5_intervals(128)
        c, s = D.batch(lo5, hi5)
        oc, os_ = oracle.batch(lo5, hi5)
        assert np.array_equal(c, oc) and np.array_equal(s, os_)
        words, cs = D.gather_bitmap(*inputs.CONFIG1)
        w = words.cpu().numpy().view(np.uint32)
        assert oracle.fnv1a64(w) == 0x166192dced6b795c and cs == D.bitmap_checksum(w)
        lst = D.gather_primes(*inputs.CONFIG1)
        assert lst.numel() == 664579
        # the fused all-reduce (F4) on a one-rank NCCL group, then back to NCCL
        assert D.attach_peers(timeout_ms=2000) is True
        assert D.stats(*inputs.CONFIG3) == (455052511, 2220822432581729238)
        D.detach_peers()
        assert D.stats(*inputs.CONFIG3) == (455052511, 2220822432581729238)
    finally:
        dist.destroy_process_group()
        sv.set_stream(None)
