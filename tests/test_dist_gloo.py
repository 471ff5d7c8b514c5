"""World-size-2 gloo tests of the multi-GPU host logic (CPU only).

The B200 path shards chains by whole groups across ranks and all-reduces the
moment vector once (dist.run_sharded). Here the per-rank moment vectors come
from the oracle's per-chain sums of each rank's shard; the test checks that
shard() covers the chains exactly once and that the all-reduced moments equal
the moments of the unsharded run (the invariant the GPU path relies on).
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_cs_0412107_b200.dist import allreduce_moments, shard


def test_shard_partition():
    for total, world, gs in ((8192, 8, 32), (1024, 3, 32), (64, 2, 1), (96, 4, 16)):
        seen = []
        for r in range(world):
            cb, ch = shard(total, world, r, gs)
            assert cb % gs == 0 and ch % gs == 0 and ch > 0
            seen.extend(range(cb, cb + ch))
        assert seen == list(range(total))
    with pytest.raises(ValueError):
        shard(64, 4, 0, 32)


def _moments(sums, cycles, gs):
    g = sums.reshape(-1, gs, *sums.shape[1:]).sum(1)
    return np.concatenate([g.sum(0).ravel(), (g * g).sum(0).ravel(), [0.0]])


def _worker(rank, world, port, q):
    import torch
    import oracle
    import workloads as W
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = W.pedigree(300, seed=3)
    total, gs = 128, 32
    cb, ch = shard(total, world, rank, gs)
    r = oracle.Matrix(c).run(7, ch, 3, 5, ("diag",), chain_begin=cb)
    mom = torch.tensor(_moments(r["diag"], 5, gs))
    allreduce_moments(mom)
    if rank == 0:
        full = oracle.Matrix(c).run(7, total, 3, 5, ("diag",))
        q.put((mom.numpy(), _moments(full["diag"], 5, gs)))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_moments_allreduce():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, want = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    np.testing.assert_allclose(got, want, rtol=1e-12)
