"""World-size-2 gloo tests of the multi-GPU host logic (CPU only).

The B200 path shards chains by whole SE groups across ranks (dist.shard) and
reduces the moment vector of include/mcinv.h at the end (dist.run_sharded:
SUM all-reduce of [S1 | M2 | divergence], mcinv_recenter, SUM all-reduce of
the M2 block). Here a stand-in Inverter implements that documented vector
layout from the oracle's per-chain sums of its shard, so run_sharded's
protocol is exercised end to end on gloo: the sharded estimate and standard
error must equal the unsharded oracle estimate (oracle.estimate, reading R15).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_cs_0412107_b200.dist import allreduce_moments, run_sharded, shard


def test_shard_partition():
    for total, world, gs in ((8192, 8, 32), (1024, 3, 32), (64, 2, 1), (96, 4, 16), (16384, 8, 32)):
        seen = []
        for r in range(world):
            cb, ch = shard(total, world, r, gs)
            assert cb % gs == 0 and ch % gs == 0 and ch > 0
            seen.extend(range(cb, cb + ch))
        assert seen == list(range(total))
    with pytest.raises(ValueError):
        shard(64, 4, 0, 32)


class FakeInverter:
    """The moment-vector contract of mcinv_accumulators / mcinv_recenter /
    mcinv_result (include/mcinv.h), fed by the oracle instead of the GPU."""

    def __init__(self, csr, outputs):
        import oracle
        self.m = oracle.Matrix(csr)
        self.n = csr.n
        self.outputs = outputs

    def run(self, seed, chains, burn_in, cycles, outputs, chain_begin=0, group_size=32, **kw):
        r = self.m.run(seed, chains, burn_in, cycles, outputs, chain_begin=chain_begin)
        self.gs, self.cycles, self.chains = group_size, cycles, chains
        # per-group sums, [G][count] per output, outputs in DIAG, PATTERN, FULL, TRACE order
        self.g = [r[o].reshape(chains // group_size, group_size, -1).sum(1) for o in outputs]
        s1 = [g.sum(0) for g in self.g]
        m2 = [((g - g.mean(0)) ** 2).sum(0) for g in self.g]
        self.acc = torch.tensor(np.concatenate(s1 + m2 + [np.zeros(1)]))
        return self

    def accumulators(self):
        return self.acc

    def recenter(self, total_chains):
        G = total_chains // self.gs
        nS1 = sum(g.shape[1] for g in self.g)
        s1 = self.acc[:nS1].numpy()
        o = 0
        for g in self.g:
            k = g.shape[1]
            self.acc[nS1 + o:nS1 + o + k] = torch.tensor(((g - s1[o:o + k] / G) ** 2).sum(0))
            o += k
        return self.acc[nS1:2 * nS1]

    def result(self, output, total_chains=None, on_device=False):
        idx = self.outputs.index(output)
        nS1 = sum(g.shape[1] for g in self.g)
        o = sum(g.shape[1] for g in self.g[:idx])
        k = self.g[idx].shape[1]
        s1 = self.acc[o:o + k].numpy()
        m2 = self.acc[nS1 + o:nS1 + o + k].numpy()
        G = total_chains // self.gs
        est = s1 / (total_chains * self.cycles)
        se = np.sqrt(m2 / (G - 1) / G) / (self.gs * self.cycles)
        return est, se


def _worker(rank, world, port, q):
    import oracle
    import workloads as W
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = W.pedigree(300, seed=3)
    total, gs = 144, 16  # 9 groups: uneven shards of 5 + 4 groups
    inv = FakeInverter(c, ("diag",))
    res = run_sharded(inv, 7, total, 3, 5, ("diag",), group_size=gs)
    if rank == 0:
        full = oracle.Matrix(c).run(7, total, 3, 5, ("diag",))
        q.put((res["diag"], oracle.estimate(full["diag"], 5, group_size=gs)))
    dist.barrier()
    dist.destroy_process_group()


def _worker_plain(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x = torch.arange(5, dtype=torch.float64) * (rank + 1)
    allreduce_moments(x)
    if rank == 0:
        q.put(x.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _spawn(target, world=2):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=target, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return got


def test_allreduce_sums():
    np.testing.assert_array_equal(_spawn(_worker_plain), np.arange(5) * 3.0)


def test_run_sharded_matches_unsharded_oracle():
    """run_sharded over 2 gloo ranks (whole groups per rank, global chain
    indices in the noise key): estimate and SE equal the unsharded oracle's."""
    (eg, sg), (eo, so) = _spawn(_worker)
    np.testing.assert_allclose(eg, eo, rtol=1e-12, atol=0)
    np.testing.assert_allclose(sg, so, rtol=1e-10, atol=0)
