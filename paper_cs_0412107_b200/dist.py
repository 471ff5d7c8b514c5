"""Multi-GPU data parallelism over chains.

Chains are independent (PAPER.md:377-423 runs each chain on its own), so GPU
r of W runs a contiguous range of whole standard-error groups, keyed by the
GLOBAL chain index in the Philox counter -- per-chain trajectories are the
same for every W. C and Q are replicated. The only exchange is at the end of
the run: a SUM all-reduce (NCCL over NVLink/NVSwitch on B200) of the moment
vector (S1 per output element, plus the divergence count), then, after each
rank recomputes its groups' scatter about the global mean (mcinv_recenter), a
SUM all-reduce of that M2 block; estimates and standard errors are then
finalized on every rank.
"""
from __future__ import annotations

from typing import Sequence


def shard(total_chains: int, world: int, rank: int, group_size: int = 32):
    """(chain_begin, chains) of ``rank``: whole groups, balanced, contiguous."""
    if total_chains % group_size:
        raise ValueError("total_chains must be a multiple of group_size")
    groups = total_chains // group_size
    if groups < world:
        raise ValueError(f"{groups} groups cannot feed {world} ranks")
    base, extra = divmod(groups, world)
    g0 = rank * base + min(rank, extra)
    gn = base + (1 if rank < extra else 0)
    return g0 * group_size, gn * group_size


def _world(group=None) -> int:
    import torch.distributed as dist
    return dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1


def allreduce_moments(acc, group=None):
    """SUM all-reduce of a moment vector (torch tensor) across the group."""
    import torch.distributed as dist
    if _world(group) > 1:
        dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)
    return acc


def reduce_moments(inv, total_chains: int, group=None):
    """The job's moments on every rank (mcinv_accumulators protocol): SUM all-reduce
    of the whole vector (S1, and the divergence count), then M2 recomputed about
    the global mean from this rank's group sums (mcinv_recenter) and a second SUM
    all-reduce of the M2 block. One GPU: the run's own moments are already final."""
    if _world(group) > 1:
        allreduce_moments(inv.accumulators(), group)
        allreduce_moments(inv.recenter(total_chains), group)
    return inv.accumulators()


def run_sharded(inv, seed: int, total_chains: int, burn_in: int, cycles: int, outputs: Sequence[str],
                group_size: int = 32, group=None, on_device: bool = False, **kw):
    """Run this rank's shard of ``total_chains`` on ``inv`` (an Inverter on
    this rank's GPU), all-reduce the moments and return
    {output: (estimate, std_error)} for the whole job."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    cb, ch = shard(total_chains, world, rank, group_size)
    inv.run(seed, ch, burn_in, cycles, outputs, chain_begin=cb, group_size=group_size, **kw)
    reduce_moments(inv, total_chains, group)
    return {o: inv.result(o, total_chains=total_chains, on_device=on_device) for o in outputs}
