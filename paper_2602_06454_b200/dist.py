"""Host-side multi-GPU plumbing for the RelayGen hot path (H6).

The path shards by trajectory (north_star "trajectory rows are
sharded across the 8 GPUs of one box"): every rank runs H1-H5 on a contiguous
block of whole trajectories, so no window or cue pattern ever crosses ranks
and there is no data-path collective.  The only exchange is one SUM
all-reduce of the uint64 statistics table (int64 view: two's-complement sums
equal unsigned sums mod 2^64), with each rank's minimum carried in its own
slot (relay_stats_init).  Works with any torch.distributed backend (NCCL on
the GPUs; gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np


def shard_trajectories(traj_offsets, world: int, rank: int) -> tuple[int, int]:
    """Contiguous trajectory block [lo, hi) of ``rank``, balanced by token count:
    trajectory k goes to the rank whose equal share of the tokens contains the
    trajectory's first token."""
    offs = np.asarray(traj_offsets, np.int64)
    n_traj = offs.shape[0] - 1
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    total = int(offs[-1] - offs[0])
    if n_traj == 0 or total == 0:
        return (0, 0) if rank else (0, n_traj)
    owner = np.minimum(((offs[:-1] - offs[0]) * world) // total, world - 1)
    ks = np.nonzero(owner == rank)[0]
    if ks.size == 0:
        lo = int(np.searchsorted(owner, rank))
        return lo, lo
    return int(ks[0]), int(ks[-1]) + 1


def local_view(tokens, traj_offsets, think_end_pos, lo: int, hi: int):
    """Slice of the token stream holding trajectories [lo, hi), with offsets and
    think-end positions rebased to the slice."""
    offs = np.asarray(traj_offsets, np.int64)
    a, b = int(offs[lo]), int(offs[hi])
    loc_offs = offs[lo:hi + 1] - a
    loc_tep = None if think_end_pos is None else np.asarray(think_end_pos, np.int64)[lo:hi] - a
    return np.asarray(tokens)[a:b], loc_offs, loc_tep, (a, b)


def allreduce_stats(stats, group=None):
    """H6: one SUM all-reduce of the (int64 view of the) uint64 stats table."""
    import torch.distributed as dist
    dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=group)
    return stats
