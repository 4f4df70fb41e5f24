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

import os

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


def safe_cuts(tokens, traj_offsets, terminator, world: int, pat_tokens=None, classes=None,
              decimal_rule=None) -> np.ndarray:
    """Row-range sharding of trajectories over ``world`` ranks at *safe cuts*
    (SURVEY §8(e)): positions p where no post-sentence window and no cue
    pattern contains both p - 1 and p — every trajectory start and every
    sentence start (tokens[p - 1] is a terminator).  A window [s, e] ends at
    the first terminator >= s, so it never crosses a sentence start; a pattern
    occurrence crosses one only if the pattern holds a terminator token
    (checked here, with class elements' classes, and rejected).  The decimal
    rule (R19) decides sentence ends from the next token, which a cut would
    hide: rejected too.  Returns world + 1 cut positions, each the safe cut
    nearest to k * n_tok / world (monotone; a rank may get an empty range when
    a long unterminated run leaves no cut near its share).  Every rank then
    runs H1-H5 on its range as trajectories of their own (``range_view``), and
    the SUM of the tables equals the one-rank table bit for bit."""
    tokens = np.asarray(tokens)
    term = np.asarray(terminator).astype(bool)
    if decimal_rule is not None:
        raise ValueError("safe cuts do not support the decimal-number rule")
    if pat_tokens is not None:
        pt = np.asarray(pat_tokens)
        if term[pt[pt >= 0]].any():
            raise ValueError("a cue pattern contains a terminator token: no sentence start is a safe cut")
        if (pt < 0).any():
            if classes is None:
                raise ValueError("class pattern elements need classes")
            for c in np.unique(-1 - pt[pt < 0]):
                if (np.asarray(classes[c]).astype(bool) & term).any():
                    raise ValueError("a cue class contains a terminator token")
    n = tokens.shape[0]
    offs = np.asarray(traj_offsets, np.int64) if traj_offsets is not None else np.array([0, n], np.int64)
    cand = np.zeros(n + 1, bool)
    cand[offs] = True
    if n:
        cand[1:n + 1] |= term[tokens]       # the position after a terminator starts a sentence
    pos = np.flatnonzero(cand)              # sorted; holds 0 and n
    cuts = np.empty(world + 1, np.int64)
    cuts[0], cuts[world] = 0, n
    for k in range(1, world):
        want = (k * n) // world
        i = int(np.searchsorted(pos, want))
        best = pos[min(i, pos.size - 1)]
        if i > 0 and want - pos[i - 1] <= best - want:
            best = pos[i - 1]
        cuts[k] = max(best, cuts[k - 1])
    return cuts


def range_view(tokens, traj_offsets, think_end_pos, lo: int, hi: int):
    """Positions [lo, hi) of the token stream as trajectories of their own: the
    trajectory boundaries inside the range plus its ends, think-end positions
    rebased and clipped to each local trajectory."""
    tokens = np.asarray(tokens)
    n = tokens.shape[0]
    offs = np.asarray(traj_offsets, np.int64) if traj_offsets is not None else np.array([0, n], np.int64)
    inner = offs[(offs > lo) & (offs < hi)]
    loc = np.concatenate([[lo], inner, [hi]]).astype(np.int64) - lo
    tep = None
    if think_end_pos is not None:
        te = np.asarray(think_end_pos, np.int64)
        starts = loc[:-1] + lo
        g = np.searchsorted(offs, starts, side="right") - 1      # global trajectory of each piece
        tep = np.clip(te[g] - lo, loc[:-1], loc[1:])
    return tokens[lo:hi], loc, tep


def torch_nccl_comm(group=None, device=None) -> int:
    """The ncclComm_t torch's ProcessGroupNCCL uses for ``group`` on ``device``
    (initialised by a barrier if it is still lazy)."""
    import torch
    import torch.distributed as dist
    g = group if group is not None else dist.group.WORLD
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    backend = g._get_backend(dev)
    ptr = 0
    try:
        ptr = int(backend._comm_ptr())
    except RuntimeError:
        ptr = 0
    if not ptr:
        dist.barrier(group=g, device_ids=[dev.index])
        ptr = int(backend._comm_ptr())
    return ptr


def _loaded_nccl_files() -> set:
    """The libnccl files mapped into this process."""
    try:
        with open("/proc/self/maps") as f:
            return {os.path.realpath(line.split()[-1]) for line in f
                    if "libnccl" in line and line.split()[-1].startswith("/")}
    except OSError:
        return set()


def torch_comm_compatible() -> tuple:
    """(ok, why): may a communicator torch's ProcessGroupNCCL built be handed to
    librelay's ncclAllReduce?  Only when librelay resolved the very library
    torch uses: the same NCCL version and the only libnccl file mapped in the
    process (a statically linked or second NCCL copy would make the ncclComm_t
    a foreign object)."""
    import torch
    import paper_2602_06454_b200 as relay
    tv = torch.cuda.nccl.version()
    tv = tv if isinstance(tv, int) else tv[0] * 10000 + tv[1] * 100 + (tv[2] if len(tv) > 2 else 0)
    rv, path = relay.nccl_version()
    files = _loaded_nccl_files()
    if rv != tv:
        return False, f"librelay resolved NCCL {rv}, torch uses {tv}"
    if os.path.realpath(path) not in files or len(files) != 1:
        return False, f"librelay's NCCL {path} is not torch's only NCCL ({sorted(files)})"
    return True, f"NCCL {rv} from {path}"


_own_comms = {}


def default_comm(group=None, device=None) -> int:
    """The communicator relay_stats_allreduce runs on: torch's own when it is
    the same NCCL library (torch_comm_compatible), else a librelay-owned one
    (NcclComm.from_group, built once per group)."""
    import torch.distributed as dist
    ok, _ = torch_comm_compatible()
    if ok:
        return torch_nccl_comm(group, device)
    key = id(group) if group is not None else 0
    if key not in _own_comms:
        import paper_2602_06454_b200 as relay
        _own_comms[key] = relay.NcclComm.from_group(dist.get_rank(group), dist.get_world_size(group), group)
    return _own_comms[key].ptr


def allreduce_stats(stats, n_cues: int, world_size: int, group=None, n_tables: int = 1,
                    comm: int | None = None, stream=None):
    """H6: one SUM all-reduce of the uint64 stats table(s).  On CUDA tensors
    over an NCCL group it is librelay's relay_stats_allreduce (ncclAllReduce
    on the caller's stream) on ``comm`` or torch's own communicator; on CPU
    tensors (the gloo tests) torch.distributed's all_reduce of the int64 view
    (two's-complement sums equal unsigned sums mod 2^64)."""
    import torch.distributed as dist
    if stats.is_cuda and dist.get_backend(group) == "nccl":
        import paper_2602_06454_b200 as relay
        ptr = comm if comm is not None else default_comm(group, stats.device)
        return relay.stats_allreduce(ptr, stats, n_cues, world_size, n_tables, stream)
    dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=group)
    return stats
