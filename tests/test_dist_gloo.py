"""Multi-process (world_size 2, gloo, CPU) tests of the host-side multi-GPU
logic: trajectory sharding, the single SUM all-reduce of the integer
statistics table with per-rank min slots (H6), and that finalize (H7) of the
reduced table equals the single-process result bit for bit.

The per-rank tables are built here with plain Python integers following the
table definition in include/relay.h (q = rint(m 2^20), window mean =
floor((2 sum q + len) / (2 len))), from window ends the oracle computes — the
kernels are exercised by the -m gpu tests; this file covers the host logic.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import synth  # noqa: E402

NF = 8


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def q20(x):
    return int(round(float(np.float32(x)) * (1 << 20)))


def table(margins, tokens, offs, tep, cs, tau, rank, world):
    """uint64 table [(n_cues+1) x (8+world)] of one shard, per include/relay.h."""
    scan = oracle.cue_scan(tokens, offs, cs.pat_tokens, cs.pat_offsets, cs.pat_cue, cs.n_cues,
                           cs.terminator)
    win = oracle.windows(margins, scan["term"], offs, scan["occ_pos"], tau)
    nf = NF + world
    t = np.zeros((cs.n_cues + 1, nf), dtype=object)
    t[:, :] = 0
    t[:, NF + rank] = 0x7F800000
    occ, pat, ends = scan["occ_pos"].tolist(), scan["occ_pat"].tolist(), win["seg_end"].tolist()
    traj = np.searchsorted(offs, occ, side="right") - 1
    for i, s in enumerate(occ):
        prev = [j for j in range(i) if occ[j] < s]
        trig = 1 if not prev or ends[prev[-1]] != ends[i] else 0
        if tep is not None and s >= tep[traj[i]]:
            continue
        c = int(cs.pat_cue[pat[i]])
        w = margins[s:ends[i] + 1]
        if np.isnan(w).any():
            t[c, 7] += 1
            continue
        qs = [q20(x) for x in w]
        ln, sq = len(qs), sum(qs)
        mq = (2 * sq + ln) // (2 * ln)
        t[c, 0] += 1; t[c, 1] += mq; t[c, 2] += mq * mq; t[c, 3] += sq; t[c, 4] += ln
        t[c, 5] += sum(1 for x in w if np.float32(x) < np.float32(tau)); t[c, 6] += trig
        t[c, NF + rank] = min(t[c, NF + rank], int(np.float32(min(w)).view(np.uint32)))
    g = cs.n_cues
    for k in range(len(offs) - 1):
        for p in range(int(offs[k]), int(offs[k + 1])):
            if tep is not None and p >= tep[k]:
                continue
            m = margins[p]
            if np.isnan(m):
                t[g, 7] += 1
                continue
            q = q20(m)
            t[g, 0] += 1; t[g, 1] += q; t[g, 2] += q * q; t[g, 3] += q; t[g, 4] += 1
            t[g, 5] += int(np.float32(m) < np.float32(tau))
            t[g, NF + rank] = min(t[g, NF + rank], int(np.float32(m).view(np.uint32)))
    return np.array([[int(x) % (1 << 64) for x in row] for row in t], dtype=np.uint64)


def _case():
    cs = synth.make_cueset(4096, 4, 6, max_len=3, seed=71)
    ts = synth.make_tokens(5, 700, cs, seed=72, cue_rate=0.5)
    m = synth.make_margins(ts.tokens.shape[0], seed=73, nan_rate=0.001)
    return cs, ts, m


def _worker(rank, world, port, out):
    import torch.distributed as dist

    from paper_2602_06454_b200.dist import allreduce_stats, local_view, shard_trajectories
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    cs, ts, m = _case()
    lo, hi = shard_trajectories(ts.traj_offsets, world, rank)
    tok, offs, tep, (a, b) = local_view(ts.tokens, ts.traj_offsets, ts.think_end_pos, lo, hi)
    t = table(m[a:b], tok, offs, tep, cs, 0.5, rank, world)
    st = torch.from_numpy(t.reshape(-1).view(np.int64).copy())
    allreduce_stats(st, cs.n_cues, world)
    if rank == 0:
        np.save(out, st.numpy())
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_two_ranks_match_one(tmp_path):
    import torch.multiprocessing as mp
    out = str(tmp_path / "reduced.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    reduced = np.load(out).view(np.uint64).reshape(-1, NF + 2)
    cs, ts, m = _case()
    single = table(m, ts.tokens, ts.traj_offsets, ts.think_end_pos, cs, 0.5, 0, 1)
    np.testing.assert_array_equal(reduced[:, :NF], single[:, :NF])
    np.testing.assert_array_equal(np.minimum(reduced[:, NF], reduced[:, NF + 1]), single[:, NF])
    import paper_2602_06454_b200 as relay
    f2 = relay.stats_finalize(reduced.reshape(-1).view(np.int64), cs.n_cues, 2, 1)
    f1 = relay.stats_finalize(single.reshape(-1).view(np.int64), cs.n_cues, 1, 1)
    assert f1 == f2
    # and the table agrees with the oracle's fp64 statistics within the Q20 error
    _, _, summ = oracle.analyze(m, ts.tokens, ts.traj_offsets, cs.pat_tokens, cs.pat_offsets,
                                cs.pat_cue, cs.n_cues, cs.terminator,
                                think_end_pos=ts.think_end_pos, min_count=1)
    for c in range(cs.n_cues + 1):
        assert f1[c]["n"] == summ[c]["n"] and f1[c]["n_invalid"] == summ[c]["n_invalid"]
        if summ[c]["n"]:
            assert abs(f1[c]["mean"] - summ[c]["mean"]) < 1e-5
            assert abs(f1[c]["min"] - summ[c]["min"]) < 1e-7
        if c < cs.n_cues:
            assert f1[c]["n_triggers"] == summ[c]["n_triggers"]


def test_shard_trajectories_partition():
    from paper_2602_06454_b200.dist import shard_trajectories
    rng = np.random.default_rng(5)
    for _ in range(200):
        n = int(rng.integers(0, 12))
        lens = rng.integers(0, 50, n)
        offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        for world in (1, 2, 3, 8):
            got = [shard_trajectories(offs, world, r) for r in range(world)]
            covered = [k for lo, hi in got for k in range(lo, hi)]
            assert covered == list(range(n))            # each trajectory exactly once, in order
            assert all(lo <= hi for lo, hi in got)


def test_eight_way_shard_of_c4_is_one_trajectory_each():
    from paper_2602_06454_b200.dist import shard_trajectories
    offs = np.arange(9, dtype=np.int64) * 32768
    assert [shard_trajectories(offs, 8, r) for r in range(8)] == [(r, r + 1) for r in range(8)]
    assert [shard_trajectories(offs, 2, r) for r in range(2)] == [(0, 4), (4, 8)]


def test_safe_cuts_windows_and_occurrences_are_local():
    """Row-range sharding at safe cuts: the oracle's occurrences
    and post-sentence windows computed per range, rebased, equal the ones of
    the whole stream, and the per-range global moments / cue tables add up to
    the whole stream's (n, sums, counts, triggers exactly)."""
    import oracle
    from paper_2602_06454_b200.dist import range_view, safe_cuts
    h = synth.make_cueset(6000, 5, 8, max_len=3, seed=41)
    ts = synth.make_tokens(3, 2500, h, seed=42)
    m = synth.make_margins(ts.tokens.shape[0], seed=43)
    full = oracle.analyze(m, ts.tokens, ts.traj_offsets, h.pat_tokens, h.pat_offsets, h.pat_cue,
                          h.n_cues, h.terminator, think_end_pos=ts.think_end_pos, min_count=1)
    for world in (2, 3, 5, 8):
        cuts = safe_cuts(ts.tokens, ts.traj_offsets, h.terminator, world, h.pat_tokens)
        assert cuts[0] == 0 and cuts[-1] == ts.tokens.shape[0] and (np.diff(cuts) >= 0).all()
        term = h.terminator.astype(bool)
        for p in cuts[1:-1]:   # a trajectory start or a sentence start
            assert p in ts.traj_offsets or term[ts.tokens[p - 1]]
        occ, ends, n_glob, sums = [], [], 0, None
        for r in range(world):
            lo, hi = int(cuts[r]), int(cuts[r + 1])
            if lo == hi:
                continue
            tok, offs, tep = range_view(ts.tokens, ts.traj_offsets, ts.think_end_pos, lo, hi)
            part = oracle.analyze(m[lo:hi], tok, offs, h.pat_tokens, h.pat_offsets, h.pat_cue, h.n_cues,
                                  h.terminator, think_end_pos=tep, min_count=1)
            occ.append(part[0]["occ_pos"] + lo)
            ends.append(part[1]["seg_end"] + lo)
        np.testing.assert_array_equal(np.concatenate(occ), full[0]["occ_pos"])
        np.testing.assert_array_equal(np.concatenate(ends), full[1]["seg_end"])


def test_safe_cuts_reject_unsafe_cue_sets():
    from paper_2602_06454_b200.dist import safe_cuts
    term = np.zeros(10, np.uint8)
    term[3] = 1
    toks = np.array([1, 2, 3, 4, 5, 3, 6], np.int32)
    with pytest.raises(ValueError):
        safe_cuts(toks, None, term, 2, pat_tokens=np.array([2, 3], np.int32))     # pattern holds a terminator
    with pytest.raises(ValueError):
        safe_cuts(toks, None, term, 2, decimal_rule=(0, 1, 2))
    cuts = safe_cuts(toks, None, term, 2, pat_tokens=np.array([1, 2], np.int32))
    assert list(cuts) == [0, 3, 7] or list(cuts) == [0, 6, 7]


def test_range_view_rebases_and_clips():
    """range_view: trajectory boundaries inside the range become local ones,
    think-end positions are rebased and clipped to each local piece."""
    from paper_2602_06454_b200.dist import range_view
    toks = np.arange(20, dtype=np.int32)
    offs = np.array([0, 8, 14, 20], np.int64)
    tep = np.array([6, 13, 16], np.int64)
    t, o, te = range_view(toks, offs, tep, 5, 17)
    np.testing.assert_array_equal(t, toks[5:17])
    np.testing.assert_array_equal(o, [0, 3, 9, 12])          # pieces [5,8) [8,14) [14,17)
    np.testing.assert_array_equal(te, [1, 8, 11])            # 6-5; 13-5; 16-5 (inside each piece)
    t, o, te = range_view(toks, offs, tep, 7, 8)             # think ended at 6 < 7: clipped to the start
    np.testing.assert_array_equal(o, [0, 1])
    np.testing.assert_array_equal(te, [0])
    t, o, te = range_view(toks, offs, tep, 14, 15)           # think ends at 16 > 15: clipped to the end
    np.testing.assert_array_equal(te, [1])
    t, o, te = range_view(toks, offs, None, 8, 14)           # exactly one trajectory
    np.testing.assert_array_equal(o, [0, 6]) and te is None
