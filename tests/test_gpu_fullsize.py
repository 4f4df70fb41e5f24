"""GPU parity at the headline sizes and end to end from logits (VERDICT r01
items 2 and 3; SURVEY §4 tier 2 "configs 1-3 fully").

* configs[1]: every one of the 32,768 x 151,936 bf16 rows of relay_margin_rows
  against the oracle (top-1/top-2 indices and statuses bit-exact, margins
  < 1e-5), in the launch configuration bench.py times.
* configs[0] and configs[1] end to end: K1 -> K2 -> K3 -> finalize through the
  Analyzer on the synthetic logits vs oracle.analyze run on the ORACLE's own
  margins of the same logits (P:139-146 margin, P:163 post-sentence window,
  P:246-249 selection).  Occurrences, window ends, trigger and invalid counts
  exact; window means/minima and every summary statistic within 1e-5; counts
  of m < tau (low-margin fractions) may differ only by margins within 1e-5 of
  tau (the two sides' margins differ by < 1e-5); selection flags may differ
  only for cues whose oracle mean lies within 2e-5 of the threshold.
* H6 multi-rank tables finalized against the oracle on the whole corpus.
* A workspace reused across problem sizes.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import synth  # noqa: E402

TOL = 1e-5
TAU = 0.5
DEV = "cuda:0"


@pytest.fixture(scope="module")
def relay():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_06454_b200 as r
    return r


def _oracle_rows(L, dtype, vocab, chunk=2048):
    """fp64 oracle over every row, in host chunks (c2 is 10 GB of logits)."""
    import os
    out = {k: [] for k in ("margin", "top1", "top2", "status", "lse")}
    for r0 in range(0, L.shape[0], chunk):
        ref = oracle.margin_rows(synth.host_rows(L[r0:r0 + chunk], dtype), dtype=dtype, vocab=vocab,
                                 threads=os.cpu_count() or 8)
        for k in out:
            out[k].append(ref[k])
    return {k: np.concatenate(v) for k, v in out.items()}


def _check_rows(got, ref):
    np.testing.assert_array_equal(got["status"], ref["status"].astype(np.uint8))
    np.testing.assert_array_equal(got["top1"], ref["top1"])
    np.testing.assert_array_equal(got["top2"], ref["top2"])
    ok = ref["status"] == 0
    assert np.all(np.isnan(got["margin"][~ok]))
    err = np.abs(got["margin"][ok].astype(np.float64) - ref["margin"][ok])
    assert err.max() < TOL, err.max()


def test_margin_rows_c2_every_row(relay):
    """configs[1]: all 32,768 rows against the oracle."""
    cs = synth.make_cueset(151936, 8, 12)
    ts = synth.make_tokens(1, 32768, cs)
    L = synth.make_logits(32768, 151936, "bf16", tokens=ts.tokens, device=DEV, chunk_rows=2048)
    out = relay.margin_rows(L)
    torch.cuda.synchronize()
    got = {k: v.cpu().numpy() for k, v in out.items() if v is not None}
    _check_rows(got, _oracle_rows(L, "bf16", 151936))
    del L, out
    torch.cuda.empty_cache()


def _end_to_end(relay, cfg, seed):
    c = synth.CONFIGS[cfg]
    V, T, dt = c["vocab"], c["traj_len"] * c["n_traj"], c["dtype"]
    h = synth.make_cueset(V, c["n_cues"], c["n_pat"], max_len=c["max_len"], seed=seed)
    ts = synth.make_tokens(c["n_traj"], c["traj_len"], h, seed=seed + 1)
    L = synth.make_logits(T, V, dt, tokens=ts.tokens, seed=seed + 2, device=DEV, chunk_rows=2048)
    cs = relay.CueSet.from_synth(h)
    an = relay.Analyzer(cs, T, V, DEV, tau=TAU)
    stats = an.run(L, torch.as_tensor(ts.tokens, device=DEV), torch.as_tensor(ts.traj_offsets, device=DEV),
                   torch.as_tensor(ts.think_end_pos, device=DEV))
    torch.cuda.synchronize()
    # H1 over every row
    ref = _oracle_rows(L, dt, V)
    got_rows = {k: v.cpu().numpy() for k, v in an.rows.items() if v is not None}
    _check_rows(got_rows, ref)
    del L
    torch.cuda.empty_cache()
    # H2..H7 on the oracle's own margins (fp32, as the paper's logprob pipeline would hand them on)
    m64 = ref["margin"]
    o_scan, o_win, o_sum = oracle.analyze(m64.astype(np.float32), ts.tokens, ts.traj_offsets, h.pat_tokens,
                                          h.pat_offsets, h.pat_cue, h.n_cues, h.terminator, tau=TAU,
                                          think_end_pos=ts.think_end_pos, min_count=3, rule=0)
    n_occ = int(an.scan["n_occ"].item())
    assert n_occ == o_scan["occ_pos"].shape[0]
    np.testing.assert_array_equal(an.scan["occ_pos"][:n_occ].cpu().numpy(), o_scan["occ_pos"])
    np.testing.assert_array_equal(an.scan["occ_pat"][:n_occ].cpu().numpy(), o_scan["occ_pat"])
    bits = an.scan["term_bits"].cpu().numpy().view(np.uint32)
    term = (bits[np.arange(T) >> 5] >> (np.arange(T) & 31)) & 1
    np.testing.assert_array_equal(term, o_scan["term"])
    seg_end = an.seg["seg_end"][:n_occ].cpu().numpy()
    np.testing.assert_array_equal(seg_end, o_win["seg_end"])
    gm = an.seg["seg_mean"][:n_occ].cpu().numpy().astype(np.float64)
    gmin = an.seg["seg_min"][:n_occ].cpu().numpy().astype(np.float64)
    glow = an.seg["seg_lowfrac"][:n_occ].cpu().numpy().astype(np.float64)
    inv = o_win["seg_invalid"] != 0
    assert np.array_equal(np.isnan(gm), inv)
    assert np.abs(gm[~inv] - o_win["seg_mean"][~inv]).max(initial=0) < TOL
    assert np.abs(gmin[~inv] - o_win["seg_min"][~inv]).max(initial=0) < TOL
    # low-margin counts: only margins within 1e-5 of tau may be decided differently
    near = np.concatenate([[0], np.cumsum(np.abs(m64 - TAU) < TOL)])
    pos = o_scan["occ_pos"]
    length = seg_end - pos + 1
    allowed = near[seg_end + 1] - near[pos]
    dlow = np.abs(np.rint(glow * length) - np.rint(o_win["seg_lowfrac"] * length))   # counts (seg_lowfrac is fp32)
    assert np.all(dlow[~inv] <= allowed[~inv])
    assert np.abs(glow[~inv] - o_win["seg_lowfrac"][~inv] - 0).max(initial=0) <= 1.0
    # the table, finalized
    fin = relay.stats_finalize(stats.cpu().numpy(), h.n_cues, 1, 3)
    g = o_sum[-1]
    thr = g["mean"] + g["se"]
    n_band = int(np.sum(np.abs(m64[ref["status"] == 0] - TAU) < TOL))
    for k in range(h.n_cues + 1):
        f, o = fin[k], o_sum[k]
        assert f["n"] == o["n"] and f["n_triggers"] == o["n_triggers"] and f["n_invalid"] == o["n_invalid"], k
        if o["n"] == 0:
            continue
        for key in ("mean", "token_mean", "min"):
            assert abs(f[key] - o[key]) < TOL, (k, key, f[key], o[key])
        if o["n"] > 1:
            assert abs(f["std"] - o["std"]) < TOL and abs(f["se"] - o["se"]) < TOL, k
        if k == h.n_cues:
            assert abs(f["low_frac"] - o["low_frac"]) * o["n"] <= n_band + 1e-6
        else:
            assert abs(f["low_frac"] - o["low_frac"]) <= n_band / max(1, o["n"]) + 1e-6
            if abs(o["mean"] - thr) > 2e-5:
                assert bool(f["selected"]) == bool(o["selected"]), k
    cs.destroy()
    return n_occ, sum(bool(f["selected"]) for f in fin[:-1])


def test_end_to_end_c1(relay):
    """configs[0]: 2,048 x 32,000 fp32, 3 cues, K1 -> K2 -> K3 -> finalize."""
    n_occ, _ = _end_to_end(relay, "c1", 501)
    assert n_occ > 10


def test_end_to_end_c2(relay):
    """configs[1]: 32,768 x 151,936 bf16, 8 cues, K1 -> K2 -> K3 -> finalize."""
    n_occ, _ = _end_to_end(relay, "c2", 601)
    assert n_occ > 100


# ------------------------------------------------------------------ H6
def _h6_corpus(seed, n_traj=6, L=3000):
    h = synth.make_cueset(151936, 8, 12, max_len=3, seed=seed)
    ts = synth.make_tokens(n_traj, L, h, seed=seed + 1)
    m = synth.make_margins(ts.tokens.shape[0], seed=seed + 2)
    return h, ts, m


def test_rank_shards_finalize_like_the_oracle(relay):
    """H6 (the global average over all positions of the calibration
    traces): trajectories sharded over world ranks, each rank's table from its
    shard, the SUM of the tables finalized == oracle.analyze of the whole
    corpus (world = 1, 2, 3, 8)."""
    h, ts, m = _h6_corpus(701, n_traj=8, L=4096)
    cs = relay.CueSet.from_synth(h)
    _, _, o_sum = oracle.analyze(m, ts.tokens, ts.traj_offsets, h.pat_tokens, h.pat_offsets, h.pat_cue,
                                 h.n_cues, h.terminator, tau=TAU, think_end_pos=ts.think_end_pos, min_count=3)
    dm = torch.as_tensor(m, device=DEV)
    for world in (1, 2, 3, 8):
        tot = None
        for r in range(world):
            t0, t1 = r * 8 // world, (r + 1) * 8 // world
            lo, hi = int(ts.traj_offsets[t0]), int(ts.traj_offsets[t1])
            st = relay.new_stats(8, r, world, DEV)
            if hi > lo:
                offs = torch.as_tensor(ts.traj_offsets[t0:t1 + 1] - lo, device=DEV)
                tep = torch.as_tensor(ts.think_end_pos[t0:t1] - lo, device=DEV)
                tok = torch.as_tensor(ts.tokens[lo:hi], device=DEV)
                relay.segment_reduce(cs, dm[lo:hi].contiguous(), relay.cue_scan(cs, tok, offs), offs, tep,
                                     stats=st, rank=r, world_size=world, tau=TAU)
            tot = st if tot is None else tot + st
        torch.cuda.synchronize()
        fin = relay.stats_finalize(tot.cpu().numpy(), 8, world, 3)
        _compare_summaries(fin, o_sum)
    cs.destroy()


def _compare_summaries(fin, o_sum):
    for k, (f, o) in enumerate(zip(fin, o_sum)):
        assert f["n"] == o["n"] and f["n_triggers"] == o["n_triggers"] and f["n_invalid"] == o["n_invalid"], k
        if o["n"]:
            for key in ("mean", "token_mean", "min", "low_frac"):
                assert abs(f[key] - o[key]) < TOL, (k, key)
        if o["n"] > 1:
            assert abs(f["std"] - o["std"]) < TOL and abs(f["se"] - o["se"]) < TOL, k
    thr = o_sum[-1]["mean"] + o_sum[-1]["se"]
    for f, o in zip(fin[:-1], o_sum[:-1]):
        if abs(o["mean"] - thr) > 2e-5:
            assert bool(f["selected"]) == bool(o["selected"])


def _p2p_oracle_worker(rank, world, port, out, fused):
    import torch.distributed as dist
    import paper_2602_06454_b200 as relay
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    h, ts, m = _h6_corpus(801)
    cs = relay.CueSet.from_synth(h)
    x = relay.StatsExchange(8, group=dist.group.WORLD)
    t0, t1 = rank * 6 // world, (rank + 1) * 6 // world
    lo, hi = int(ts.traj_offsets[t0]), int(ts.traj_offsets[t1])
    tok = torch.as_tensor(ts.tokens[lo:hi], device="cuda:0")
    offs = torch.as_tensor(ts.traj_offsets[t0:t1 + 1] - lo, device="cuda:0")
    tep = torch.as_tensor(ts.think_end_pos[t0:t1] - lo, device="cuda:0")
    st = relay.new_stats(8, rank, world, "cuda:0")
    relay.segment_reduce(cs, torch.as_tensor(m[lo:hi], device="cuda:0"), relay.cue_scan(cs, tok, offs), offs,
                         tep, stats=st, rank=rank, world_size=world, tau=TAU, exchange=x if fused else None)
    if not fused:
        x.stats_allreduce(st, 8)
    torch.cuda.synchronize()
    torch.save(st.cpu(), f"{out}.{rank}")
    dist.barrier()
    x.close()
    cs.destroy()
    dist.destroy_process_group()


@pytest.mark.parametrize("fused", [False, True])
def test_p2p_allreduce_finalizes_like_the_oracle(relay, tmp_path, fused):
    """H6 over peer memory with 3 ranks (processes sharing cuda:0): EVERY
    rank's all-reduced table finalizes like oracle.analyze of the whole
    corpus (not only like the one-rank CUDA table)."""
    import socket
    import torch.multiprocessing as mp
    sck = socket.socket()
    sck.bind(("127.0.0.1", 0))
    port = sck.getsockname()[1]
    sck.close()
    out = str(tmp_path / "h6")
    world = 3
    mp.spawn(_p2p_oracle_worker, args=(world, port, out, fused), nprocs=world, join=True)
    h, ts, m = _h6_corpus(801)
    _, _, o_sum = oracle.analyze(m, ts.tokens, ts.traj_offsets, h.pat_tokens, h.pat_offsets, h.pat_cue,
                                 h.n_cues, h.terminator, tau=TAU, think_end_pos=ts.think_end_pos, min_count=3)
    for r in range(world):
        tab = torch.load(f"{out}.{r}").numpy()
        _compare_summaries(relay.stats_finalize(tab, 8, world, 3), o_sum)


# ------------------------------------------------------- workspace reuse
def test_workspace_reused_across_sizes(relay):
    """One workspace, registered for the largest problem, serves smaller ones
    after larger ones (and back): every result equals a fresh workspace's
    (a size-dependent layout put persistent counters on stale
    data)."""
    h = synth.make_cueset(151936, 8, 12, max_len=3, seed=901)
    cs = relay.CueSet.from_synth(h)
    ws = relay.workspace(131072, 131072, 64, DEV)
    for n_traj, L in ((4, 32768), (2, 32768), (1, 20000), (4, 32768), (3, 1000)):
        ts = synth.make_tokens(n_traj, L, h, seed=902 + n_traj + L)
        n = ts.tokens.shape[0]
        tok = torch.as_tensor(ts.tokens, device=DEV)
        offs = torch.as_tensor(ts.traj_offsets, device=DEV)
        m = torch.as_tensor(synth.make_margins(n, seed=903), device=DEV)
        sa = relay.cue_scan(cs, tok, offs, 131072, ws=ws)
        a = relay.segment_reduce(cs, m, sa, offs, ws=ws)
        sb = relay.cue_scan(cs, tok, offs, 131072)
        b = relay.segment_reduce(cs, m, sb, offs)
        torch.cuda.synchronize()
        assert torch.equal(a["stats"], b["stats"])
        k = int(sb["n_occ"].item())
        assert k == int(sa["n_occ"].item()) and k > 0
        assert torch.equal(sa["occ_pos"][:k], sb["occ_pos"][:k])
        assert torch.equal(a["seg_end"][:k], b["seg_end"][:k])
    for B in (64, 32, 64, 7, 48):
        L = synth.make_logits(B, 151936, "bf16", seed=904 + B, device=DEV)
        state = torch.zeros(B, dtype=torch.uint8, device=DEV)
        hist = torch.full((B, 7), -1, dtype=torch.int32, device=DEV)
        r1 = relay.step_switch(cs, L, state.clone(), hist.clone(), ws=ws)
        r2 = relay.step_switch(cs, L, state.clone(), hist.clone())
        torch.cuda.synchronize()
        for key in ("top1", "top2", "flag"):
            assert torch.equal(r1[key], r2[key]), (B, key)
    with pytest.raises(relay.RelayError):   # above the registered capacity
        ts = synth.make_tokens(1, 140000, h, seed=905)
        relay.cue_scan(cs, torch.as_tensor(ts.tokens, device=DEV), None, 131072, ws=ws)
    cs.destroy()
