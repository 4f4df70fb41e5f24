"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by
element, on the same seeded synthetic inputs.

Bars (north_star): indices, statuses, cue positions, window ends, counts and
trigger counts bit-exact; margins and statistics within 1e-5 absolute.  Where
a float decides an integer (m < tau), both sides decide on the same fp32
margins (K3 is fed synthetic fp32 margins, never K1's output).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import synth  # noqa: E402

TOL = 1e-5


@pytest.fixture(scope="module")
def relay():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_06454_b200 as r
    return r


DEV = "cuda:0"


def _rows_check(relay, logits, dtype, vocab, iota=1.0, rows=None):
    out = relay.margin_rows(logits, vocab=vocab, inv_temperature=iota)
    torch.cuda.synchronize()
    host = synth.host_rows(logits if rows is None else logits[rows], dtype)
    ref = oracle.margin_rows(host, dtype=dtype, vocab=vocab, inv_temperature=iota, threads=8)
    sel = slice(None) if rows is None else rows
    got = {k: v[sel].cpu().numpy() for k, v in out.items() if v is not None}
    np.testing.assert_array_equal(got["status"], ref["status"].astype(np.uint8))
    np.testing.assert_array_equal(got["top1"], ref["top1"])
    np.testing.assert_array_equal(got["top2"], ref["top2"])
    ok = ref["status"] == 0
    assert np.all(np.isnan(got["margin"][~ok]))
    err = np.abs(got["margin"][ok] - ref["margin"][ok])
    assert err.size == 0 or err.max() < TOL, err.max()
    lerr = np.abs(got["lse"][ok] - ref["lse"][ok]) / np.maximum(1.0, np.abs(ref["lse"][ok]))
    assert lerr.size == 0 or lerr.max() < 1e-5
    return got, ref


# ------------------------------------------------------------------ H1
@pytest.mark.parametrize("dtype", ["bf16", "f16", "f32"])
@pytest.mark.parametrize("vocab,stride", [(1000, 1000), (1000, 1003), (4099, 4113), (2, 2), (37, 40)])
def test_margin_rows_ragged(relay, dtype, vocab, stride):
    L = synth.make_logits(300, vocab, dtype, row_stride=stride, seed=vocab + stride, device=DEV)
    _rows_check(relay, L, dtype, vocab)


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_margin_rows_edge_rows(relay, dtype):
    V = 5000
    tdt = {"bf16": torch.bfloat16, "f32": torch.float32}[dtype]
    rows = []
    z = torch.randn(V) * 2
    rows.append(z.clone())
    r = z.clone(); r[17] = float("nan"); rows.append(r)               # NaN -> status 1
    r = z.clone(); r[4000] = float("inf"); rows.append(r)             # +inf -> status 1
    rows.append(torch.full((V,), float("-inf")))                      # all -inf -> 2
    r = torch.full((V,), float("-inf")); r[1234] = 3.0; rows.append(r)  # one finite
    r = torch.full((V,), float("-inf")); r[0] = 3.0; rows.append(r)
    r = torch.full((V,), float("-inf")); r[V - 1] = 3.0; rows.append(r)
    r = torch.full((V,), float("-inf")); r[9] = float("nan"); rows.append(r)  # NaN among -inf
    rows.append(torch.zeros(V))                                       # uniform
    rows.append(torch.full((V,), -0.0))
    r = torch.zeros(V); r[::2] = -0.0; rows.append(r)                 # +-0 ties
    r = z.clone(); r[100] = 50.0; r[4999] = 50.0; rows.append(r)     # top-1 tie at the ends
    r = z.clone(); r[3] = 50.0; r[7] = 40.0; r[4998] = 40.0; rows.append(r)  # top-2 tie
    r = torch.arange(V, dtype=torch.float32) * 1e-3; rows.append(r)  # ascending (slow path)
    r = -torch.arange(V, dtype=torch.float32) * 1e-3; rows.append(r)  # descending
    r = torch.full((V,), 1e-40); r[5] = 2e-40; r[6] = 2e-40; rows.append(r)  # subnormals
    r = z.clone() * 1e30; rows.append(r)                              # huge magnitudes
    r = torch.full((V,), -1e30); r[77] = -1e30 + 1e24; rows.append(r)
    L = torch.stack(rows).to(tdt).to(DEV)
    got, ref = _rows_check(relay, L, dtype, V)
    assert got["status"].tolist()[:4] == [0, 1, 1, 2]
    assert got["top1"][4] == 1234 and got["top2"][4] == 0 and got["margin"][4] == 1.0
    assert got["margin"][8] == 0.0 and got["top1"][8] == 0 and got["top2"][8] == 1


@pytest.mark.parametrize("groups", ["0", "1"])
def test_step_switch_edge_rows(relay, monkeypatch, groups):
    """K4 (whole rows, redux.sync merges of the warps' partials) on the K1
    edge rows -- NaN, +-inf, all -inf, one finite, uniform, +-0 ties, exact
    top-1 / top-2 ties at the row ends, ascending / descending, subnormal,
    huge -- replicated past the SM count, two-CTA and grouped layouts."""
    monkeypatch.setenv("RELAY_K4_GROUPS", groups)
    V = 5000
    z = torch.randn(V, generator=torch.Generator().manual_seed(7)) * 2
    rows = [z.clone()]
    r = z.clone(); r[17] = float("nan"); rows.append(r)
    r = z.clone(); r[4000] = float("inf"); rows.append(r)
    rows.append(torch.full((V,), float("-inf")))
    r = torch.full((V,), float("-inf")); r[1234] = 3.0; rows.append(r)
    rows.append(torch.zeros(V))
    rows.append(torch.full((V,), -0.0))
    r = torch.zeros(V); r[::2] = -0.0; rows.append(r)
    r = torch.zeros(V); r[1::2] = -0.0; rows.append(r)
    r = z.clone(); r[100] = 50.0; r[4999] = 50.0; rows.append(r)
    r = z.clone(); r[3] = 50.0; r[7] = 40.0; r[4998] = 40.0; rows.append(r)
    r = torch.arange(V, dtype=torch.float32) * 1e-3; rows.append(r)
    r = -torch.arange(V, dtype=torch.float32) * 1e-3; rows.append(r)
    r = torch.full((V,), 1e-40); r[5] = 2e-40; r[6] = 2e-40; rows.append(r)
    r = z.clone() * 1e30; rows.append(r)
    B = 3 * len(rows) + 200      # > the SM count: the two-rows-per-SM layouts
    L = torch.stack([rows[b % len(rows)] for b in range(B)]).to(torch.bfloat16).to(DEV)
    h, cs = _cs_pair(relay, V, 2, 4, 2, seed=61)
    state = torch.zeros(B, dtype=torch.uint8, device=DEV)
    hist = torch.full((B, 7), -1, dtype=torch.int32, device=DEV)
    out = relay.step_switch(cs, L, state, hist)
    torch.cuda.synchronize()
    ref = oracle.margin_rows(synth.host_rows(L, "bf16"), dtype="bf16", vocab=V, threads=8)
    np.testing.assert_array_equal(out["top1"].cpu().numpy(), ref["top1"])
    np.testing.assert_array_equal(out["top2"].cpu().numpy(), ref["top2"])
    ok = ref["status"] == 0
    m = out["margin"].cpu().numpy()
    assert np.all(np.isnan(m[~ok]))
    assert np.abs(m[ok] - ref["margin"][ok]).max() < TOL
    cs.destroy()


@pytest.mark.parametrize("groups", ["1", "0"])
@pytest.mark.parametrize("n_rows", [1, 2, 3, 443, 445, 889, 1333])
def test_margin_rows_counts_and_groups(relay, monkeypatch, n_rows, groups):
    """K1's row-to-CTA mapping at the edges: fewer rows than CTAs, an odd last
    row for the consumer groups (rows b, b + grid, b + 2 grid, ...), more rows
    than two per CTA; with and without the consumer groups."""
    monkeypatch.setenv("RELAY_K1_GROUPS", groups)
    L = synth.make_logits(n_rows, 3001, "bf16", seed=700 + n_rows, device=DEV)
    _rows_check(relay, L, "bf16", 3001)


def test_margin_rows_temperature(relay):
    L = synth.make_logits(64, 3000, "bf16", seed=5, device=DEV)
    _rows_check(relay, L, "bf16", 3000, iota=1.0 / 0.6)


def test_margin_rows_misaligned_base(relay):
    """A view starting one element in: every row start is 2 bytes off 16."""
    base = synth.make_logits(65, 2049, "bf16", seed=6, device=DEV)
    flat = base.reshape(-1)[1:1 + 64 * 2049].reshape(64, 2049)
    _rows_check(relay, flat, "bf16", 2049)


def test_margin_rows_c1_full(relay):
    """configs[0]: 2,048 x 32,000 fp32, every row against the oracle."""
    cs = synth.make_cueset(32000, 3, 3)
    ts = synth.make_tokens(1, 2048, cs)
    L = synth.make_logits(2048, 32000, "f32", tokens=ts.tokens, device=DEV)
    _rows_check(relay, L, "f32", 32000)


def test_margin_rows_c2_sampled(relay):
    """configs[1] launch shape (32,768 x 151,936 bf16): 192 sampled rows."""
    cs = synth.make_cueset(151936, 8, 12)
    ts = synth.make_tokens(1, 32768, cs)
    L = synth.make_logits(32768, 151936, "bf16", tokens=ts.tokens, device=DEV, chunk_rows=2048)
    rng = np.random.default_rng(0)
    rows = np.unique(np.concatenate([rng.choice(32768, 190, replace=False), [0, 32767]]))
    _rows_check(relay, L, "bf16", 151936, rows=torch.as_tensor(rows))
    del L
    torch.cuda.empty_cache()


def test_margin_rows_deterministic(relay):
    L = synth.make_logits(500, 151936, "bf16", seed=9, device=DEV)
    a = relay.margin_rows(L)
    b = relay.margin_rows(L)
    torch.cuda.synchronize()
    for k in a:
        if a[k] is not None:
            x, y = a[k], b[k]
            if x.is_floating_point():
                x, y = torch.nan_to_num(x, 7.0), torch.nan_to_num(y, 7.0)
            assert torch.equal(x, y), k


def test_margin_rows_invalid_args(relay):
    L = torch.zeros((4, 1), device=DEV)
    with pytest.raises(relay.RelayError):
        relay.margin_rows(L)                       # vocab 1
    L = torch.zeros((4, 8), device=DEV)
    with pytest.raises(relay.RelayError):
        relay.margin_rows(L, inv_temperature=0.0)
    with pytest.raises(relay.RelayError):
        relay.margin_rows(L, vocab=9)              # stride < vocab


# ------------------------------------------------------------------ H2
def _cs_pair(relay, vocab, n_cues, n_pat, max_len, seed, mode=0, **kw):
    h = synth.make_cueset(vocab, n_cues, n_pat, max_len=max_len, seed=seed, **kw)
    return h, relay.CueSet.from_synth(h, mode=mode)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("n_traj,traj_len,n_pat,max_len", [
    (1, 2048, 3, 3), (3, 5000, 12, 3), (7, 333, 32, 6), (1, 1, 3, 2), (64, 1024, 32, 6)])
def test_cue_scan(relay, mode, n_traj, traj_len, n_pat, max_len):
    vocab = 151936
    h, cs = _cs_pair(relay, vocab, min(n_pat, 8), n_pat, max_len, seed=n_pat * 7 + max_len, mode=mode)
    ts = synth.make_tokens(n_traj, traj_len, h, seed=n_traj + traj_len, cue_rate=0.5)
    tok = torch.as_tensor(ts.tokens, device=DEV)
    offs = torch.as_tensor(ts.traj_offsets, device=DEV)
    out = relay.cue_scan(cs, tok, offs)
    torch.cuda.synchronize()
    ref = oracle.cue_scan(ts.tokens, ts.traj_offsets, h.pat_tokens, h.pat_offsets, h.pat_cue,
                          h.n_cues, h.terminator, mode)
    n = int(out["n_occ"].item())
    assert n == ref["occ_pos"].shape[0]
    np.testing.assert_array_equal(out["occ_pos"][:n].cpu().numpy(), ref["occ_pos"])
    np.testing.assert_array_equal(out["occ_pat"][:n].cpu().numpy(), ref["occ_pat"])
    bits = out["term_bits"].cpu().numpy().view(np.uint32)
    term = (bits[np.arange(ts.tokens.shape[0]) >> 5] >> (np.arange(ts.tokens.shape[0]) & 31)) & 1
    np.testing.assert_array_equal(term.astype(np.uint8), ref["term"])


def test_cue_scan_boundaries_and_empty_trajectories(relay):
    """Patterns never cross a trajectory end; empty trajectories; positions
    outside every trajectory never start an occurrence."""
    h = synth.CueSet(np.array([5, 5, 6, 7], np.int32), np.array([0, 1, 3, 4], np.int32),
                     np.array([0, 0, 1], np.int32), 2, 16, np.eye(16, dtype=np.uint8)[0])
    cs = relay.CueSet.from_synth(h)
    tokens = np.array([5, 6, 5, 5, 6, 7, 0, 5, 6, 5], np.int32)
    for offs in ([0, 10], [0, 3, 3, 7, 10], [2, 5, 8], [0, 4, 5, 5, 9]):
        offs = np.array(offs, np.int64)
        out = relay.cue_scan(cs, torch.as_tensor(tokens, device=DEV), torch.as_tensor(offs, device=DEV))
        torch.cuda.synchronize()
        ref = oracle.cue_scan(tokens, offs, h.pat_tokens, h.pat_offsets, h.pat_cue, 2, h.terminator)
        n = int(out["n_occ"].item())
        assert out["occ_pos"][:n].tolist() == ref["occ_pos"].tolist()
        assert out["occ_pat"][:n].tolist() == ref["occ_pat"].tolist()


def test_cue_scan_graph_replay_epochs(relay):
    """K2's look-back words carry a per-launch epoch (no reset pass): a CUDA
    graph replayed over in-place refilled token streams, and a run of eager
    launches on the same workspace, give the oracle's occurrences every time."""
    h, cs = _cs_pair(relay, 151936, 8, 12, 3, seed=131)
    streams = [synth.make_tokens(3, 11000, h, seed=132 + i, cue_rate=0.3 + 0.2 * i) for i in range(4)]
    n = streams[0].tokens.shape[0]
    ws = relay.workspace(n, n, 0, DEV)
    tok = torch.as_tensor(streams[0].tokens, device=DEV)
    offs = torch.as_tensor(streams[0].traj_offsets, device=DEV)
    out = relay.cue_scan(cs, tok, offs, n, ws=ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream(device=DEV)
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            relay.cue_scan(cs, tok, offs, n, ws=ws, out=out, stream=side)
    torch.cuda.synchronize()

    def check(ts):
        ref = oracle.cue_scan(ts.tokens, ts.traj_offsets, h.pat_tokens, h.pat_offsets, h.pat_cue,
                              h.n_cues, h.terminator, 0)
        k = int(out["n_occ"].item())
        assert k == ref["occ_pos"].shape[0]
        np.testing.assert_array_equal(out["occ_pos"][:k].cpu().numpy(), ref["occ_pos"])
        np.testing.assert_array_equal(out["occ_pat"][:k].cpu().numpy(), ref["occ_pat"])

    for rep in range(8):
        ts = streams[rep % 4]
        tok.copy_(torch.as_tensor(ts.tokens, device=DEV))
        g.replay()
        torch.cuda.synchronize()
        check(ts)
    for rep in range(40):   # eager launches on the same workspace advance the epoch further
        ts = streams[rep % 4]
        tok.copy_(torch.as_tensor(ts.tokens, device=DEV))
        relay.cue_scan(cs, tok, offs, n, ws=ws, out=out)
        if rep % 9 == 0:
            torch.cuda.synchronize()
            check(ts)
    cs.destroy()


def test_cue_scan_capacity_overflow(relay):
    h, cs = _cs_pair(relay, 4096, 3, 3, 2, seed=3)
    ts = synth.make_tokens(1, 20000, h, cue_rate=0.9)
    tok = torch.as_tensor(ts.tokens, device=DEV)
    full = relay.cue_scan(cs, tok)
    torch.cuda.synchronize()
    n = int(full["n_occ"].item())
    cap = n // 3
    part = relay.cue_scan(cs, tok, occ_capacity=cap)
    torch.cuda.synchronize()
    assert int(part["n_occ"].item()) == n          # true count reported
    assert torch.equal(part["occ_pos"][:cap], full["occ_pos"][:cap])


def test_cueset_rejects_bad_patterns(relay):
    term = np.zeros(16, np.uint8)
    with pytest.raises(relay.RelayError):   # duplicate
        relay.CueSet([1, 2, 1, 2], [0, 2, 4], [0, 0], 1, term, 16)
    with pytest.raises(relay.RelayError):   # token out of range
        relay.CueSet([1, 99], [0, 2], [0], 1, term, 16)
    with pytest.raises(relay.RelayError):   # empty pattern
        relay.CueSet([1], [0, 0, 1], [0, 0], 1, term, 16)
    with pytest.raises(relay.RelayError):   # too long
        relay.CueSet(list(range(9)), [0, 9], [0], 1, term, 16)
    with pytest.raises(relay.RelayError):   # cue id out of range
        relay.CueSet([1], [0, 1], [3], 2, term, 16)


# ---------------------------------------------------------------- H3-H7
def _segment_case(relay, n_traj, traj_len, n_cues, n_pat, max_len, seed, think=False,
                  nan_rate=0.0, mode=0, tau=0.5, world=1):
    vocab = 151936
    h, cs = _cs_pair(relay, vocab, n_cues, n_pat, max_len, seed=seed, mode=mode)
    ts = synth.make_tokens(n_traj, traj_len, h, seed=seed + 1)
    m = synth.make_margins(ts.tokens.shape[0], seed=seed + 2, nan_rate=nan_rate, tau=tau)
    tok = torch.as_tensor(ts.tokens, device=DEV)
    offs = torch.as_tensor(ts.traj_offsets, device=DEV)
    tep = torch.as_tensor(ts.think_end_pos, device=DEV) if think else None
    scan = relay.cue_scan(cs, tok, offs)
    seg = relay.segment_reduce(cs, torch.as_tensor(m, device=DEV), scan, offs, tep, tau=tau)
    torch.cuda.synchronize()
    o_scan, o_win, o_sum = oracle.analyze(m, ts.tokens, ts.traj_offsets, h.pat_tokens,
                                          h.pat_offsets, h.pat_cue, h.n_cues, h.terminator, tau=tau,
                                          think_end_pos=ts.think_end_pos if think else None,
                                          mode=mode, min_count=1)
    return h, cs, ts, m, scan, seg, o_scan, o_win, o_sum


def _compare_segments(relay, h, scan, seg, o_scan, o_win, o_sum, world=1, min_count=1):
    n = int(scan["n_occ"].item())
    assert n == o_scan["occ_pos"].shape[0]
    np.testing.assert_array_equal(seg["seg_end"][:n].cpu().numpy(), o_win["seg_end"])
    inv = o_win["seg_invalid"].astype(bool)
    for k in ("seg_mean", "seg_min", "seg_lowfrac"):
        got = seg[k][:n].cpu().numpy().astype(np.float64)
        assert np.all(np.isnan(got[inv]))
        err = np.abs(got[~inv] - o_win[k][~inv])
        bar = 0.0 if k == "seg_min" else (1e-6 if k == "seg_mean" else 1e-7)
        assert err.size == 0 or err.max() <= bar, (k, err.max())
    fin = relay.stats_finalize(seg["stats"].cpu().numpy(), h.n_cues, world, min_count=min_count)
    for c in range(h.n_cues + 1):
        g, r = fin[c], o_sum[c]
        assert g["n"] == r["n"] and g["n_invalid"] == r["n_invalid"], (c, g, r)
        if c < h.n_cues:
            assert g["n_triggers"] == r["n_triggers"], (c, g, r)
        if r["n"] == 0:
            continue
        for f in ("mean", "token_mean", "min", "low_frac"):
            assert abs(g[f] - r[f]) < TOL, (c, f, g[f], r[f])
        if not np.isnan(r["std"]):
            assert abs(g["std"] - r["std"]) < TOL and abs(g["se"] - r["se"]) < TOL, (c, g, r)
        assert g["selected"] == r["selected"] or abs(
            r["mean"] - (o_sum[-1]["mean"] + o_sum[-1]["se"])) < 2e-6, (c, g, r)
    return fin


@pytest.mark.parametrize("case", [
    dict(n_traj=1, traj_len=2048, n_cues=3, n_pat=3, max_len=3, seed=1),
    dict(n_traj=1, traj_len=32768, n_cues=8, n_pat=12, max_len=3, seed=2),
    dict(n_traj=8, traj_len=4096, n_cues=8, n_pat=12, max_len=3, seed=3, think=True),
    dict(n_traj=5, traj_len=3001, n_cues=6, n_pat=20, max_len=6, seed=4, nan_rate=0.002),
    dict(n_traj=3, traj_len=2500, n_cues=4, n_pat=9, max_len=4, seed=5, mode=1),
    dict(n_traj=64, traj_len=700, n_cues=32, n_pat=32, max_len=6, seed=6, think=True),
])
def test_segment_reduce(relay, case):
    h, cs, ts, m, scan, seg, o_scan, o_win, o_sum = _segment_case(relay, **case)
    _compare_segments(relay, h, scan, seg, o_scan, o_win, o_sum)


def test_segment_reduce_golden_trace(relay, golden_dir):
    import json
    import os
    g = json.load(open(os.path.join(golden_dir, "trace_fixture.json")))
    pats = g["patterns"]
    po = np.zeros(len(pats) + 1, np.int32)
    po[1:] = np.cumsum([len(p) for p in pats])
    term = np.zeros(g["vocab"], np.uint8)
    term[g["terminator_ids"]] = 1
    cs = relay.CueSet([t for p in pats for t in p], po, g["pat_cue"], g["n_cues"], term, g["vocab"])
    tok = torch.as_tensor(np.array(g["tokens"], np.int32), device=DEV)
    offs = torch.as_tensor(np.array(g["traj_offsets"], np.int64), device=DEV)
    scan = relay.cue_scan(cs, tok, offs)
    seg = relay.segment_reduce(cs, torch.as_tensor(np.array(g["margins"], np.float32), device=DEV),
                               scan, offs, tau=g["tau"])
    torch.cuda.synchronize()
    n = int(scan["n_occ"].item())
    assert scan["occ_pos"][:n].tolist() == [o["s"] for o in g["occurrences"]]
    assert seg["seg_end"][:n].tolist() == [o["e"] for o in g["occurrences"]]
    fin = relay.stats_finalize(seg["stats"].cpu().numpy(), 2, 1, min_count=1)
    for c, e in enumerate(g["cues"]):
        assert fin[c]["n"] == e["n"] and fin[c]["n_triggers"] == e["n_triggers"]
        for f in ("mean", "std", "se", "token_mean", "min", "low_frac"):
            assert abs(fin[c][f] - e[f]) < TOL
    assert [f["selected"] for f in fin[:2]] == g["selected_rule0_min_count_1"]


def test_stats_table_rank_split_is_bit_identical(relay):
    """H6: two ranks each reduce half of the trajectories into their own
    table; the element-wise sum equals the one-rank table (min slots aside)
    and finalizes identically — the property the NCCL sum relies on."""
    vocab = 151936
    h, cs = _cs_pair(relay, vocab, 8, 12, 3, seed=21)
    ts = synth.make_tokens(8, 4096, h, seed=22)
    m = torch.as_tensor(synth.make_margins(ts.tokens.shape[0], seed=23), device=DEV)
    tok = torch.as_tensor(ts.tokens, device=DEV)
    offs = torch.as_tensor(ts.traj_offsets, device=DEV)
    one = relay.segment_reduce(cs, m, relay.cue_scan(cs, tok, offs), offs)["stats"]
    tabs = []
    for r in range(2):
        lo, hi = r * 4 * 4096, (r + 1) * 4 * 4096
        o2 = torch.as_tensor(ts.traj_offsets[4 * r:4 * r + 5] - lo, device=DEV)
        sc = relay.cue_scan(cs, tok[lo:hi].contiguous(), o2)
        st = relay.new_stats(8, r, 2, DEV)
        relay.segment_reduce(cs, m[lo:hi].contiguous(), sc, o2, stats=st, rank=r, world_size=2)
        tabs.append(st)
    torch.cuda.synchronize()
    tot = (tabs[0] + tabs[1]).cpu().numpy().reshape(9, 10)
    base = one.cpu().numpy().reshape(9, 9)
    np.testing.assert_array_equal(tot[:, :8], base[:, :8])
    np.testing.assert_array_equal(np.minimum(tot[:, 8], tot[:, 9]), base[:, 8])
    f1 = relay.stats_finalize(base.reshape(-1), 8, 1, 1)
    f2 = relay.stats_finalize(tot.reshape(-1), 8, 2, 1)
    assert f1 == f2


def _stats_p2p_worker(rank, world, port, out, fused=False):
    import torch.distributed as dist
    import paper_2602_06454_b200 as relay
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    vocab, n_traj, L = 151936, 6, 3000
    h = synth.make_cueset(vocab, 8, 12, max_len=3, seed=21)
    cs = relay.CueSet.from_synth(h)
    x = relay.StatsExchange(8, group=dist.group.WORLD)
    res = []
    for call in range(3):               # both buffer parities, then the first again
        ts = synth.make_tokens(n_traj, L, h, seed=22 + call)
        m = synth.make_margins(ts.tokens.shape[0], seed=23 + call)
        t0, t1 = rank * n_traj // world, (rank + 1) * n_traj // world
        lo, hi = int(ts.traj_offsets[t0]), int(ts.traj_offsets[t1])
        tok = torch.as_tensor(ts.tokens[lo:hi], device="cuda:0")
        offs = torch.as_tensor(ts.traj_offsets[t0:t1 + 1] - lo, device="cuda:0")
        st = relay.new_stats(8, rank, world, "cuda:0")
        relay.segment_reduce(cs, torch.as_tensor(m[lo:hi], device="cuda:0"), relay.cue_scan(cs, tok, offs), offs,
                             stats=st, rank=rank, world_size=world, exchange=x if fused else None)
        if not fused:
            x.stats_allreduce(st, 8)
        torch.cuda.synchronize()
        res.append(st.cpu())
    if rank == 0:
        torch.save(res, out)
    dist.barrier()
    x.close()
    cs.destroy()
    dist.destroy_process_group()


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("world", [2, 3])
def test_stats_allreduce_p2p(relay, tmp_path, world, fused):
    """H6 over peer memory (no NCCL), world ranks as processes on cuda:0:
    relay_stats_allreduce_p2p after K3, or fused into K3's last CTA
    (relay_segment_reduce_p2p).  Three consecutive passes of per-rank
    trajectory-shard tables each finalize exactly like the one-rank table
    (counts and Q20 moments bit-identical, the min over the rank slots)."""
    import socket
    import torch.multiprocessing as mp
    sck = socket.socket(); sck.bind(("127.0.0.1", 0)); port = sck.getsockname()[1]; sck.close()
    out = str(tmp_path / "stats_p2p.pt")
    mp.spawn(_stats_p2p_worker, args=(world, port, out, fused), nprocs=world, join=True)
    got = torch.load(out)
    h, cs = _cs_pair(relay, 151936, 8, 12, 3, seed=21)
    for call, g in enumerate(got):
        ts = synth.make_tokens(6, 3000, h, seed=22 + call)
        m = torch.as_tensor(synth.make_margins(ts.tokens.shape[0], seed=23 + call), device=DEV)
        tok = torch.as_tensor(ts.tokens, device=DEV)
        offs = torch.as_tensor(ts.traj_offsets, device=DEV)
        one = relay.segment_reduce(cs, m, relay.cue_scan(cs, tok, offs), offs)["stats"].cpu().numpy().reshape(9, 9)
        tot = g.numpy().reshape(9, 8 + world)
        np.testing.assert_array_equal(tot[:, :8], one[:, :8])
        np.testing.assert_array_equal(tot[:, 8:].min(axis=1), one[:, 8])
        assert relay.stats_finalize(tot.reshape(-1), 8, world, 1) == relay.stats_finalize(one.reshape(-1), 8, 1, 1)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_safe_cut_row_shards_sum_to_one_table(relay, world):
    """One trajectory split over ranks at safe cuts (SURVEY §8(e),
    dist.safe_cuts / range_view): every rank's K2 + K3 on its row range as
    trajectories of their own; the SUM of the tables equals the one-rank
    table bit for bit (counts, Q20 moments, triggers; min over the slots)."""
    from paper_2602_06454_b200.dist import range_view, safe_cuts
    vocab = 151936
    h, cs = _cs_pair(relay, vocab, 8, 12, 3, seed=121)
    ts = synth.make_tokens(1, 32768, h, seed=122)
    m = synth.make_margins(ts.tokens.shape[0], seed=123)
    dm = torch.as_tensor(m, device=DEV)
    tok = torch.as_tensor(ts.tokens, device=DEV)
    offs = torch.as_tensor(ts.traj_offsets, device=DEV)
    tep = torch.as_tensor(ts.think_end_pos, device=DEV)
    one = relay.segment_reduce(cs, dm, relay.cue_scan(cs, tok, offs), offs, tep)["stats"]
    cuts = safe_cuts(ts.tokens, ts.traj_offsets, h.terminator, world, h.pat_tokens)
    tot = None
    for r in range(world):
        lo, hi = int(cuts[r]), int(cuts[r + 1])
        st = relay.new_stats(8, r, world, DEV)
        if hi > lo:
            t, o, te = range_view(ts.tokens, ts.traj_offsets, ts.think_end_pos, lo, hi)
            o_d = torch.as_tensor(o, device=DEV)
            sc = relay.cue_scan(cs, torch.as_tensor(t, device=DEV), o_d)
            relay.segment_reduce(cs, dm[lo:hi].contiguous(), sc, o_d, torch.as_tensor(te, device=DEV), stats=st,
                                 rank=r, world_size=world)
        tot = st if tot is None else tot + st
    torch.cuda.synchronize()
    tot = tot.cpu().numpy().reshape(9, 8 + world)
    base = one.cpu().numpy().reshape(9, 9)
    np.testing.assert_array_equal(tot[:, :8], base[:, :8])
    np.testing.assert_array_equal(tot[:, 8:].min(axis=1), base[:, 8])


def test_segment_reduce_deterministic(relay):
    args = dict(n_traj=8, traj_len=4096, n_cues=8, n_pat=12, max_len=3, seed=31)
    a = _segment_case(relay, **args)
    b = _segment_case(relay, **args)
    assert torch.equal(a[5]["stats"], b[5]["stats"])
    n = int(a[4]["n_occ"].item())
    assert n == int(b[4]["n_occ"].item())
    for k in ("seg_end", "seg_mean", "seg_min", "seg_lowfrac"):
        x, y = a[5][k][:n], b[5][k][:n]
        if x.is_floating_point():
            x, y = torch.nan_to_num(x, 7.0), torch.nan_to_num(y, 7.0)
        assert torch.equal(x, y), k


def test_analyzer_end_to_end_small(relay):
    """H1 -> H2 -> H3..H7 through the Analyzer vs the oracle on its own margins:
    exact structure, statistics within 1e-5 (low counts within the +-1e-5 band)."""
    h, cs = _cs_pair(relay, 4096, 3, 4, 3, seed=41)
    ts = synth.make_tokens(2, 1500, h, seed=42)
    n = ts.tokens.shape[0]
    L = synth.make_logits(n, 4096, "bf16", tokens=ts.tokens, seed=43, device=DEV)
    an = relay.Analyzer(cs, n, 4096, DEV)
    stats = an.run(L, torch.as_tensor(ts.tokens, device=DEV), torch.as_tensor(ts.traj_offsets, device=DEV))
    torch.cuda.synchronize()
    ref = oracle.margin_rows(synth.host_rows(L, "bf16"), dtype="bf16", threads=8)
    m64 = ref["margin"]
    got_m = an.rows["margin"].cpu().numpy()
    ok = ref["status"] == 0
    assert np.abs(got_m[ok] - m64[ok]).max() < TOL
    o_scan, o_win, o_sum = oracle.analyze(m64.astype(np.float32), ts.tokens, ts.traj_offsets,
                                          h.pat_tokens, h.pat_offsets, h.pat_cue, h.n_cues,
                                          h.terminator, min_count=1)
    fin = relay.stats_finalize(stats.cpu().numpy(), h.n_cues, 1, 1)
    for c in range(h.n_cues + 1):
        assert fin[c]["n"] == o_sum[c]["n"]
        if o_sum[c]["n"]:
            assert abs(fin[c]["mean"] - o_sum[c]["mean"]) < TOL
            assert abs(fin[c]["token_mean"] - o_sum[c]["token_mean"]) < TOL
    # low-margin fraction: counts may only differ for margins within 1e-5 of tau
    band = np.sum(np.abs(m64[ok] - 0.5) < TOL)
    assert abs(fin[-1]["low_frac"] - o_sum[-1]["low_frac"]) * fin[-1]["n"] <= band + 1e-9


# ------------------------------------------------------------------ H8
def _step_reference(h, lg_host, dtype, vocab, state, hist, small_run, sampled, gate, max_seg):
    ref = oracle.margin_rows(lg_host, dtype=dtype, vocab=vocab)
    B = state.shape[0]
    flags, cues = np.zeros(B, np.uint8), np.zeros(B, np.int16)
    st2, hi2, sr2 = state.copy(), hist.copy(), small_run.copy()
    for b in range(B):
        tok = int(sampled[b]) if sampled is not None else int(ref["top1"][b])
        f, c, s, hh, r = oracle.step_one(tok, np.float32(ref["margin"][b]), int(state[b]), hist[b],
                                         int(small_run[b]), h.pat_tokens, h.pat_offsets, h.pat_cue,
                                         h.terminator, h.think_end, gate, max_seg)
        flags[b], cues[b], st2[b], hi2[b], sr2[b] = f, c, s, hh, r
    return ref, flags, cues, st2, hi2, sr2


@pytest.mark.parametrize("greedy", [False, True])
@pytest.mark.parametrize("B,vocab,dtype,max_seg,gate", [
    (256, 152064, "bf16", 0, -1.0), (37, 5003, "f16", 3, -1.0), (64, 32000, "f32", 0, 0.5)])
def test_step_switch(relay, greedy, B, vocab, dtype, max_seg, gate):
    h, cs = _cs_pair(relay, vocab, 8, 12, 3, seed=51)
    rng = np.random.default_rng(52)
    state = rng.choice([0, 0, 1, 3], B).astype(np.uint8)
    hist = np.full((B, 7), -1, np.int32)
    small_run = rng.integers(0, 4, B).astype(np.int32)
    sampled = rng.integers(3000, vocab, B).astype(np.int32)
    for b in range(B):                       # plant cue completions, terminators, </think>
        kind = rng.integers(0, 5)
        p = h.patterns[int(rng.integers(0, len(h.patterns)))]
        hist[b, 7 - (len(p) - 1):] = p[:-1] if len(p) > 1 else hist[b, 7:]
        if kind == 0:
            sampled[b] = p[-1]
        elif kind == 1:
            sampled[b] = int(rng.choice(synth.TERMINATOR_IDS))
        elif kind == 2:
            sampled[b] = h.think_end
    tokens = None if greedy else sampled
    L = synth.make_logits(B, vocab, dtype, tokens=sampled, seed=53, device=DEV)
    ref, flags, cues, st2, hi2, sr2 = _step_reference(h, synth.host_rows(L, dtype), dtype, vocab,
                                                      state, hist, small_run, tokens, gate, max_seg)
    d_state = torch.as_tensor(state, device=DEV)
    d_hist = torch.as_tensor(hist, device=DEV)
    d_sr = torch.as_tensor(small_run, device=DEV)
    d_samp = None if greedy else torch.as_tensor(sampled, device=DEV)
    out = relay.step_switch(cs, L, d_state, d_hist, d_sr, d_samp, margin_gate=gate,
                            max_small_segment=max_seg)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out["top1"].cpu().numpy(), ref["top1"])
    np.testing.assert_array_equal(out["top2"].cpu().numpy(), ref["top2"])
    ok = ref["status"] == 0
    assert np.abs(out["margin"].cpu().numpy()[ok] - ref["margin"][ok]).max() < TOL
    got_flags = out["flag"].cpu().numpy()
    if gate >= 0:   # the gate decision may only differ within 1e-5 of the gate
        near = np.abs(ref["margin"] - gate) < TOL
        keep = ~near
    else:
        keep = np.ones(B, bool)
    np.testing.assert_array_equal(got_flags[keep], flags[keep])
    np.testing.assert_array_equal(out["cue_id"].cpu().numpy()[keep], cues[keep])
    np.testing.assert_array_equal(d_state.cpu().numpy()[keep], st2[keep])
    np.testing.assert_array_equal(d_hist.cpu().numpy()[keep], hi2[keep])
    np.testing.assert_array_equal(d_sr.cpu().numpy()[keep], sr2[keep])
    assert (got_flags == 1).sum() > 0 or greedy


def test_offline_triggers_equal_online_switches(relay):
    """SURVEY §4 tier 6 on the GPU path: replaying token streams through K4
    step by step (each stream's next token as the sampled token) fires
    large->small exactly as often per cue as K2/K3 count per-sentence first
    occurrences (n_triggers), for a substring-free pattern set without
    terminators (R13); the answer stage (after </think>) fires nothing."""
    V, B, L = 8192, 48, 1500
    h = synth.make_cueset(V, 5, 9, max_len=3, seed=131, prefix_pair=False, substring_free=True)
    cs = relay.CueSet.from_synth(h)
    ts = synth.make_tokens(B, L, h, seed=132, cue_rate=0.4)
    tok = torch.as_tensor(ts.tokens, device=DEV)
    offs = torch.as_tensor(ts.traj_offsets, device=DEV)
    tep = torch.as_tensor(ts.think_end_pos, device=DEV)
    m = torch.as_tensor(synth.make_margins(B * L, seed=133), device=DEV)
    seg = relay.segment_reduce(cs, m, relay.cue_scan(cs, tok, offs), offs, tep)
    torch.cuda.synchronize()
    offline = [c["n_triggers"] for c in relay.stats_finalize(seg["stats"].cpu().numpy(), 5, 1, 1)[:5]]
    streams = torch.as_tensor(ts.tokens.reshape(B, L), device=DEV)
    logits = synth.make_logits(B, V, "bf16", seed=134, device=DEV)
    state = torch.zeros(B, dtype=torch.uint8, device=DEV)
    hist = torch.full((B, 7), -1, dtype=torch.int32, device=DEV)
    small = torch.zeros(B, dtype=torch.int32, device=DEV)
    ws = relay.workspace(0, 0, B, DEV)
    online = torch.zeros(5, dtype=torch.int64, device=DEV)
    out = None
    for t in range(L):
        out = relay.step_switch(cs, logits, state, hist, small, streams[:, t].contiguous(), ws=ws, out=out)
        fired = out["flag"] == 1
        online.index_add_(0, out["cue_id"][fired].long(), torch.ones(int(fired.sum()), dtype=torch.int64,
                                                                      device=DEV))
    torch.cuda.synchronize()
    assert online.cpu().tolist() == offline and sum(offline) > 100


def test_step_switch_graph_replay(relay):
    """Captured in a CUDA graph and replayed: the arrival counters reset
    themselves; replaying a token stream matches the oracle step by step."""
    vocab, B, T = 8192, 16, 40
    h, cs = _cs_pair(relay, vocab, 4, 6, 3, seed=61)
    rng = np.random.default_rng(62)
    ts = synth.make_tokens(B, T, h, seed=63, cue_rate=0.6, mean_sentence=4)
    toks = ts.tokens.reshape(B, T)
    L = synth.make_logits(B, vocab, "bf16", seed=64, device=DEV)
    d_state = torch.zeros(B, dtype=torch.uint8, device=DEV)
    d_hist = torch.full((B, 7), -1, dtype=torch.int32, device=DEV)
    d_sr = torch.zeros(B, dtype=torch.int32, device=DEV)
    d_samp = torch.zeros(B, dtype=torch.int32, device=DEV)
    ws = relay.workspace(0, 0, B, DEV)
    out = relay.step_switch(cs, L, d_state, d_hist, d_sr, d_samp, ws=ws)   # warm-up allocs
    d_state.zero_(); d_hist.fill_(-1); d_sr.zero_()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            relay.step_switch(cs, L, d_state, d_hist, d_sr, d_samp, ws=ws, out=out)
    torch.cuda.synchronize()
    state = np.zeros(B, np.uint8); hist = np.full((B, 7), -1, np.int32); sr = np.zeros(B, np.int32)
    ref = oracle.margin_rows(synth.host_rows(L, "bf16"), dtype="bf16")
    for t in range(T):
        d_samp.copy_(torch.as_tensor(toks[:, t], device=DEV))
        g.replay()
        torch.cuda.synchronize()
        for b in range(B):
            f, c, state[b], hist[b], sr[b] = oracle.step_one(
                int(toks[b, t]), np.float32(ref["margin"][b]), int(state[b]), hist[b], int(sr[b]),
                h.pat_tokens, h.pat_offsets, h.pat_cue, h.terminator, h.think_end)
            assert out["flag"][b].item() == f and out["cue_id"][b].item() == c
        np.testing.assert_array_equal(d_state.cpu().numpy(), state)
        np.testing.assert_array_equal(d_hist.cpu().numpy(), hist)
    del rng


def _segment_custom(relay, tokens, offs, margins, h, tau=0.5, think=None, mode=0):
    cs = relay.CueSet.from_synth(h, mode=mode)
    tok = torch.as_tensor(np.asarray(tokens, np.int32), device=DEV)
    d_offs = torch.as_tensor(np.asarray(offs, np.int64), device=DEV)
    tep = None if think is None else torch.as_tensor(np.asarray(think, np.int64), device=DEV)
    scan = relay.cue_scan(cs, tok, d_offs)
    seg = relay.segment_reduce(cs, torch.as_tensor(margins, device=DEV), scan, d_offs, tep, tau=tau)
    torch.cuda.synchronize()
    o_scan, o_win, o_sum = oracle.analyze(margins, tokens, offs, h.pat_tokens, h.pat_offsets,
                                          h.pat_cue, h.n_cues, h.terminator, tau=tau,
                                          think_end_pos=think, mode=mode, min_count=1)
    _compare_segments(relay, h, scan, seg, o_scan, o_win, o_sum)


def test_segment_reduce_windows_spanning_tiles(relay):
    """Unterminated runs longer than several 2,048-token tiles: the look-back
    must chain tile heads until a sentence end (K3 carry)."""
    h = synth.make_cueset(8192, 3, 4, max_len=2, seed=81)
    rng = np.random.default_rng(82)
    n = 20000
    tokens = rng.integers(synth.OTHER_BASE, 8192, n).astype(np.int32)
    for s in (5, 1000, 2047, 2048, 4100, 9000, 15000, 19990):      # cue starts
        p = h.patterns[int(rng.integers(0, len(h.patterns)))]
        tokens[s:s + len(p)] = p
    tokens[13000] = synth.TERMINATOR_IDS[0]                          # one sentence end
    m = synth.make_margins(n, seed=83)
    _segment_custom(relay, tokens, [0, n], m, h)
    _segment_custom(relay, tokens, [0, 7000, 7000, 16000, n], m, h, think=[6000, 7000, 15500, n])


def test_segment_reduce_many_tiny_trajectories(relay):
    h = synth.make_cueset(4096, 3, 5, max_len=3, seed=84)
    ts = synth.make_tokens(3000, 7, h, seed=85, cue_rate=0.7, mean_sentence=3)
    m = synth.make_margins(ts.tokens.shape[0], seed=86, nan_rate=0.01)
    _segment_custom(relay, ts.tokens, ts.traj_offsets, m, h, think=ts.think_end_pos)
    _segment_custom(relay, ts.tokens, ts.traj_offsets, m, h, mode=1)


def test_segment_reduce_graph_replay_resets_lookback(relay):
    """K3's look-back flags are reset by the last tile: replays stay exact."""
    h, cs = _cs_pair(relay, 151936, 8, 12, 3, seed=87)
    ts = synth.make_tokens(2, 9000, h, seed=88)
    m = torch.as_tensor(synth.make_margins(ts.tokens.shape[0], seed=89), device=DEV)
    tok = torch.as_tensor(ts.tokens, device=DEV)
    offs = torch.as_tensor(ts.traj_offsets, device=DEV)
    ws = relay.workspace(tok.shape[0], tok.shape[0], 0, DEV)
    scan = relay.cue_scan(cs, tok, offs, ws=ws)
    first = relay.segment_reduce(cs, m, scan, offs, ws=ws)["stats"].clone()
    for _ in range(5):
        again = relay.segment_reduce(cs, m, scan, offs, ws=ws)["stats"]
        torch.cuda.synchronize()
        assert torch.equal(first, again)


# ------------------------------------------------- full BASELINE sizes
def test_c4_shape_sampled(relay):
    """configs[3] corpus on one GPU (8 x 32,768 x 151,936 bf16, 79.7 GB): the
    Analyzer pass; sampled rows vs the oracle; K2/K3 vs the oracle on two
    sampled trajectories (trajectories are independent)."""
    free = torch.cuda.mem_get_info()[0]
    if free < 95e9:
        pytest.skip("needs ~90 GB of free HBM")
    h, cs = _cs_pair(relay, 151936, 8, 12, 3, seed=91)
    ts = synth.make_tokens(8, 32768, h, seed=92)
    n = ts.tokens.shape[0]
    L = synth.make_logits(n, 151936, "bf16", tokens=ts.tokens, seed=93, device=DEV, chunk_rows=4096)
    an = relay.Analyzer(cs, n, 151936, DEV)
    an.run(L, torch.as_tensor(ts.tokens, device=DEV), torch.as_tensor(ts.traj_offsets, device=DEV),
           torch.as_tensor(ts.think_end_pos, device=DEV))
    torch.cuda.synchronize()
    rng = np.random.default_rng(94)
    rows = np.unique(np.concatenate([rng.choice(n, 60, replace=False), [0, 32767, 32768, n - 1]]))
    ref = oracle.margin_rows(synth.host_rows(L[torch.as_tensor(rows, device=DEV)], "bf16"), dtype="bf16",
                             threads=8)
    got_m = an.rows["margin"][torch.as_tensor(rows, device=DEV)].cpu().numpy()
    np.testing.assert_array_equal(an.rows["top1"][torch.as_tensor(rows, device=DEV)].cpu().numpy(), ref["top1"])
    np.testing.assert_array_equal(an.rows["top2"][torch.as_tensor(rows, device=DEV)].cpu().numpy(), ref["top2"])
    ok = ref["status"] == 0
    assert np.abs(got_m[ok] - ref["margin"][ok]).max() < TOL
    del L
    torch.cuda.empty_cache()
    # K2/K3 on the GPU margins' structure: occurrences and windows per sampled trajectory
    nocc = int(an.scan["n_occ"].item())
    occ = an.scan["occ_pos"][:nocc].cpu().numpy()
    ends = an.seg["seg_end"][:nocc].cpu().numpy()
    for k in (2, 7):
        a, b = int(ts.traj_offsets[k]), int(ts.traj_offsets[k + 1])
        o = oracle.cue_scan(ts.tokens[a:b], None, h.pat_tokens, h.pat_offsets, h.pat_cue, h.n_cues,
                            h.terminator)
        sel = (occ >= a) & (occ < b)
        np.testing.assert_array_equal(occ[sel] - a, o["occ_pos"])
        w = oracle.windows(np.zeros(b - a, np.float32), o["term"], None, o["occ_pos"], 0.5)
        np.testing.assert_array_equal(ends[sel] - a, w["seg_end"])


def test_c5_shape_streamed(relay):
    """configs[4]: 64 x 16,384 tokens, 32 patterns of length 1-6, logits
    streamed in 2,048-row chunks from a rotating pool (the 318 GB corpus never
    exists at once).  Sampled rows vs the oracle; K2/K3 (on synthetic margins)
    vs the oracle on three sampled trajectories."""
    V, R, K = 151936, 2048, 4
    h, cs = _cs_pair(relay, V, 32, 32, 6, seed=95, mode=0, min_len=1)
    ts = synth.make_tokens(64, 16384, h, seed=96)
    n = ts.tokens.shape[0]
    pool = [synth.make_logits(R, V, "bf16", seed=97 + i, device=DEV) for i in range(K)]
    an = relay.Analyzer(cs, n, V, DEV)
    chunks = ((c * R, pool[c % K]) for c in range(n // R))
    tok = torch.as_tensor(ts.tokens, device=DEV)
    offs = torch.as_tensor(ts.traj_offsets, device=DEV)
    an.run_streamed(chunks, tok, offs)
    torch.cuda.synchronize()
    rng = np.random.default_rng(98)
    rows = np.unique(np.concatenate([rng.choice(n, 40, replace=False), [0, n - 1]]))
    for r in rows.tolist():
        ref = oracle.margin_rows(synth.host_rows(pool[(r // R) % K][r % R:r % R + 1], "bf16"), dtype="bf16")
        assert an.rows["top1"][r].item() == ref["top1"][0] and an.rows["top2"][r].item() == ref["top2"][0]
        if ref["status"][0] == 0:
            assert abs(an.rows["margin"][r].item() - ref["margin"][0]) < TOL
    # stage-wise K2/K3 with synthetic margins on the full stream
    m = synth.make_margins(n, seed=99)
    seg = relay.segment_reduce(cs, torch.as_tensor(m, device=DEV), an.scan, offs, ws=an.ws)
    torch.cuda.synchronize()
    nocc = int(an.scan["n_occ"].item())
    occ = an.scan["occ_pos"][:nocc].cpu().numpy()
    pat = an.scan["occ_pat"][:nocc].cpu().numpy()
    ends = seg["seg_end"][:nocc].cpu().numpy()
    means = seg["seg_mean"][:nocc].cpu().numpy()
    for k in (0, 33, 63):
        a, b = int(ts.traj_offsets[k]), int(ts.traj_offsets[k + 1])
        o = oracle.cue_scan(ts.tokens[a:b], None, h.pat_tokens, h.pat_offsets, h.pat_cue, h.n_cues,
                            h.terminator)
        w = oracle.windows(m[a:b], o["term"], None, o["occ_pos"], 0.5)
        sel = (occ >= a) & (occ < b)
        np.testing.assert_array_equal(occ[sel] - a, o["occ_pos"])
        np.testing.assert_array_equal(pat[sel], o["occ_pat"])
        np.testing.assert_array_equal(ends[sel] - a, w["seg_end"])
        assert np.abs(means[sel] - w["seg_mean"]).max() < 1e-6


# ------------------------------------------- N1: vocabulary-parallel margin
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("P", [2, 3, 8])
def test_margin_tp_shards_equal_full_rows(relay, dtype, P):
    """Partials of P column shards, combined, equal the full-row result: the
    same indices and (within 1e-5) the oracle's margins."""
    V = 30011
    L = synth.make_logits(200, V, dtype, seed=P, device=DEV)
    bounds = np.linspace(0, V, P + 1).astype(int)
    parts = torch.stack([relay.margin_partials(L[:, a:b], int(a)) for a, b in zip(bounds[:-1], bounds[1:])])
    got = relay.margin_combine(parts)
    full = relay.margin_rows(L)
    torch.cuda.synchronize()
    ref = oracle.margin_rows(synth.host_rows(L, dtype), dtype=dtype, threads=8)
    np.testing.assert_array_equal(got["top1"].cpu().numpy(), ref["top1"])
    np.testing.assert_array_equal(got["top2"].cpu().numpy(), ref["top2"])
    np.testing.assert_array_equal(got["status"].cpu().numpy(), ref["status"].astype(np.uint8))
    ok = ref["status"] == 0
    assert np.abs(got["margin"].cpu().numpy()[ok] - ref["margin"][ok]).max() < TOL
    assert np.abs(got["margin"].cpu().numpy()[ok] - full["margin"].cpu().numpy()[ok]).max() < 2e-6


def test_margin_tp_edge_rows(relay):
    """Shards holding only -inf, NaN in one shard, top-1 tie across shards."""
    V = 64
    rows = torch.randn(6, V) * 2
    rows[0, :32] = float("-inf")                  # first shard empty
    rows[1, 40] = float("nan")                    # NaN in the second shard
    rows[2, 5] = 30.0; rows[2, 50] = 30.0         # tie across shards: lowest index wins
    rows[3, :] = float("-inf"); rows[3, 63] = 1.0
    rows[4, :] = 0.5                              # uniform
    L = rows.to(torch.bfloat16).to(DEV)
    parts = torch.stack([relay.margin_partials(L[:, :32], 0), relay.margin_partials(L[:, 32:], 32)])
    got = relay.margin_combine(parts)
    torch.cuda.synchronize()
    ref = oracle.margin_rows(synth.host_rows(L, "bf16"), dtype="bf16")
    np.testing.assert_array_equal(got["status"].cpu().numpy(), ref["status"].astype(np.uint8))
    np.testing.assert_array_equal(got["top1"].cpu().numpy(), ref["top1"])
    np.testing.assert_array_equal(got["top2"].cpu().numpy(), ref["top2"])


def _tp_worker(rank, world, port, out):
    import torch.distributed as dist
    import paper_2602_06454_b200 as relay
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    V = 20000
    L = synth.make_logits(96, V, "bf16", seed=5, device="cuda:0")
    a, b = rank * V // world, (rank + 1) * V // world
    res = relay.margin_rows_tp(L[:, a:b], a)
    if rank == 0:
        torch.save({k: v.cpu() for k, v in res.items()}, out)
    dist.destroy_process_group()


def test_margin_tp_two_ranks_gloo(relay, tmp_path):
    """margin_rows_tp over a 2-rank group (both ranks on cuda:0, gloo): the
    all-gather + combine path equals the full-row kernel."""
    import socket
    import torch.multiprocessing as mp
    sck = socket.socket(); sck.bind(("127.0.0.1", 0)); port = sck.getsockname()[1]; sck.close()
    out = str(tmp_path / "tp.pt")
    mp.spawn(_tp_worker, args=(2, port, out), nprocs=2, join=True)
    got = torch.load(out)
    L = synth.make_logits(96, 20000, "bf16", seed=5, device=DEV)
    full = relay.margin_rows(L)
    torch.cuda.synchronize()
    assert torch.equal(got["top1"], full["top1"].cpu()) and torch.equal(got["top2"], full["top2"].cpu())
    assert (got["margin"] - full["margin"].cpu()).abs().max().item() < 2e-6


def _tp_p2p_worker(rank, world, port, out):
    import torch.distributed as dist
    import paper_2602_06454_b200 as relay
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    V = 20011
    bounds = [k * V // world for k in range(world + 1)]
    a, b = bounds[rank], bounds[rank + 1]
    x = relay.TpExchange(rows_cap=200, group=dist.group.WORLD)
    res = []
    for call, (n, seed) in enumerate([(96, 5), (200, 6), (0, 7), (37, 8), (96, 9)]):
        L = synth.make_logits(max(n, 1), V, "bf16", seed=seed, device="cuda:0")[:n]
        o = x.margin_rows(L[:, a:b], a)
        torch.cuda.synchronize()
        res.append({k: v.cpu() for k, v in o.items()})
    if rank == 0:
        torch.save(res, out)
    dist.barrier()
    x.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_margin_tp_p2p_fused(relay, tmp_path, world):
    """relay_margin_rows_tp (the exchange fused into the streaming kernel over
    CUDA-IPC peer memory), world ranks as processes on cuda:0: five
    consecutive calls (both buffer parities, an empty call, row counts
    below and at rows_cap) each equal the full-row kernel."""
    import socket
    import torch.multiprocessing as mp
    sck = socket.socket(); sck.bind(("127.0.0.1", 0)); port = sck.getsockname()[1]; sck.close()
    out = str(tmp_path / "tp_p2p.pt")
    mp.spawn(_tp_p2p_worker, args=(world, port, out), nprocs=world, join=True)
    got = torch.load(out)
    for (n, seed), g in zip([(96, 5), (200, 6), (0, 7), (37, 8), (96, 9)], got):
        assert g["margin"].shape[0] == n
        if n == 0:
            continue
        L = synth.make_logits(n, 20011, "bf16", seed=seed, device=DEV)
        full = relay.margin_rows(L)
        torch.cuda.synchronize()
        assert torch.equal(g["top1"], full["top1"].cpu()) and torch.equal(g["top2"], full["top2"].cpu())
        assert torch.equal(g["status"], full["status"].cpu())
        ok = full["status"].cpu() == 0
        assert (g["margin"][ok] - full["margin"].cpu()[ok]).abs().max().item() < 2e-6


def test_margin_tp_p2p_single_rank(relay, tmp_path):
    """world 1: no peers; the fused path reduces to partial + combine on one GPU."""
    import socket
    import torch.multiprocessing as mp
    sck = socket.socket(); sck.bind(("127.0.0.1", 0)); port = sck.getsockname()[1]; sck.close()
    out = str(tmp_path / "tp_p2p1.pt")
    mp.spawn(_tp_p2p_worker, args=(1, port, out), nprocs=1, join=True)
    got = torch.load(out)
    L = synth.make_logits(96, 20011, "bf16", seed=5, device=DEV)
    full = relay.margin_rows(L)
    torch.cuda.synchronize()
    assert torch.equal(got[0]["top1"], full["top1"].cpu())


# ------------------------------------------------------ N3 offload estimate
def _offload_case(relay, h, ts, sel, mode=0, think=True):
    cs = relay.CueSet.from_synth(h, mode=mode)
    n = ts.tokens.shape[0]
    tok = torch.as_tensor(ts.tokens, device=DEV)
    offs = torch.as_tensor(ts.traj_offsets, device=DEV)
    tep = torch.as_tensor(ts.think_end_pos, device=DEV) if think else None
    m = synth.make_margins(n, seed=1)
    scan = relay.cue_scan(cs, tok, offs)
    seg = relay.segment_reduce(cs, torch.as_tensor(m, device=DEV), scan, offs, tep)
    got = relay.offload_estimate(cs, scan, seg, torch.as_tensor(sel, device=DEV), n, offs, tep)
    torch.cuda.synchronize()
    o_scan, o_win, _ = oracle.analyze(m, ts.tokens, ts.traj_offsets, h.pat_tokens, h.pat_offsets,
                                      h.pat_cue, h.n_cues, h.terminator, mode=mode, min_count=1)
    ref = oracle.offload(n, ts.traj_offsets, ts.think_end_pos if think else None, o_scan["occ_pos"],
                         o_scan["occ_pat"], o_win["seg_end"], h.pat_offsets, h.pat_cue, sel)
    np.testing.assert_array_equal(got.cpu().numpy(), ref)
    return ref


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("think", [True, False])
def test_offload_estimate(relay, mode, think):
    h = synth.make_cueset(8192, 6, 10, max_len=3, seed=111)
    ts = synth.make_tokens(9, 3000, h, seed=112, cue_rate=0.5)
    rng = np.random.default_rng(113)
    for _ in range(3):
        sel = (rng.random(6) < 0.5).astype(np.uint8)
        ref = _offload_case(relay, h, ts, sel, mode, think)
        assert (ref.sum(axis=1) == 3000).all()


def test_offload_estimate_golden(relay, golden_dir):
    import json
    import os
    g = json.load(open(os.path.join(golden_dir, "trace_fixture.json")))
    pats = g["patterns"]
    po = np.zeros(len(pats) + 1, np.int32)
    po[1:] = np.cumsum([len(p) for p in pats])
    term = np.zeros(g["vocab"], np.uint8)
    term[g["terminator_ids"]] = 1
    h = synth.CueSet(np.array([t for p in pats for t in p], np.int32), po, np.array(g["pat_cue"], np.int32),
                     g["n_cues"], g["vocab"], term, -1, [tuple(p) for p in pats])
    ts = synth.TokenStream(np.array(g["tokens"], np.int32), np.array(g["traj_offsets"], np.int64),
                           np.array([7, 12], np.int64))
    ref = _offload_case(relay, h, ts, np.array([1, 1], np.uint8))
    assert ref.tolist() == [[3, 4, 3], [2, 0, 1]]          # hand-traced case C


@pytest.mark.parametrize("case", [
    dict(n_traj=8, traj_len=4096, n_cues=8, n_pat=12, max_len=3, seed=41, think=True),
    dict(n_traj=5, traj_len=3001, n_cues=6, n_pat=20, max_len=6, seed=42, nan_rate=0.002),
    dict(n_traj=64, traj_len=700, n_cues=32, n_pat=32, max_len=6, seed=43, think=True),
    dict(n_traj=300, traj_len=37, n_cues=4, n_pat=8, max_len=3, seed=44),
])
def test_segment_reduce_per_trajectory_tables(relay, case):
    """Per-trajectory tables (P:476-494 calibration-size study): all merged
    equal the single table bit for bit, and a subset merged finalizes like the
    oracle run on just that subset of trajectories."""
    h, cs, ts, m, scan, seg, o_scan, o_win, o_sum = _segment_case(relay, **case)
    think = case.get("think", False)
    offs = torch.as_tensor(ts.traj_offsets, device=DEV)
    tep = torch.as_tensor(ts.think_end_pos, device=DEV) if think else None
    per = relay.segment_reduce(cs, torch.as_tensor(m, device=DEV), scan, offs, tep,
                               per_trajectory=True)
    torch.cuda.synchronize()
    n_traj = case["n_traj"]
    words = relay.stats_words(h.n_cues, 1)
    tabs = per["stats"].cpu().numpy()
    assert tabs.shape[0] == n_traj * words
    np.testing.assert_array_equal(relay.stats_merge(tabs, h.n_cues, 1),
                                  seg["stats"].cpu().numpy().view(np.uint64))
    rng = np.random.default_rng(case["seed"])
    mask = rng.random(n_traj) < 0.4
    mask[0] = True
    sub = relay.stats_merge(tabs, h.n_cues, 1, mask)
    keep = np.flatnonzero(mask)
    o = ts.traj_offsets
    toks = np.concatenate([ts.tokens[o[k]:o[k + 1]] for k in keep])
    mm = np.concatenate([m[o[k]:o[k + 1]] for k in keep])
    so = np.concatenate([[0], np.cumsum([o[k + 1] - o[k] for k in keep])]).astype(np.int64)
    ste = (np.array([ts.think_end_pos[k] - o[k] for k in keep], np.int64) + so[:-1]) if think else None
    _, _, r_sum = oracle.analyze(mm, toks, so, h.pat_tokens, h.pat_offsets, h.pat_cue, h.n_cues,
                                 h.terminator, tau=0.5, think_end_pos=ste, mode=0, min_count=1)
    fin = relay.stats_finalize(sub, h.n_cues, 1, min_count=1)
    for c in range(h.n_cues + 1):
        g, r = fin[c], r_sum[c]
        assert g["n"] == r["n"] and g["n_invalid"] == r["n_invalid"], (c, g, r)
        if c < h.n_cues:
            assert g["n_triggers"] == r["n_triggers"], (c, g, r)
        if r["n"] == 0:
            continue
        for f in ("mean", "token_mean", "min", "low_frac"):
            assert abs(g[f] - r[f]) < TOL, (c, f, g[f], r[f])


def test_analyzer_per_trajectory_tables(relay):
    """Analyzer with per-trajectory tables: merged, the same table as the
    one-table Analyzer on the same logits (bit for bit)."""
    vocab = 4096
    h, cs = _cs_pair(relay, vocab, 6, 10, 3, seed=51)
    ts = synth.make_tokens(6, 1500, h, seed=52)
    n_tok = ts.tokens.shape[0]
    logits = synth.make_logits(n_tok, vocab, "bf16", seed=53, device=DEV)
    tok = torch.as_tensor(ts.tokens, device=DEV)
    offs = torch.as_tensor(ts.traj_offsets, device=DEV)
    one = relay.Analyzer(cs, n_tok, vocab, DEV).run(logits, tok, offs).clone()
    per = relay.Analyzer(cs, n_tok, vocab, DEV, per_trajectory_tables=6).run(logits, tok, offs)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(relay.stats_merge(per.cpu().numpy(), 6, 1),
                                  one.cpu().numpy().view(np.uint64))


def test_stats_allreduce_library_comm(relay):
    """H6 through the C ABI on a one-rank library-owned NCCL communicator: the
    all-reduce of a real table is the identity (sum over one rank), in place,
    on the caller's stream."""
    vocab = 151936
    h, cs = _cs_pair(relay, vocab, 8, 12, 3, seed=61)
    ts = synth.make_tokens(4, 4096, h, seed=62)
    m = torch.as_tensor(synth.make_margins(ts.tokens.shape[0], seed=63), device=DEV)
    tok = torch.as_tensor(ts.tokens, device=DEV)
    offs = torch.as_tensor(ts.traj_offsets, device=DEV)
    st = relay.segment_reduce(cs, m, relay.cue_scan(cs, tok, offs), offs, per_trajectory=True)["stats"]
    before = st.clone()
    comm = relay.NcclComm(relay.nccl_unique_id(), 1, 0)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    relay.stats_allreduce(comm.ptr, st, 8, 1, n_tables=4, stream=s)
    s.synchronize()
    assert torch.equal(st, before)
    comm.close()


def test_stats_allreduce_torch_comm(relay, tmp_path):
    """H6 on torch's own ProcessGroupNCCL communicator (one rank): the dist
    helper routes CUDA tables through relay_stats_allreduce."""
    import torch.distributed as dist

    from paper_2602_06454_b200.dist import allreduce_stats, torch_nccl_comm
    if dist.is_initialized():
        pytest.skip("a process group already exists")
    dist.init_process_group("nccl", init_method=f"file://{tmp_path}/pg", rank=0, world_size=1,
                            device_id=torch.device(DEV))
    try:
        st = relay.new_stats(5, 0, 1, DEV)
        st[:] = torch.arange(st.numel(), device=DEV)
        ref = st.clone()
        assert torch_nccl_comm() != 0
        allreduce_stats(st, 5, 1)
        torch.cuda.synchronize()
        assert torch.equal(st, ref)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["strided", "flat", "dynamic", "hybrid", "cluster", "groups"])
@pytest.mark.parametrize("B,vocab,dtype", [(256, 152064, "bf16"), (37, 5003, "f16"), (300, 32000, "f32")])
def test_step_switch_work_split_modes(relay, monkeypatch, mode, B, vocab, dtype):
    """K4's work splits (whole rows per CTA; equal flat slices merged by the
    last arriver; dynamic chunks; hybrid: one whole row per SM plus equal
    slices of the rest; groups: one CTA per SM streaming two rows at once)
    all match the oracle, including graph replays that rely on the
    self-resetting counters."""
    if mode == "groups":
        monkeypatch.setenv("RELAY_K4_GROUPS", "1")
        mode = "strided"
    monkeypatch.setenv("RELAY_K4_MODE", mode)
    for greedy in (False, True):    # greedy: the switch reads the row's top-1 on every lane
        test_step_switch(relay, greedy, B, vocab, dtype, 0, -1.0)
    if B == 37:
        test_step_switch_graph_replay(relay)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("decimal", [False, True])
def test_class_patterns_and_decimal_rule(relay, mode, decimal):
    """N4: token-class pattern elements (K2 matching) and the decimal-number
    sentence rule (K2 terminator bits -> K3 windows and table) match the
    oracle exactly on a planted stream; several tiles and trajectories."""
    cc = synth.make_class_case(8192, 6, 2500, seed=91 + mode)
    dec = cc.decimal_rule if decimal else None
    cs = relay.CueSet(cc.cs.pat_tokens, cc.cs.pat_offsets, cc.cs.pat_cue, cc.cs.n_cues,
                      cc.cs.terminator, cc.cs.vocab, cc.cs.think_end, mode, cc.classes, dec)
    ts = cc.ts
    m = synth.make_margins(ts.tokens.shape[0], seed=93)
    tok = torch.as_tensor(ts.tokens, device=DEV)
    offs = torch.as_tensor(ts.traj_offsets, device=DEV)
    tep = torch.as_tensor(ts.think_end_pos, device=DEV)
    scan = relay.cue_scan(cs, tok, offs)
    seg = relay.segment_reduce(cs, torch.as_tensor(m, device=DEV), scan, offs, tep)
    torch.cuda.synchronize()
    o_scan, o_win, o_sum = oracle.analyze(m, ts.tokens, ts.traj_offsets, cc.cs.pat_tokens,
                                          cc.cs.pat_offsets, cc.cs.pat_cue, cc.cs.n_cues,
                                          cc.cs.terminator, think_end_pos=ts.think_end_pos,
                                          mode=mode, min_count=1, classes=cc.classes,
                                          decimal_rule=dec)
    n = int(scan["n_occ"].item())
    assert n == o_scan["occ_pos"].shape[0] and n > 50
    np.testing.assert_array_equal(scan["occ_pos"][:n].cpu().numpy(), o_scan["occ_pos"])
    np.testing.assert_array_equal(scan["occ_pat"][:n].cpu().numpy(), o_scan["occ_pat"])
    bits = scan["term_bits"].cpu().numpy().view(np.uint32)
    got_term = (bits[np.arange(ts.tokens.shape[0]) >> 5] >> (np.arange(ts.tokens.shape[0]) & 31)) & 1
    np.testing.assert_array_equal(got_term, o_scan["term"])
    if decimal:   # the rule really removed sentence ends
        assert (o_scan["term"] < cc.cs.terminator[ts.tokens]).sum() > 10
    _compare_segments(relay, cc.cs, scan, seg, o_scan, o_win, o_sum)


@pytest.mark.parametrize("greedy", [False, True])
def test_step_switch_class_patterns(relay, greedy):
    """K4 completes class-valued patterns like the oracle's step rule."""
    cc = synth.make_class_case(32000, 1, 64, seed=95)
    h = cc.cs
    cs = relay.CueSet(h.pat_tokens, h.pat_offsets, h.pat_cue, h.n_cues, h.terminator, h.vocab,
                      h.think_end, 0, cc.classes)
    rng = np.random.default_rng(96)
    B = 200
    members = [np.flatnonzero(cc.classes[c]) for c in range(cc.classes.shape[0])]
    hist = np.full((B, 7), -1, np.int32)
    sampled = rng.integers(3000, 32000, B).astype(np.int32)
    for b in range(B):           # hist = a pattern instance minus its last element
        p = h.patterns[int(rng.integers(0, len(h.patterns)))]
        inst = [e if e >= 0 else int(rng.choice(members[-1 - e])) for e in p]
        if len(inst) > 1:
            hist[b, 7 - (len(inst) - 1):] = inst[:-1]
        if rng.random() < 0.7:
            sampled[b] = inst[-1]
    state = np.zeros(B, np.uint8)
    small_run = np.zeros(B, np.int32)
    L = synth.make_logits(B, 32000, "bf16", tokens=sampled, seed=97, device=DEV)
    ref = oracle.margin_rows(synth.host_rows(L, "bf16"), dtype="bf16")
    d_state = torch.as_tensor(state, device=DEV)
    d_hist = torch.as_tensor(hist, device=DEV)
    d_sr = torch.as_tensor(small_run, device=DEV)
    out = relay.step_switch(cs, L, d_state, d_hist, d_sr,
                            None if greedy else torch.as_tensor(sampled, device=DEV))
    torch.cuda.synchronize()
    n_l2s = 0
    for b in range(B):
        tok = int(ref["top1"][b]) if greedy else int(sampled[b])
        f, c, st, hh, sr = oracle.step_one(tok, np.float32(ref["margin"][b]), 0, hist[b], 0,
                                           h.pat_tokens, h.pat_offsets, h.pat_cue, h.terminator,
                                           h.think_end, classes=cc.classes)
        assert out["flag"][b].item() == f and out["cue_id"][b].item() == c, b
        assert d_state[b].item() == st
        np.testing.assert_array_equal(d_hist[b].cpu().numpy(), hh)
        n_l2s += f == 1
    assert n_l2s > 50


# ---------------------------------------------------------------- N2 sampler
def _oracle_sample_tolerant(host_rows, dtype, vocab, u, got, T, k, p):
    """Oracle draws; where the kernel's fp32 draw differs, it must be the
    oracle's draw for a uniform or top_p within 1e-5 (a CDF edge)."""
    want = oracle.sample_rows(host_rows, u, dtype=dtype, vocab=vocab, temperature=T, top_k=k, top_p=p)
    bad = np.flatnonzero(want != got)
    for b in bad:
        alts = set()
        for du in (-1e-5, 1e-5):
            for dp in (0.0, -1e-5, 1e-5):
                uu = min(max(u[b] + du, 0.0), 1 - 1e-12)
                pp = min(max(p + dp, 1e-9), 1.0)
                alts.add(int(oracle.sample_rows(host_rows[b:b + 1], [uu], dtype=dtype, vocab=vocab,
                                                temperature=T, top_k=k, top_p=pp)[0]))
        assert int(got[b]) in alts, (b, int(got[b]), int(want[b]), alts)
    return want, bad.size


@pytest.mark.parametrize("B,vocab,dtype,T,k,p", [
    (256, 152064, "bf16", 0.6, 20, 0.95),     # configs[2] with the paper's Qwen3 sampling
    (64, 151936, "bf16", 0.6, 64, 1.0),
    (37, 5003, "f16", 1.0, 1, 0.95),
    (50, 32000, "f32", 0.6, 20, 0.5),
    (9, 40, "f32", 0.8, 64, 0.9),             # vocab < top_k
    (256, 152064, "bf16", 0.6, 0, 0.95),      # configs[2] with R1-Distill sampling: no top-k
    (1000, 8192, "bf16", 0.6, 20, 0.95),      # more rows than CTAs: K4/K5 loop rows per CTA
    (1000, 8192, "bf16", 0.6, 0, 0.95),
    (37, 5003, "f16", 1.0, 0, 1.0),
    (50, 32000, "f32", 0.6, 0, 0.5),
])
def test_step_sample(relay, B, vocab, dtype, T, k, p):
    """N2: the drawn token matches the oracle sampler (R20); margins/indices as
    K1/K4; the switch runs on the drawn token."""
    if vocab > 4096:
        h, cs = _cs_pair(relay, vocab, 4, 8, 3, seed=71)
    else:                                   # tiny vocabulary: a tiny cue set
        term = np.zeros(vocab, np.uint8)
        term[3] = 1
        h = synth.CueSet(np.array([1, 2, 5], np.int32), np.array([0, 2, 3], np.int32),
                         np.array([0, 1], np.int32), 2, vocab, term, vocab - 1, [(1, 2), (5,)])
        cs = relay.CueSet.from_synth(h)
    rng = np.random.default_rng(72)
    L = synth.make_logits(B, vocab, dtype, seed=73, device=DEV)
    host = synth.host_rows(L, dtype)
    u = rng.random(B).astype(np.float32)
    state = np.zeros(B, np.uint8)
    hist = np.full((B, 7), -1, np.int32)
    d_state = torch.as_tensor(state, device=DEV)
    d_hist = torch.as_tensor(hist, device=DEV)
    out = relay.step_sample(cs, L, torch.as_tensor(u, device=DEV), d_state, d_hist, temperature=T,
                            top_k=k, top_p=p)
    torch.cuda.synchronize()
    ref = oracle.margin_rows(host, dtype=dtype, vocab=vocab)
    np.testing.assert_array_equal(out["top1"].cpu().numpy(), ref["top1"])
    np.testing.assert_array_equal(out["top2"].cpu().numpy(), ref["top2"])
    ok = ref["status"] == 0
    assert np.abs(out["margin"].cpu().numpy()[ok] - ref["margin"][ok]).max() < TOL
    got = out["sampled"].cpu().numpy()
    want, n_edge = _oracle_sample_tolerant(host, dtype, vocab, u.astype(np.float64), got, T, k, p)
    assert n_edge <= max(1, B // 50)
    assert (got[~ok] == -1).all()
    if k == 1:
        np.testing.assert_array_equal(got[ok], ref["top1"][ok])
    if k == 0:   # the rows whose nucleus is wider than 64 tokens took the slow path
        assert len(set(got[ok].tolist())) > 1
    # the switch saw the drawn token
    flags = out["flag"].cpu().numpy()
    for b in range(B):
        f, c, st, hh, sr = oracle.step_one(int(got[b]), np.float32(ref["margin"][b]), 0, hist[b], 0,
                                           h.pat_tokens, h.pat_offsets, h.pat_cue, h.terminator,
                                           h.think_end)
        assert flags[b] == f and d_state[b].item() == st


@pytest.mark.parametrize("B,vocab,dtype,T,k,p", [
    (256, 152064, "bf16", 0.6, 20, 0.95),     # configs[2], Qwen3 sampling
    (1000, 8192, "bf16", 0.6, 20, 0.95),      # rows per CTA > 1: both candidate lists alternate
    (200, 32000, "f32", 1.0, 64, 1.0),        # top-k 64: lists overflow, rows go to K5
    (37, 5003, "f16", 0.8, 5, 0.9),
])
def test_step_sample_fused_draw(relay, monkeypatch, B, vocab, dtype, T, k, p):
    """The opt-in fused top-k draw in K4 (RELAY_K4_FUSE=1): the same checks as
    test_step_sample (drawn tokens vs the oracle sampler, the switch on them)."""
    monkeypatch.setenv("RELAY_K4_FUSE", "1")
    test_step_sample(relay, B, vocab, dtype, T, k, p)


def test_step_sample_pathological_rows(relay):
    """A constant row (every logit a candidate: the exact fallback), rows with
    -inf tails, a NaN row, and the distribution of draws on a constant row."""
    vocab, B = 5000, 64
    h, cs = _cs_pair(relay, vocab, 2, 4, 2, seed=75)
    rows = np.random.default_rng(76).normal(0, 1, (B, vocab)).astype(np.float32)
    rows[0] = 1.25                        # constant: top-k = the first k indices
    rows[1, 30:] = -np.inf                # only 30 finite entries
    rows[2, :] = -np.inf
    rows[2, [7, 4000]] = [0.0, 0.0]       # two finite, tied
    rows[3, 11] = np.nan
    u = (np.arange(B) + 0.5) / B
    u = u.astype(np.float32)
    L = torch.as_tensor(rows, device=DEV)
    st = torch.zeros(B, dtype=torch.uint8, device=DEV)
    hi = torch.full((B, 7), -1, dtype=torch.int32, device=DEV)
    out = relay.step_sample(cs, L, torch.as_tensor(u, device=DEV), st, hi, temperature=0.6,
                            top_k=20, top_p=0.95)
    torch.cuda.synchronize()
    got = out["sampled"].cpu().numpy()
    _oracle_sample_tolerant(rows, "f32", vocab, u.astype(np.float64), got, 0.6, 20, 0.95)
    assert got[3] == -1 and got[2] in (7, 4000) and 0 <= got[0] < 20 and 0 <= got[1] < 30
    # constant row, many uniforms: uniform over the first ceil(0.95 * 20) = 19 indices
    many = np.tile(rows[0], (B, 1))
    out2 = relay.step_sample(cs, torch.as_tensor(many, device=DEV), torch.as_tensor(u, device=DEV),
                             st.zero_(), hi.fill_(-1), temperature=0.6, top_k=20, top_p=0.95)
    torch.cuda.synchronize()
    g2 = out2["sampled"].cpu().numpy()
    assert set(g2.tolist()) <= set(range(19)) and len(set(g2.tolist())) >= 17


def test_step_sample_no_top_k_pathological_rows(relay):
    """No top-k: a constant row (every entry one value: the kept ties and the
    draw are resolved in index order), flat and sparse rows, NaN rows."""
    vocab, B = 5000, 24
    h, cs = _cs_pair(relay, vocab, 2, 4, 2, seed=85)
    rng = np.random.default_rng(86)
    rows = rng.normal(0, 0.3, (B, vocab)).astype(np.float32)   # flat: wide nuclei
    rows[0] = 1.25
    rows[1] = np.repeat(rng.normal(0, 1, 50), 100).astype(np.float32)   # blocks of ties
    rows[2, 30:] = -np.inf
    rows[3, 11] = np.nan
    u = rng.random(B).astype(np.float32)
    st = torch.zeros(B, dtype=torch.uint8, device=DEV)
    hi = torch.full((B, 7), -1, dtype=torch.int32, device=DEV)
    for p in (0.95, 0.3, 1.0):
        out = relay.step_sample(cs, torch.as_tensor(rows, device=DEV), torch.as_tensor(u, device=DEV),
                                st.zero_(), hi.fill_(-1), temperature=0.6, top_k=0, top_p=p)
        torch.cuda.synchronize()
        got = out["sampled"].cpu().numpy()
        _oracle_sample_tolerant(rows, "f32", vocab, u.astype(np.float64), got, 0.6, 0, p)
        assert got[3] == -1


@pytest.mark.parametrize("dtype", ["bf16", "f16"])
def test_step_sample_no_top_k_16bit_rows(relay, dtype):
    """No top-k on 16-bit rows (the exact-key nucleus path): flat rows whose
    nucleus spans thousands of tied values, a range crossing zero (keys span
    every tiny binade: level-2 bins), large logits (one key per level-1 bin),
    constant and tied-block rows, -0/+0 ties, sparse and NaN rows."""
    vocab, B = 152064, 16
    h, cs = _cs_pair(relay, vocab, 2, 4, 2, seed=87)
    rng = np.random.default_rng(88)
    rows = rng.normal(0, 2.5, (B, vocab)).astype(np.float32)
    rows[0] = 1.25                                            # constant
    rows[1] = rng.normal(0, 0.05, vocab)                      # flat around 0
    rows[2] = rng.normal(0, 0.05, vocab) + 30.0               # flat, large values
    rows[3] = np.repeat(rng.normal(0, 1, 1188), 128)[:vocab]  # blocks of ties
    rows[4] = rng.normal(0, 1.0, vocab) * 0.3                 # small z1: keys cross zero
    rows[5] = np.where(rng.random(vocab) < 0.5, -0.0, 0.0)    # -0 / +0 ties (IEEE equal)
    rows[5, 100:110] = 0.5
    rows[6, 40:] = -np.inf                                    # sparse
    rows[7, 11] = np.nan
    rows[8] = rng.normal(0, 2.5, vocab) + 40.0                # large logits, wide nucleus
    rows[9] = np.linspace(-1, 1, vocab)[::-1]                 # strictly descending
    L = torch.as_tensor(rows, device=DEV).to(torch.bfloat16 if dtype == "bf16" else torch.float16)
    host = synth.host_rows(L, dtype)
    u = rng.random(B).astype(np.float32)
    u[:3] = [0.0, 0.999999, 0.5]
    st = torch.zeros(B, dtype=torch.uint8, device=DEV)
    hi = torch.full((B, 7), -1, dtype=torch.int32, device=DEV)
    for p in (0.95, 0.3, 1.0):
        out = relay.step_sample(cs, L, torch.as_tensor(u, device=DEV), st.zero_(), hi.fill_(-1),
                                temperature=0.6, top_k=0, top_p=p)
        torch.cuda.synchronize()
        got = out["sampled"].cpu().numpy()
        _oracle_sample_tolerant(host, dtype, vocab, u.astype(np.float64), got, 0.6, 0, p)
        assert got[7] == -1 and 0 <= got[6] < 40


@pytest.mark.parametrize("dtype,T,p", [("bf16", 0.6, 0.95), ("bf16", 1.0, 0.5), ("bf16", 0.6, 1.0),
                                       ("f32", 0.6, 0.95), ("f16", 1.0, 0.9)])
def test_step_sample_no_top_k_wide_nuclei(relay, dtype, T, p):
    """No top-k on rows whose kept set reaches far past the top 64 (every row
    takes the nucleus kernel K6): logits of scale 0.3-3 around offsets that
    put z1 below and above the lump / key-range limits; the drawn token
    matches the oracle sampler except at CDF edges."""
    vocab, B = 32000, 96
    h, cs = _cs_pair(relay, vocab, 2, 4, 2, seed=89)
    rng = np.random.default_rng(90)
    scale = rng.choice([0.3, 0.8, 1.5, 3.0], B)[:, None]
    shift = rng.choice([-20.0, 0.0, 5.0, 40.0], B)[:, None]
    rows = (rng.normal(0, 1, (B, vocab)) * scale + shift).astype(np.float32)
    tdt = {"bf16": torch.bfloat16, "f16": torch.float16, "f32": torch.float32}[dtype]
    L = torch.as_tensor(rows, device=DEV).to(tdt)
    host = synth.host_rows(L, dtype)
    u = rng.random(B).astype(np.float32)
    st = torch.zeros(B, dtype=torch.uint8, device=DEV)
    hi = torch.full((B, 7), -1, dtype=torch.int32, device=DEV)
    out = relay.step_sample(cs, L, torch.as_tensor(u, device=DEV), st, hi, temperature=T, top_k=0, top_p=p)
    torch.cuda.synchronize()
    got = out["sampled"].cpu().numpy()
    want, n_edge = _oracle_sample_tolerant(host, dtype, vocab, u.astype(np.float64), got, T, 0, p)
    assert n_edge <= 2
    assert len(set(got.tolist())) > B // 2      # wide nuclei: mostly distinct draws


@pytest.mark.parametrize("top_k", [20, 0])
def test_step_sample_graph_replay(relay, top_k):
    """Captured in a CUDA graph (PDL edges included) and replayed with new
    uniforms: every replay matches the oracle (top_k 0: K6 and its
    self-re-arming list, with flat rows that take it, and the per-row
    readiness counters across replays)."""
    vocab, B = 32000, 48
    h, cs = _cs_pair(relay, vocab, 4, 6, 3, seed=77)
    L = synth.make_logits(B, vocab, "bf16", seed=78, device=DEV)
    if top_k == 0:
        L[::5] = (torch.randn(len(range(0, B, 5)), vocab, device=DEV) * 0.5).to(L.dtype)  # wide nuclei
    host = synth.host_rows(L, "bf16")
    d_u = torch.zeros(B, dtype=torch.float32, device=DEV)
    st = torch.zeros(B, dtype=torch.uint8, device=DEV)
    hi = torch.full((B, 7), -1, dtype=torch.int32, device=DEV)
    ws = relay.workspace(0, 0, B, DEV)
    out = relay.step_sample(cs, L, d_u, st, hi, top_k=top_k, ws=ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            relay.step_sample(cs, L, d_u, st, hi, top_k=top_k, ws=ws, out=out)
    torch.cuda.synchronize()
    rng = np.random.default_rng(79)
    for _ in range(4):
        u = rng.random(B).astype(np.float32)
        d_u.copy_(torch.as_tensor(u, device=DEV))
        st.zero_(); hi.fill_(-1)
        g.replay()
        torch.cuda.synchronize()
        _oracle_sample_tolerant(host, "bf16", vocab, u.astype(np.float64), out["sampled"].cpu().numpy(),
                                0.6, top_k, 0.95)


def test_read_probe_runs(relay):
    """relay_read_probe (bench.py's read-only ceiling) streams buffers of any
    multiple-of-16 size, including one smaller than a TMA chunk."""
    for n in (16, 4096, 32768 * 7 + 48, 50_000_000):
        buf = torch.ones(n // 2, dtype=torch.bfloat16, device=DEV)
        out = relay.read_probe(buf)
        torch.cuda.synchronize()
        assert out.numel() == relay._lib.relay_read_probe_words()
