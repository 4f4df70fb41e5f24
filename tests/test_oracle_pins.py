"""Pins for the CPU oracle (no GPU): the oracle checked against what the paper
and the mathematics fix, never against itself.

Each test names what pins it: a worked example (SPEC.md S:n or PAPER.md P:n),
a closed form, an invariance, a hand-traced golden file, or brute force on
tiny inputs computed here by a *different* procedure (sorting + math.fsum,
set enumeration) than the oracle's plain loops.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle

NINF = float("-inf")


def _f(x):
    return float(x) if not isinstance(x, str) else float(x.replace("inf", "inf"))


# ------------------------------------------------------------------ H1 margin
def test_golden_rows(golden_dir):
    """tests/golden/margin_rows.json: S:58-60 worked examples + hand closed forms."""
    g = json.load(open(os.path.join(golden_dir, "margin_rows.json")))
    for r in g["rows"]:
        z = np.array([float(v) for v in r["z"]], np.float32)
        st, i1, i2, m, _ = oracle.margin_row(z)
        assert (st, i1, i2) == (r["status"], r["i1"], r["i2"]), r
        if r["margin"] == "nan":
            assert math.isnan(m)
        else:
            assert abs(m - r["margin"]) < 1e-9, (r, m)


def test_length_one_row_is_invalid():
    with pytest.raises(ValueError):
        oracle.margin_row(np.array([1.0], np.float32))


def test_closed_form_two_entries():
    """V = 2 with gap d: p1 - p2 = (1 - e^-d)/(1 + e^-d) = tanh(d/2) (algebra on P:142)."""
    rng = np.random.default_rng(1)
    for _ in range(200):
        a, b = (float(x) for x in rng.normal(0, 4, 2).astype(np.float32))
        st, i1, i2, m, lse = oracle.margin_row(np.array([a, b], np.float32))
        d = abs(float(a) - float(b))
        assert abs(m - math.tanh(d / 2)) < 1e-12
        assert i1 == (0 if a >= b else 1) and i2 == 1 - i1
        assert abs(lse - (max(a, b) + math.log1p(math.exp(-d)))) < 1e-12


def _brute(z):
    """Brute force: order all entries by (value desc, index asc) with a sort and
    sum the softmax with math.fsum (a different procedure from the oracle's)."""
    order = sorted(range(len(z)), key=lambda j: (-z[j], j))
    i1, i2 = order[0], order[1]
    M = z[i1]
    S = math.fsum(math.exp(v - M) for v in z if v != NINF)
    p2 = 0.0 if z[i2] == NINF else math.exp(z[i2] - M) / S
    return i1, i2, 1.0 / S - p2


def test_brute_force_small_rows():
    """Tiny rows full of ties and -inf entries vs the sort-based brute force."""
    rng = np.random.default_rng(2)
    for _ in range(3000):
        V = int(rng.integers(2, 10))
        z = rng.integers(-3, 4, V).astype(np.float32)
        z[rng.random(V) < 0.15] = NINF
        if np.all(np.isneginf(z)):
            continue
        st, i1, i2, m, _ = oracle.margin_row(z)
        bi1, bi2, bm = _brute([float(v) for v in z])
        assert st == 0 and (i1, i2) == (bi1, bi2), (z, i1, i2, bi1, bi2)
        assert abs(m - bm) < 1e-12


def test_range_and_bounds():
    """0 <= m <= p1 <= 1."""
    rng = np.random.default_rng(3)
    for _ in range(300):
        z = rng.normal(0, 3, int(rng.integers(2, 300))).astype(np.float32)
        st, i1, i2, m, lse = oracle.margin_row(z)
        p1 = math.exp(float(z[i1]) - lse)
        assert 0.0 <= m <= p1 + 1e-15 <= 1.0 + 1e-15


def test_uniform_and_one_hot():
    """Uniform -> m = 0, i1 = 0, i2 = 1; one finite entry -> m = 1 (north_star pins)."""
    for V in (2, 7, 151936):
        st, i1, i2, m, _ = oracle.margin_row(np.full(V, 0.25, np.float32))
        assert (st, i1, i2, m) == (0, 0, 1, 0.0)
        z = np.full(V, NINF, np.float32)
        z[V // 2] = 3.0
        st, i1, i2, m, _ = oracle.margin_row(z)
        assert (st, i1, m) == (0, V // 2, 1.0) and i2 == (0 if V // 2 else 1)
    z = np.zeros(151936, np.float32)
    z[5] = 100.0
    assert oracle.margin_row(z)[3] == 1.0          # 1 - 5.65e-39 rounds to 1


def test_shift_invariance_and_permutation():
    """softmax(z + c) = softmax(z) (exact for small-integer fp32 logits); a
    permutation of the entries permutes i1/i2 (ties aside)."""
    rng = np.random.default_rng(4)
    for _ in range(200):
        V = int(rng.integers(3, 50))
        z = rng.permutation(V).astype(np.float32) - V // 2        # distinct integers
        c = float(rng.integers(-20, 20))
        a = oracle.margin_row(z)
        b = oracle.margin_row(z + np.float32(c))
        assert a[1:3] == b[1:3] and abs(a[3] - b[3]) < 1e-12
        perm = rng.permutation(V)
        p = oracle.margin_row(z[perm])
        assert perm[p[1]] == a[1] and perm[p[2]] == a[2] and abs(p[3] - a[3]) < 1e-12


def test_tail_entries_only_change_S():
    """Appending entries below the top 2 leaves i1, i2 and p1-p2 = (1-e^-d)/S
    with the enlarged S (S:91 'invariant under appending' holds for p-lists;
    for logits the normaliser grows): check against the closed form."""
    z = np.array([5.0, 4.0], np.float32)
    ext = np.concatenate([z, np.array([1.0, 0.0, -2.0], np.float32)])
    st, i1, i2, m, _ = oracle.margin_row(ext)
    S = 1 + math.exp(-1) + math.exp(-4) + math.exp(-5) + math.exp(-7)
    assert (i1, i2) == (0, 1) and abs(m - (1 - math.exp(-1)) / S) < 1e-12


def test_temperature_is_scaling():
    """inv_temperature iota: softmax(z * iota) == softmax of the scaled row."""
    rng = np.random.default_rng(5)
    z = rng.integers(-8, 8, 40).astype(np.float32)
    a = oracle.margin_row(z, inv_temperature=2.0)
    b = oracle.margin_row(z * np.float32(2.0))
    assert a[:3] == b[:3] and abs(a[3] - b[3]) < 1e-12


def test_16bit_decoding_matches_numpy():
    """bf16 = top half of binary32; f16 decoded by numpy's own float16."""
    rng = np.random.default_rng(6)
    bits = rng.integers(0, 1 << 16, 4000).astype(np.uint16)
    f16 = bits.view(np.float16).astype(np.float64)
    bf = (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    # decode through the oracle: a 2-entry row [x, -inf] gives status/i1 and lse = x
    ninf_f16, ninf_bf = np.uint16(0xFC00), np.uint16(0xFF80)
    for k in range(0, 4000, 7):
        for vals, code, ninf in ((f16, "f16", ninf_f16), (bf, "bf16", ninf_bf)):
            x = vals[k]
            st, i1, i2, m, lse = oracle.margin_row(np.array([bits[k], ninf], np.uint16), dtype=code)
            if np.isnan(x) or (np.isinf(x) and x > 0):
                assert st == 1
            elif np.isinf(x):
                assert st == 2
            else:
                assert st == 0 and i1 == 0 and lse == x


def test_row_stride_skips_nan_padding():
    """oracle_margin_rows with row_stride > vocab (VERDICT r01 nit): the
    padding columns hold NaN, so reading one would make the row status 1; every
    row must equal the sort + math.fsum brute force on its first `vocab`
    entries, for f32 and for bf16 / f16 bit patterns, at several strides."""
    rng = np.random.default_rng(17)
    for vocab, stride in ((5, 8), (7, 7 + 1), (33, 40), (2, 9)):
        z = rng.integers(-4, 5, (23, vocab)).astype(np.float32)
        z[rng.random(z.shape) < 0.1] = NINF
        z[np.all(np.isneginf(z), axis=1), 0] = 1.0
        pad = np.full((23, stride), np.nan, np.float32)
        pad[:, :vocab] = z
        bits = (pad.view(np.uint32) >> 16).astype(np.uint16)       # bf16: exact for these small integers
        h16 = pad.astype(np.float16).view(np.uint16)
        for arr, code in ((pad, None), (bits, "bf16"), (h16, "f16")):
            got = oracle.margin_rows(arr, dtype=code, vocab=vocab)
            for r in range(23):
                i1, i2, m = _brute([float(v) for v in z[r]])
                assert got["status"][r] == 0, (vocab, stride, code, r)
                assert (got["top1"][r], got["top2"][r]) == (i1, i2)
                assert abs(got["margin"][r] - m) < 1e-12


def test_threads_do_not_change_results():
    rng = np.random.default_rng(7)
    L = rng.normal(0, 2, (37, 513)).astype(np.float32)
    a = oracle.margin_rows(L, threads=1)
    b = oracle.margin_rows(L, threads=5)
    for k in a:
        np.testing.assert_array_equal(a[k], b[k])


# --------------------------------------------------------- golden trace H2-H7
def _cs_from_fixture(g):
    pats = g["patterns"]
    offs = np.zeros(len(pats) + 1, np.int32)
    offs[1:] = np.cumsum([len(p) for p in pats])
    term = np.zeros(g["vocab"], np.uint8)
    term[g["terminator_ids"]] = 1
    return (np.array([t for p in pats for t in p], np.int32), offs,
            np.array(g["pat_cue"], np.int32), term)


def test_golden_trace(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "trace_fixture.json")))
    pt, po, pc, term = _cs_from_fixture(g)
    m = np.array(g["margins"], np.float32)
    for min_count, key in ((1, "selected_rule0_min_count_1"), (3, "selected_rule0_min_count_3")):
        scan, win, summ = oracle.analyze(m, g["tokens"], g["traj_offsets"], pt, po, pc,
                                         g["n_cues"], term, tau=g["tau"], min_count=min_count)
        occ = g["occurrences"]
        assert scan["occ_pos"].tolist() == [o["s"] for o in occ]
        assert scan["occ_pat"].tolist() == [o["pat"] for o in occ]
        assert win["seg_end"].tolist() == [o["e"] for o in occ]
        for k, o in enumerate(occ):
            # margins are fp32 inputs: 1e-7 covers their rounding
            assert abs(win["seg_mean"][k] - o["mean"]) < 1e-7
            assert abs(win["seg_min"][k] - o["min"]) < 1e-7
            assert abs(win["seg_lowfrac"][k] - o["lowfrac"]) < 1e-12
        for c, e in enumerate(g["cues"]):
            s = summ[c]
            assert s["n"] == e["n"] and s["n_triggers"] == e["n_triggers"]
            for f in ("mean", "std", "se", "token_mean", "min", "low_frac"):
                assert abs(s[f] - e[f]) < 2e-7, (c, f, s[f], e[f])
        gl = summ[-1]
        for f in ("mean", "std", "se", "min", "low_frac"):
            assert abs(gl[f] - g["global"][f]) < 2e-7, (f, gl[f])
        assert gl["n"] == g["global"]["n"]
        assert [s["selected"] for s in summ[:-1]] == g[key]


# ---------------------------------------------------------- SPEC stats pins
def _one_traj_stats(margins, cue_positions, term_positions=(), tau=0.5, min_count=1, rule=0):
    """Drive cue_stats with cue occurrences at given positions (single pattern)."""
    n = len(margins)
    term = np.zeros(n, np.uint8)
    term[list(term_positions)] = 1
    occ = np.array(cue_positions, np.int32)
    win = oracle.windows(np.array(margins, np.float32), term, None, occ, tau)
    summ = oracle.cue_stats(np.array(margins, np.float32), None, None, occ,
                            np.zeros(len(occ), np.int32), np.array([0], np.int32), 1, tau, win,
                            min_count, rule)
    return win, summ


@pytest.mark.parametrize("vals,mean,std,se", [
    ([0.0, 1.0], 0.5, 0.5, 0.35355339),
    ([0.2, 0.4, 0.6, 0.8], 0.5, 0.22360680, 0.11180340),
    ([0.5, 0.5, 0.5], 0.5, 0.0, 0.0),
])
def test_global_stats_spec_examples(vals, mean, std, se):
    _, summ = _one_traj_stats(vals, [])
    g = summ[-1]
    assert abs(g["mean"] - mean) < 1e-7 and abs(g["std"] - std) < 1e-7 and abs(g["se"] - se) < 1e-7


def test_global_needs_two_positions():
    _, summ = _one_traj_stats([0.3], [])
    assert math.isnan(summ[-1]["se"]) and summ[0]["selected"] == 0


def test_window_spec_examples():
    """S:223-225."""
    w, _ = _one_traj_stats([0.1, 0.7], [1])
    assert w["seg_end"][0] == 1 and abs(w["seg_mean"][0] - 0.7) < 1e-7
    w, _ = _one_traj_stats([0.2, 0.4, 0.6, 0.9], [0], term_positions=[2])
    assert w["seg_end"][0] == 2 and abs(w["seg_mean"][0] - 0.4) < 1e-7
    w, _ = _one_traj_stats([0.9, 0.1, 0.3], [1])
    assert w["seg_end"][0] == 2 and abs(w["seg_mean"][0] - 0.2) < 1e-7


def test_per_cue_spec_examples():
    """window means {0.4, 0.6} -> mean 0.5, SE 0.0707; single 0.8 -> SE 0."""
    # two one-token sentences (each cue token is its own terminator)
    _, summ = _one_traj_stats([0.4, 0.6, 0.5], [0, 1], term_positions=[0, 1])
    c = summ[0]
    assert c["n"] == 2 and abs(c["mean"] - 0.5) < 1e-7 and abs(c["se"] - 0.07071068) < 1e-7
    _, summ = _one_traj_stats([0.8, 0.2], [0], term_positions=[0])
    assert summ[0]["n"] == 1 and abs(summ[0]["mean"] - 0.8) < 1e-7 and summ[0]["se"] == 0.0


# dyadic fixture: mu = 9/16, sigma = 1/4, SE = 1/16 exactly; the cue window (the
# last four tokens, no terminator) has mean 5/8 = mu + SE exactly.
_TIE = [1/8, 3/8, 3/4, 3/4, 5/8, 1/4, 7/8, 5/8, 1/2, 1/2, 1/2, 5/8, 1, 1/2, 1/8, 7/8]


def test_selection_tie_is_selected():
    """S:674 / P:249 'at least one standard error': mean == mu + SE -> selected."""
    _, summ = _one_traj_stats(_TIE, [12])
    g, c = summ[-1], summ[0]
    assert (g["mean"], g["std"], g["se"]) == (9 / 16, 1 / 4, 1 / 16)
    assert c["mean"] == 5 / 8 and c["selected"] == 1


def test_selection_just_below_is_rejected():
    """Lowering one window token by 2^-20 lowers the cue mean by 2^-22 but
    mu + SE by only ~9e-8 (hand derivative): rejected."""
    v = list(_TIE)
    v[12] = 1 - 2 ** -20
    _, summ = _one_traj_stats(v, [12])
    assert summ[0]["selected"] == 0


def test_selection_spec_values():
    """S:241-242 with mu = 0.5, SE = 0.02 realised as margins 0.46/0.54 x2 (n=4,
    sigma=0.04): cues in separate far-away trajectories are not possible here,
    so check the rule arithmetic on the summary directly."""
    _, summ = _one_traj_stats([0.46, 0.54, 0.46, 0.54], [])
    g = summ[-1]
    assert abs(g["mean"] - 0.5) < 1e-7 and abs(g["se"] - 0.02) < 1e-7
    thr = g["mean"] + g["se"]
    assert 0.53 >= thr and not (0.51 >= thr)


def test_selection_rules_and_min_count():
    # cue windows: one window of mean 0.9 among low background
    m = [0.1] * 20 + [0.9, 0.9]
    _, s0 = _one_traj_stats(m, [20], rule=0, min_count=1)
    _, s3 = _one_traj_stats(m, [20], rule=0, min_count=3)
    _, s2 = _one_traj_stats(m, [20], rule=2, min_count=1)
    assert s0[0]["selected"] == 1 and s3[0]["selected"] == 0 and s2[0]["selected"] == 1
    # rule 1 uses the cue's own SE (0 for one occurrence) -> mean >= mu
    _, s1 = _one_traj_stats(m, [20], rule=1, min_count=1)
    assert s1[0]["selected"] == 1
    low = [0.9] * 20 + [0.1, 0.1]
    for rule in (0, 1, 2):
        _, s = _one_traj_stats(low, [20], rule=rule)
        assert s[0]["selected"] == 0    # below the global mean: never selected


# ------------------------------------------------- brute force: cue scan etc.
def _brute_scan(tokens, offs, pats, mode, pat_cue):
    """All (s, p) pairs by slicing; keep the longest per start (LONGEST) or per
    (start, cue) (ALL)."""
    hits = {}
    for a, b in zip(offs[:-1], offs[1:]):
        for p, pat in enumerate(pats):
            L = len(pat)
            for s in range(a, b - L + 1):
                if list(tokens[s:s + L]) == list(pat):
                    key = (s,) if mode == 0 else (s, pat_cue[p])
                    if key not in hits or len(pats[hits[key]]) < L:
                        hits[key] = p
    keys = sorted(hits)
    return [k[0] for k in keys], [hits[k] for k in keys]


def test_cue_scan_brute_force():
    rng = np.random.default_rng(8)
    for trial in range(300):
        V = 6
        n = int(rng.integers(0, 60))
        tokens = rng.integers(0, V, n).astype(np.int32)
        cuts = sorted(set(rng.integers(0, n + 1, int(rng.integers(0, 4))).tolist()) | {0, n})
        offs = np.array(cuts, np.int64)
        pats = []
        while len(pats) < int(rng.integers(1, 6)):
            p = tuple(int(x) for x in rng.integers(0, V, int(rng.integers(1, 4))))
            if p not in pats:
                pats.append(p)
        pat_cue = rng.integers(0, 3, len(pats)).astype(np.int32)
        po = np.zeros(len(pats) + 1, np.int32)
        po[1:] = np.cumsum([len(p) for p in pats])
        pt = np.array([t for p in pats for t in p], np.int32)
        term_tab = (rng.random(V) < 0.3).astype(np.uint8)
        for mode in (0, 1):
            r = oracle.cue_scan(tokens, offs, pt, po, pat_cue, 3, term_tab, mode)
            bs, bp = _brute_scan(tokens, offs, pats, mode, pat_cue)
            assert r["occ_pos"].tolist() == bs and r["occ_pat"].tolist() == bp
            assert r["term"].tolist() == [int(term_tab[t]) for t in tokens]


def test_scan_edge_cases():
    """Survey 8(c) cases: pattern truncated at the end, spanning trajectories,
    [a] vs [a,b] at the same start, overlapping [a,b]/[b,c], empty trajectory,
    all-terminator stream; ALL mode on two cues at one start."""
    pats = [(1,), (1, 2), (2, 3)]
    pt = np.array([1, 1, 2, 2, 3], np.int32)
    po = np.array([0, 1, 3, 5], np.int32)
    pc = np.array([0, 1, 2], np.int32)
    term = np.zeros(5, np.uint8)
    term[4] = 1
    r = oracle.cue_scan([1, 2, 3, 1], None, pt, po, pc, 3, term)
    assert r["occ_pos"].tolist() == [0, 1, 3] and r["occ_pat"].tolist() == [1, 2, 0]
    r = oracle.cue_scan([0, 1, 2, 3], [0, 2, 2, 4], pt, po, pc, 3, term)   # empty middle traj
    assert r["occ_pos"].tolist() == [1, 2] and r["occ_pat"].tolist() == [0, 2]
    r = oracle.cue_scan([4, 4, 4], None, pt, po, pc, 3, term)
    assert r["occ_pos"].size == 0 and r["term"].tolist() == [1, 1, 1]
    r = oracle.cue_scan([1, 2], None, pt, po, pc, 3, term, mode=1)
    assert r["occ_pos"].tolist() == [0, 0] and r["occ_pat"].tolist() == [0, 1]
    r = oracle.cue_scan([], None, pt, po, pc, 3, term)
    assert r["occ_pos"].size == 0


def test_windows_and_stats_brute_force():
    """Random streams: windows by Python next()/slices, per-cue means by
    statistics over lists, triggers by set-of-sentences."""
    import statistics
    rng = np.random.default_rng(9)
    for trial in range(200):
        n = int(rng.integers(1, 80))
        m = rng.random(n).astype(np.float32)
        term = (rng.random(n) < 0.2).astype(np.uint8)
        cuts = sorted(set(rng.integers(0, n + 1, int(rng.integers(0, 3))).tolist()) | {0, n})
        offs = np.array(cuts, np.int64)
        occ = np.array(sorted(rng.choice(n, int(rng.integers(0, min(n, 8) + 1)), replace=False)),
                       np.int32)
        occ_pat = rng.integers(0, 2, occ.size).astype(np.int32)
        pat_cue = np.array([0, 1], np.int32)
        w = oracle.windows(m, term, offs, occ, 0.5)
        summ = oracle.cue_stats(m, offs, None, occ, occ_pat, pat_cue, 2, 0.5, w, 1, 0)
        ends = []
        for k, s in enumerate(occ.tolist()):
            b = next(bb for aa, bb in zip(cuts[:-1], cuts[1:]) if aa <= s < bb)
            e = next((t for t in range(s, b) if term[t]), b - 1)
            ends.append(e)
            seg = [float(x) for x in m[s:e + 1]]
            assert w["seg_end"][k] == e
            assert abs(w["seg_mean"][k] - math.fsum(seg) / len(seg)) < 1e-12
            assert w["seg_min"][k] == min(seg)
            assert abs(w["seg_lowfrac"][k] - sum(x < 0.5 for x in seg) / len(seg)) < 1e-12
        for c in (0, 1):
            idx = [k for k in range(occ.size) if occ_pat[k] == c]
            means = [float(w["seg_mean"][k]) for k in idx]
            assert summ[c]["n"] == len(idx)
            if idx:
                assert abs(summ[c]["mean"] - statistics.fmean(means)) < 1e-12
                assert abs(summ[c]["std"] - statistics.pstdev(means)) < 1e-12
            seen, trig = set(), 0
            for k in range(occ.size):      # sentence key = window end (same traj)
                if ends[k] not in seen and occ_pat[k] == c:
                    trig += 1
                seen.add(ends[k])
            assert summ[c]["n_triggers"] == trig
        allm = [float(x) for x in m]
        assert abs(summ[-1]["mean"] - statistics.fmean(allm)) < 1e-12
        if n >= 2:
            assert abs(summ[-1]["std"] - statistics.pstdev(allm)) < 1e-12


def test_think_end_and_nan_exclusion():
    m = np.array([0.9, 0.1, np.nan, 0.5, 0.7, 0.2], np.float32)
    term = np.array([0, 1, 0, 1, 0, 0], np.uint8)
    occ = np.array([0, 2, 4], np.int32)
    w = oracle.windows(m, term, None, occ, 0.5)
    assert w["seg_invalid"].tolist() == [0, 1, 0] and math.isnan(w["seg_mean"][1])
    s = oracle.cue_stats(m, None, np.array([4]), occ, np.zeros(3, np.int32),
                         np.array([0], np.int32), 1, 0.5, w, 1, 0)
    # occurrence at 4 >= think_end 4 excluded; NaN window counted invalid
    assert s[0]["n"] == 1 and s[0]["n_invalid"] == 1
    # global: positions 0..3 minus the NaN -> 0.9, 0.1, 0.5
    assert s[-1]["n"] == 3 and s[-1]["n_invalid"] == 1
    assert abs(s[-1]["mean"] - 0.5) < 1e-7


# --------------------------------------------------------- H8 state machine
# Hand-written truth table.  Patterns:
# [20] -> cue 0, [21, 22] -> cue 1, [31] -> cue 2.  Terminators {30, 31}.
# </think> = 40.  Other = 50.  max_small_segment = 3.
_PT = np.array([20, 21, 22, 31], np.int32)
_PO = np.array([0, 1, 3, 4], np.int32)
_PC = np.array([0, 1, 2], np.int32)
_TERM = np.zeros(64, np.uint8)
_TERM[[30, 31]] = 1
H0 = [-1] * 6 + [21]          # a large turn that just emitted 21
CLR = [-1] * 7
# (state, small_run, tok, hist) -> (flag, cue, state', hist', small_run')
TABLE = [
    # Reasoning, Large (state 0)
    ((0, 0, 40, H0), (3, -1, 3, CLR, 0)),                       # K -> TO_ANSWER
    ((0, 0, 22, H0), (1, 1, 1, CLR, 0)),                        # C -> L2S(cue 1)
    ((0, 0, 20, H0), (1, 0, 1, CLR, 0)),                        # C -> L2S(cue 0)
    ((0, 0, 31, H0), (1, 2, 1, CLR, 0)),                        # C&T -> L2S(cue 2)
    ((0, 0, 30, H0), (0, -1, 0, [-1] * 5 + [21, 30], 0)),       # T -> NONE, hist += tok
    ((0, 0, 50, H0), (0, -1, 0, [-1] * 5 + [21, 50], 0)),       # O -> NONE
    ((0, 0, 22, CLR), (0, -1, 0, [-1] * 6 + [22], 0)),          # 22 alone completes nothing
    # Reasoning, Small (state 1), no budget hit (small_run 0)
    ((1, 0, 40, CLR), (3, -1, 3, CLR, 0)),
    ((1, 0, 20, CLR), (0, -1, 1, CLR, 1)),                      # cue on small: ignored
    ((1, 0, 31, CLR), (2, -1, 0, CLR, 0)),                      # C&T -> S2L
    ((1, 0, 30, CLR), (2, -1, 0, CLR, 0)),                      # T -> S2L
    ((1, 0, 50, CLR), (0, -1, 1, CLR, 1)),                      # O -> NONE
    # Reasoning, Small with budget hit (small_run 2, max 3)
    ((1, 2, 40, CLR), (3, -1, 3, CLR, 0)),
    ((1, 2, 20, CLR), (4, -1, 0, CLR, 0)),                      # budget
    ((1, 2, 31, CLR), (2, -1, 0, CLR, 0)),                      # terminator beats budget
    ((1, 2, 30, CLR), (2, -1, 0, CLR, 0)),
    ((1, 2, 50, CLR), (4, -1, 0, CLR, 0)),
    # Answer, Small (state 3): nothing fires, nothing changes
    ((3, 5, 40, CLR), (0, -1, 3, CLR, 5)),
    ((3, 5, 20, CLR), (0, -1, 3, CLR, 5)),
    ((3, 5, 31, CLR), (0, -1, 3, CLR, 5)),
    ((3, 5, 30, CLR), (0, -1, 3, CLR, 5)),
    ((3, 5, 50, CLR), (0, -1, 3, CLR, 5)),
    # invalid token id: nothing
    ((0, 0, -1, H0), (0, -1, 0, H0, 0)),
]


@pytest.mark.parametrize("inp,exp", TABLE)
def test_switch_truth_table(inp, exp):
    state, sr, tok, hist = inp
    flag, cue, st, h, sr2 = oracle.step_one(tok, 0.9, state, hist, sr, _PT, _PO, _PC, _TERM,
                                            40, -1.0, 3)
    assert (flag, cue, st, h.tolist(), sr2) == (exp[0], exp[1], exp[2], exp[3], exp[4])


def test_switch_margin_gate():
    """Optional gate (off in the paper): below the gate the cue does not fire."""
    f, c, st, h, _ = oracle.step_one(22, 0.3, 0, H0, 0, _PT, _PO, _PC, _TERM, 40, 0.5, 0)
    assert (f, st) == (0, 0) and h.tolist()[-1] == 22
    f, c, st, h, _ = oracle.step_one(22, 0.3, 0, H0, 0, _PT, _PO, _PC, _TERM, 40, 0.2, 0)
    assert (f, c, st) == (1, 1, 1)


def test_offline_online_trigger_agreement():
    """Replaying a stream through the step machine (large keeps control at every
    sentence start) fires L2S exactly at the per-sentence first occurrences of
    a substring-free pattern set without terminators (R13)."""
    rng = np.random.default_rng(10)
    pats = [(20,), (21, 22), (23, 24, 25)]
    pt = np.array([t for p in pats for t in p], np.int32)
    po = np.array([0, 1, 3, 6], np.int32)
    pc = np.array([0, 1, 2], np.int32)
    for trial in range(100):
        toks = []
        while len(toks) < 120:
            if rng.random() < 0.4:
                toks.extend(pats[int(rng.integers(0, 3))])
            toks.extend(rng.integers(20, 27, int(rng.integers(0, 4))).tolist())
            toks.append(int(rng.choice([30, 50, 50])))
        toks = np.array(toks, np.int32)
        scan = oracle.cue_scan(toks, None, pt, po, pc, 3, _TERM)
        w = oracle.windows(np.ones(len(toks), np.float32), scan["term"], None, scan["occ_pos"], 0.5)
        expected, seen = [], set()
        for k, s in enumerate(scan["occ_pos"].tolist()):
            if w["seg_end"][k] not in seen:
                expected.append(s + len(pats[scan["occ_pat"][k]]) - 1)   # completion index
            seen.add(w["seg_end"][k])
        # online: large model active at each sentence start; small takes over after a cue
        # and returns on the terminator (the offline stream stands in for both models)
        state, hist, sr, fired = 0, [-1] * 7, 0, []
        for t, tok in enumerate(toks.tolist()):
            f, c, state, hist, sr = oracle.step_one(tok, 1.0, state, hist, sr, pt, po, pc, _TERM,
                                                    40, -1.0, 0)
            hist = hist.tolist()
            if f == 1:
                fired.append(t)
        assert fired == expected


# ------------------------------------------------------- N3 offload estimate
def test_offload_golden(golden_dir):
    """Hand-traced on tests/golden/trace_fixture.json (R17): cases A-C."""
    g = json.load(open(os.path.join(golden_dir, "trace_fixture.json")))
    pt, po, pc, term = _cs_from_fixture(g)
    m = np.array(g["margins"], np.float32)
    scan, win, _ = oracle.analyze(m, g["tokens"], g["traj_offsets"], pt, po, pc, g["n_cues"], term,
                                  tau=g["tau"], min_count=1)
    args = (13, g["traj_offsets"])
    occ = (scan["occ_pos"], scan["occ_pat"], win["seg_end"], po, pc)
    # A: cue 0 selected, no answer stage.  traj0: sentence [0,4] first selected
    # occurrence s=1 ([5,6] completes at 2) -> small 3,4; sentence [5,9]: s=5
    # completes at 6 -> small 7,8,9.  traj1: cue 1 only -> none.
    a = oracle.offload(*args, None, *occ, np.array([1, 0], np.uint8))
    assert a.tolist() == [[5, 5, 0], [3, 0, 0]]
    # B: cue 1 selected.  traj0: s=0 completes at 0 -> small 1..4; traj1: s=11 -> small 12.
    b = oracle.offload(*args, None, *occ, np.array([0, 1], np.uint8))
    assert b.tolist() == [[6, 4, 0], [2, 1, 0]]
    # C: both selected, think_end = [7, 12].  traj0: s=0 -> small 1..4; s=5
    # completes at 6, clamp to te-1=6 -> none; s=8,9 after te.  answer 7..9.
    # traj1: s=11 completes at 11 = te-1 -> none; answer 12.
    c = oracle.offload(*args, np.array([7, 12]), *occ, np.array([1, 1], np.uint8))
    assert c.tolist() == [[3, 4, 3], [2, 0, 1]]
    # nothing selected: all reasoning on the large model
    d = oracle.offload(*args, np.array([7, 12]), *occ, np.array([0, 0], np.uint8))
    assert d.tolist() == [[7, 0, 3], [2, 0, 1]]


def test_offload_matches_step_replay():
    """The estimate equals replaying the trace through the runtime state machine
    (step_one) with the selected patterns, for substring-free pattern sets
    without terminators (R13/R17): small-model tokens are those generated
    while the state is 'small' during reasoning."""
    rng = np.random.default_rng(12)
    pats = [(20,), (21, 22), (23, 24, 25)]
    pt = np.array([t for p in pats for t in p], np.int32)
    po = np.array([0, 1, 3, 6], np.int32)
    pc = np.array([0, 1, 2], np.int32)
    for trial in range(100):
        toks = []
        while len(toks) < 150:
            if rng.random() < 0.4:
                toks.extend(pats[int(rng.integers(0, 3))])
            toks.extend(rng.integers(20, 27, int(rng.integers(0, 4))).tolist())
            toks.append(int(rng.choice([30, 50, 50])))
        toks = np.array(toks[:150], np.int32)
        te = int(rng.integers(100, 150))
        sel = (rng.random(3) < 0.6).astype(np.uint8)
        scan = oracle.cue_scan(toks, None, pt, po, pc, 3, _TERM)
        w = oracle.windows(np.ones(150, np.float32), scan["term"], None, scan["occ_pos"], 0.5)
        est = oracle.offload(150, None, np.array([te]), scan["occ_pos"], scan["occ_pat"], w["seg_end"],
                             po, pc, sel)
        keep = [p for p in range(3) if sel[pc[p]]]
        spt = np.array([t for p in keep for t in pats[p]] or [99], np.int32)
        spo = np.zeros(len(keep) + 1, np.int32)
        spo[1:] = np.cumsum([len(pats[p]) for p in keep]) if keep else [1]
        spc = np.array([pc[p] for p in keep] or [0], np.int32)
        state, hist, sr, small = 0, [-1] * 7, 0, 0
        for t in range(te):
            if state & 1:
                small += 1
            f, c, state, hist, sr = oracle.step_one(int(toks[t]), 1.0, state, hist, sr, spt, spo, spc,
                                                    _TERM, 40, -1.0, 0)
            hist = hist.tolist()
        assert est[0].tolist() == [te - small, small, 150 - te], (trial, est, small)


def test_selection_rule_all_candidates():
    m = [0.9] * 20 + [0.1, 0.1]
    _, s = _one_traj_stats(m, [20], rule=3, min_count=1)
    assert s[0]["selected"] == 1          # below the mean, still a candidate
    _, s = _one_traj_stats(m, [20], rule=3, min_count=2)
    assert s[0]["selected"] == 0          # min_count still applies
