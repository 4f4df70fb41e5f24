"""N4 (text-faithful cue semantics) without a GPU: the host cue-set builder
(paper_2602_06454_b200.cues) against SPEC's worked examples, and the oracle's
token-class matching and decimal-number sentence rule pinned to things other
than itself (SPEC S:168-172's trace, reduction to the class-free oracle,
brute force, both pattern orders)."""
import numpy as np
import pytest

import oracle
import synth


@pytest.fixture(scope="module")
def cues():
    import __graft_entry__
    __graft_entry__._build_lib()
    from paper_2602_06454_b200 import cues as c
    return c


# ------------------------------------------------------------ host builder
def test_expand_variants_spec_examples(cues):
    # S:153-156 (Table 6 surfaces): "thus" -> Thus, Thus,, thus; "so" -> "So ", "So,"; "ah" -> "Ah,"
    assert {"Thus", "Thus,", "thus"} <= cues.expand_variants("thus")
    assert {"So ", "So,"} <= cues.expand_variants("so")
    assert "Ah," in cues.expand_variants("ah")
    assert len(cues.expand_variants("now")) == 6
    with pytest.raises(ValueError):
        cues.expand_variants("")


def test_pool_has_24_canonicals(cues):
    # the Table 5 pool has 24 unique canonicals ("therefore" twice)
    assert len(cues.pool_canonicals()) == 24
    assert cues.pool_canonicals().count("therefore") == 1


def test_switch_cue_sets_are_pool_variants(cues):
    # tab:switch_cue_sets draws from the pool's variants; the one
    # exception is Qwen3's "Also", absent from Table 5 (noted in DESIGN.md)
    variants = set().union(*(cues.expand_variants(c) for c in cues.pool_canonicals()))
    outside = {s for cs in cues.SWITCH_CUES.values() for s in cs if s not in variants}
    assert outside == {"Also"}
    assert len(cues.SWITCH_CUES["Qwen3-32B/Qwen3-1.7B"]) == 28
    assert len(cues.SWITCH_CUES["R1-Distill-Qwen-32B/R1-Distill-Qwen-1.5B"]) == 25


def _toy_vocab():
    words = ["<pad>", "So", ",", " the", " answer", "Thus", ".", " 3", "5", " holds", "value",
             "Wait", " x", "!", "\n", "Now", "12", "7."]
    ids = {w: i for i, w in enumerate(words)}

    def encode(text):               # greedy longest-match word tokenizer
        out, i = [], 0
        while i < len(text):
            for w in sorted(words, key=len, reverse=True):
                if w and text.startswith(w, i):
                    out.append(ids[w])
                    i += len(w)
                    break
            else:
                raise ValueError(text)
        return out
    return words, ids, encode


def test_token_classes_and_terminators(cues):
    words, ids, _ = _toy_vocab()
    cl = cues.token_classes(words)
    assert cl[cues.SPACE_INITIAL, ids[" the"]] and not cl[cues.SPACE_INITIAL, ids["So"]]
    assert cl[cues.PERIOD, ids["."]] and not cl[cues.PERIOD, ids["7."]]
    assert cl[cues.DIGIT_END, ids[" 3"]] and cl[cues.DIGIT_START, ids["5"]]
    assert cl[cues.DIGIT_END, ids["12"]] and not cl[cues.DIGIT_END, ids["7."]]
    term = cues.terminator_table(words)
    assert [words[i] for i in np.flatnonzero(term)] == [".", "!", "\n", "7."]


def test_build_patterns_space_surface(cues):
    words, ids, encode = _toy_vocab()
    pt, po, pc, names = cues.build_patterns(["So ", "So,", "Thus", "So "], encode)
    pats = [pt[po[i]:po[i + 1]].tolist() for i in range(len(po) - 1)]
    assert pats == [[ids["So"], -1 - cues.SPACE_INITIAL], [ids["So"], ids[","]], [ids["Thus"]]]
    assert names == ["so", "thus"] and pc.tolist() == [0, 0, 1]


# ------------------------------------------------------- oracle: classes
def _scan(tokens, offs, cs, classes=None, decimal_rule=None, mode=0):
    return oracle.cue_scan(tokens, offs, cs.pat_tokens, cs.pat_offsets, cs.pat_cue, cs.n_cues,
                           cs.terminator, mode, classes, decimal_rule)


def test_singleton_classes_reduce_to_tokens():
    """A class holding exactly one token t matches exactly like t: replacing
    token elements by singleton classes leaves the scan unchanged."""
    cs = synth.make_cueset(4096, 5, 10, max_len=3, seed=81)
    ts = synth.make_tokens(4, 1500, cs, seed=82, cue_rate=0.4)
    base = _scan(ts.tokens, ts.traj_offsets, cs)
    distinct = sorted(set(cs.pat_tokens.tolist()))[:8]
    classes = np.zeros((len(distinct), 4096), np.uint8)
    for c, t in enumerate(distinct):
        classes[c, t] = 1
    pt = np.array([-1 - distinct.index(t) if t in distinct else t for t in cs.pat_tokens], np.int32)
    cs2 = synth.CueSet(pt, cs.pat_offsets, cs.pat_cue, cs.n_cues, cs.vocab, cs.terminator)
    for mode in (0, 1):
        a = _scan(ts.tokens, ts.traj_offsets, cs, mode=mode)
        b = _scan(ts.tokens, ts.traj_offsets, cs2, classes, mode=mode)
        np.testing.assert_array_equal(a["occ_pos"], b["occ_pos"])
        np.testing.assert_array_equal(a["occ_pat"], b["occ_pat"])
    np.testing.assert_array_equal(base["term"], b["term"])


def test_wildcard_class_brute_force():
    """[a, ANY] with ANY = the whole vocabulary occurs exactly at the starts s
    with tokens[s] == a and s + 1 inside s's trajectory."""
    rng = np.random.default_rng(83)
    V = 64
    tokens = rng.integers(0, V, 3000).astype(np.int32)
    offs = np.array([0, 700, 701, 1900, 3000], np.int64)
    a = 7
    cs = synth.CueSet(np.array([a, -1], np.int32), np.array([0, 2], np.int32),
                      np.array([0], np.int32), 1, V, np.zeros(V, np.uint8))
    got = _scan(tokens, offs, cs, np.ones((1, V), np.uint8))["occ_pos"]
    ends = offs[1:]
    want = [s for s in range(3000) if tokens[s] == a and s + 1 < ends[np.searchsorted(ends, s, "right")]]
    assert got.tolist() == want


def test_equal_length_matches_take_the_lower_index():
    """R18: two same-length patterns matching at one start -> the lower index."""
    V = 16
    so, the = 3, 9
    space = np.zeros((1, V), np.uint8)
    space[0, the] = 1
    tokens = np.array([1, so, the, 2, so, 5], np.int32)
    for first, second, want in (([so, -1], [so, the], 0), ([so, the], [so, -1], 0)):
        cs = synth.CueSet(np.array(first + second, np.int32), np.array([0, 2, 4], np.int32),
                          np.array([0, 1], np.int32), 2, V, np.zeros(V, np.uint8))
        r = _scan(tokens, None, cs, space)
        assert r["occ_pos"].tolist() == [1] and r["occ_pat"].tolist() == [want]


def test_decimal_rule_spec_example():
    """["value", " 3", ".", "5", " holds", "."] from 0 -> 5 (the decimal
    point at 2 is skipped); without the rule the window ends at 2."""
    words, ids, encode = _toy_vocab()
    from paper_2602_06454_b200 import cues
    V = len(words)
    toks = np.array([ids[w] for w in ["value", " 3", ".", "5", " holds", "."]], np.int32)
    cl = cues.token_classes(words)
    term_tab = cues.terminator_table(words)
    cs = synth.CueSet(np.array([ids["value"]], np.int32), np.array([0, 1], np.int32),
                      np.array([0], np.int32), 1, V, term_tab)
    m = np.linspace(0.1, 0.6, 6).astype(np.float32)
    on = _scan(toks, None, cs, cl, cues.DECIMAL_RULE)
    off = _scan(toks, None, cs, cl)
    assert on["term"].tolist() == [0, 0, 0, 0, 0, 1] and off["term"].tolist() == [0, 0, 1, 0, 0, 1]
    assert oracle.windows(m, on["term"], None, on["occ_pos"], 0.5)["seg_end"].tolist() == [5]
    assert oracle.windows(m, off["term"], None, off["occ_pos"], 0.5)["seg_end"].tolist() == [2]
    # the neighbours must lie in the period's trajectory
    offs = np.array([0, 3, 6], np.int64)
    assert _scan(toks, offs, cs, cl, cues.DECIMAL_RULE)["term"].tolist() == [0, 0, 1, 0, 0, 1]


def test_step_one_class_suffix():
    """The decode-step switch completes "So " when the sampled token is any
    space-initial token (and not on "So,")."""
    V = 16
    so, comma = 3, 4
    space = np.zeros((1, V), np.uint8)
    space[0, [9, 10]] = 1
    pt, po, pc = np.array([so, -1], np.int32), np.array([0, 2], np.int32), np.array([2], np.int32)
    term = np.zeros(V, np.uint8)
    hist = np.full(7, -1, np.int32)
    hist[-1] = so
    for tok, flag, cue in ((9, 1, 2), (10, 1, 2), (comma, 0, -1)):
        f, c, st, h, sr = oracle.step_one(tok, 0.5, 0, hist, 0, pt, po, pc, term, 15, classes=space)
        assert (f, c) == (flag, cue)
