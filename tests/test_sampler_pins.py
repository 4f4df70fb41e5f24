"""N2 oracle pins (no GPU): the sampler reading R20 (temperature, top-k, top-p,
inverse CDF with a given uniform) fixed by a hand-computed example, its
reductions to argmax and to plain softmax inverse-CDF sampling, invariances,
and the status rows."""
import numpy as np

import oracle


def test_hand_example():
    # z = ln(1, 2, 3, 4), T = 1: ranked tokens 3, 2, 1, 0 with p = .4 .3 .2 .1.
    # top_p = 1: u .35 -> 3 (cum .4), .45 -> 2 (cum .7), .95 -> 0 (cum 1.0).
    # top_p = .6: higher-ranked mass 0, .4, .7, .9 -> keep tokens 3, 2 (mass .7);
    # u .5 -> target .35 -> 3; u .6 -> target .42 -> 2.
    z = np.log(np.array([[1, 2, 3, 4]], np.float32))
    for u, p, want in ((0.35, 1.0, 3), (0.45, 1.0, 2), (0.95, 1.0, 0), (0.5, 0.6, 3), (0.6, 0.6, 2)):
        assert oracle.sample_rows(z, [u], temperature=1.0, top_k=4, top_p=p)[0] == want
    # top_k = 2 keeps tokens 3, 2 (p .4, .3): u .6 -> target .42 -> 2
    assert oracle.sample_rows(z, [0.6], temperature=1.0, top_k=2, top_p=1.0)[0] == 2


def test_top1_and_tiny_top_p_are_argmax():
    rng = np.random.default_rng(1)
    rows = rng.normal(0, 2, (20, 300)).astype(np.float32)
    rows[3, [5, 9]] = rows[3].max() + 1      # tie: the lower index is the argmax
    ref = oracle.margin_rows(rows)["top1"]
    u = rng.random(20)
    assert (oracle.sample_rows(rows, u, top_k=1, top_p=1.0) == ref).all()
    assert (oracle.sample_rows(rows, u, top_k=50, top_p=1e-9) == ref).all()
    assert ref[3] == 5


def test_full_softmax_inverse_cdf():
    """K = V and top_p = 1 is plain inverse-CDF sampling from softmax(z / T)
    with the entries ordered by (value desc, index asc)."""
    rng = np.random.default_rng(2)
    V, T = 40, 0.6
    z = rng.normal(0, 1.5, V).astype(np.float32)
    order = np.lexsort((np.arange(V), -z.astype(np.float64)))
    w = np.exp((z[order].astype(np.float64) - z.max()) / T)
    cdf = np.cumsum(w) / w.sum()
    us = (np.arange(997) + 0.5) / 997
    got = oracle.sample_rows(np.tile(z, (len(us), 1)), us, temperature=T, top_k=V, top_p=1.0)
    want = order[np.searchsorted(cdf, us, side="right")]
    assert (got == want).all()


def test_shift_invariance_and_status_rows():
    rng = np.random.default_rng(3)
    rows = rng.normal(0, 2, (8, 500)).astype(np.float32)
    u = rng.random(8)
    a = oracle.sample_rows(rows, u, top_k=20, top_p=0.95)
    b = oracle.sample_rows(rows + np.float32(8.0), u, top_k=20, top_p=0.95)
    assert (a == b).all()
    bad = rows.copy()
    bad[0, 7] = np.nan
    bad[1, 3] = np.inf
    bad[2, :] = -np.inf
    got = oracle.sample_rows(bad, u, top_k=20, top_p=0.95)
    assert got[:3].tolist() == [-1, -1, -1] and (got[3:] == a[3:]).all()


def test_minus_inf_entries_are_never_drawn():
    z = np.full((1, 30), -np.inf, np.float32)
    z[0, [4, 17]] = [1.0, 0.5]
    for u in np.linspace(0, 0.999, 11):
        assert oracle.sample_rows(z, [u], temperature=0.6, top_k=20, top_p=1.0)[0] in (4, 17)


def test_no_top_k_is_the_whole_vocabulary():
    """top_k = 0 (the R1-Distill setting: top-p only) keeps every entry:
    the same draws as top_k = vocab, and with top_p = 1 plain inverse-CDF
    sampling over softmax(z / T)."""
    rng = np.random.default_rng(4)
    rows = rng.normal(0, 2, (16, 300)).astype(np.float32)
    u = rng.random(16)
    a = oracle.sample_rows(rows, u, top_k=0, top_p=0.95)
    b = oracle.sample_rows(rows, u, top_k=300, top_p=0.95)
    assert (a == b).all()
    z = rows[0].astype(np.float64)
    order = np.lexsort((np.arange(300), -z))
    w = np.exp((z[order] - z.max()) / 0.6)
    cdf = np.cumsum(w) / w.sum()
    us = (np.arange(101) + 0.5) / 101
    got = oracle.sample_rows(np.tile(rows[0], (101, 1)), us, top_k=0, top_p=1.0)
    assert (got == order[np.searchsorted(cdf, us, side="right")]).all()
