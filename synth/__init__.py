"""Seeded synthetic inputs shaped like RelayGen's workloads (shared by tests/bench).

This module holds NONE of the method's arithmetic (no softmax, margin, matching,
windowing or statistics).  It only draws inputs: token streams with sentences,
switch cues and a ``</think>`` boundary, logit rows with a planted top-1/top-2
structure, and margin series.  Both the CUDA path and the oracle consume the
exact same arrays it returns; nothing here is computed by either side.

The recipe follows the paper's workload shapes:
  * trajectories of up to 32,768 tokens (generation cap), `<think>` ...
    `</think>` then an answer;
  * vocabularies 151,936 (Qwen3) / 152,064 (R1-Distill-Qwen) / 32,000;
  * switch-cue sets of 1-32 surfaces (tab:switch_cue_sets has 28 and 25,
    P:689-701), each surface a token pattern of 1-6 tokens;
  * margins that fluctuate between confident (~1) and uncertain (~0) regions
    (fig:margin_trajectory).
Every density below (sentence length, cue rate, stage lengths) is a synthetic
choice: the paper states none of them.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

BASE_SEED = 0x260206454          # from the arXiv id

THINK_START = 1000
THINK_END = 1001
TERMINATOR_IDS = np.arange(100, 140, dtype=np.int32)   # 40 sentence-ending ids
CUE_TOKEN_BASE = 2000                                  # cue-pattern token ids
OTHER_BASE = 3000                                      # everything else


@dataclass
class CueSet:
    """Switch-cue patterns in CSR form plus the terminator table."""
    pat_tokens: np.ndarray            # int32 [sum len]
    pat_offsets: np.ndarray           # int32 [n_pat + 1]
    pat_cue: np.ndarray               # int32 [n_pat] -> cue id
    n_cues: int
    vocab: int
    terminator: np.ndarray            # uint8 [vocab]
    think_end: int = THINK_END
    patterns: list = field(default_factory=list)

    @property
    def n_pat(self) -> int:
        return int(self.pat_offsets.shape[0] - 1)


def make_cueset(vocab: int, n_cues: int, n_patterns: int, min_len: int = 1, max_len: int = 3,
                seed: int = BASE_SEED, prefix_pair: bool = True,
                substring_free: bool = False) -> CueSet:
    """Random distinct token patterns, 1+ per cue (variant clusters as in
    tab:switch_cue_sets: "Thus", "Thus," ...).  With ``prefix_pair`` one pattern
    is a proper prefix of another (like "Thus" / "Thus,")."""
    rng = np.random.default_rng(seed)
    assert n_patterns >= n_cues
    pats: list[tuple[int, ...]] = []
    cues: list[int] = []
    pool = np.arange(CUE_TOKEN_BASE, CUE_TOKEN_BASE + 64, dtype=np.int64)
    tries = 0
    while len(pats) < n_patterns:
        tries += 1
        assert tries < 100000, "cannot draw distinct patterns"
        cue = len(pats) if len(pats) < n_cues else int(rng.integers(0, n_cues))
        if prefix_pair and len(pats) == 1 and max_len > 1 and len(pats[0]) < max_len:
            p = pats[0] + (int(rng.choice(pool)),)       # extends pattern 0
        else:
            ln = int(rng.integers(min_len, max_len + 1))
            p = tuple(int(x) for x in rng.choice(pool, size=ln))
        if p in pats:
            continue
        if substring_free and any(_contains(q, p) or _contains(p, q) for q in pats):
            continue
        pats.append(p)
        cues.append(cue)
    offs = np.zeros(len(pats) + 1, np.int32)
    offs[1:] = np.cumsum([len(p) for p in pats])
    term = np.zeros(vocab, np.uint8)
    term[TERMINATOR_IDS[TERMINATOR_IDS < vocab]] = 1
    return CueSet(np.array([t for p in pats for t in p], np.int32), offs,
                  np.array(cues, np.int32), n_cues, vocab, term, THINK_END, pats)


def _contains(big, small) -> bool:
    n, m = len(big), len(small)
    return any(tuple(big[i:i + m]) == tuple(small) for i in range(n - m + 1))


@dataclass
class TokenStream:
    tokens: np.ndarray          # int32 [n_tok]
    traj_offsets: np.ndarray    # int64 [n_traj + 1]
    think_end_pos: np.ndarray   # int64 [n_traj]: position of </think> (answer follows)


def make_tokens(n_traj: int, traj_len: int, cs: CueSet, seed: int = BASE_SEED,
                cue_rate: float = 0.2, mean_sentence: float = 22.0,
                long_run_rate: float = 0.01, think_frac: float = 0.85) -> TokenStream:
    """Sentences of geometric length (mean 22) ended by one of 40 terminator ids,
    1% long unterminated runs of 200-2,000 tokens (math blocks), a switch-cue
    pattern at a sentence start with probability 0.2, Zipf-distributed other
    tokens, `<think>` first and `</think>` at ~85% of the trajectory."""
    rng = np.random.default_rng(seed)
    vocab = cs.vocab
    n_other = max(16, vocab - OTHER_BASE)
    toks = np.empty(n_traj * traj_len, np.int32)
    think = np.empty(n_traj, np.int64)
    pats = cs.patterns
    for k in range(n_traj):
        out = [THINK_START]
        think_at = int(traj_len * think_frac)
        placed = False
        while len(out) < traj_len:
            if not placed and len(out) >= think_at:
                think[k] = k * traj_len + len(out)
                out.append(THINK_END)
                placed = True
                continue
            if pats and rng.random() < cue_rate:
                out.extend(pats[int(rng.integers(0, len(pats)))])
            if rng.random() < long_run_rate:
                body = int(rng.integers(200, 2001))
                terminated = False
            else:
                body = int(rng.geometric(1.0 / mean_sentence))
                terminated = True
            z = rng.zipf(1.3, size=body) % n_other
            out.extend((OTHER_BASE + z).astype(np.int64).tolist())
            if terminated:
                out.append(int(rng.choice(TERMINATOR_IDS)))
        if not placed:
            think[k] = k * traj_len + traj_len - 1
            out[traj_len - 1] = THINK_END
        toks[k * traj_len:(k + 1) * traj_len] = np.array(out[:traj_len], np.int32) % vocab
    offs = np.arange(n_traj + 1, dtype=np.int64) * traj_len
    return TokenStream(toks, offs, think)


def make_margins(n_tok: int, seed: int = BASE_SEED, nan_rate: float = 0.0,
                 tau: float | None = 0.5) -> np.ndarray:
    """A margin series in [0, 1] (fp32) alternating confident / uncertain
    stretches; some values sit exactly at tau and at 0 / 1; optional NaNs."""
    rng = np.random.default_rng(seed)
    conf = rng.random(n_tok) < 0.7
    m = np.where(conf, 1.0 - rng.random(n_tok) * 0.05, rng.random(n_tok)).astype(np.float32)
    pick = rng.random(n_tok)
    if tau is not None:
        m[pick < 0.01] = np.float32(tau)
    m[(pick >= 0.01) & (pick < 0.015)] = 0.0
    m[(pick >= 0.015) & (pick < 0.02)] = 1.0
    if nan_rate > 0:
        m[rng.random(n_tok) < nan_rate] = np.nan
    return m


def make_logits(n_rows: int, vocab: int, dtype: str = "bf16", row_stride: int | None = None,
                tokens: np.ndarray | None = None, seed: int = BASE_SEED, device="cpu",
                chunk_rows: int = 1024, edge_rows: bool = True, pad_value: float = float("nan")):
    """Logit rows [n_rows, row_stride] (torch tensor on ``device``).

    Background ~ N(0, 2.5^2) (unclipped).  Per row t the runner-up sits 3 above
    the row's background maximum and the top at runner-up + gap; with
    probability 0.9 the top-1 id is
    ``tokens[t]`` (else the runner-up is), mimicking T = 0.6 sampling.
    Gap: 70% "confident" U[3, 12], 30% "uncertain" U[0, 2] with a third
    candidate at runner-up - U[0, 0.5].  Edge rows: 1% exact top-1 ties, 1% exact
    top-2 ties, 0.1% rows with only 20 finite entries (rest -inf), 0.1%
    uniform rows.  Columns [vocab, row_stride) hold ``pad_value`` (NaN by
    default: any kernel that reads the padding fails the tests).  Values are
    rounded to ``dtype`` (round-to-nearest-even).
    """
    import torch
    stride = vocab if row_stride is None else row_stride
    tdt = {"bf16": torch.bfloat16, "f16": torch.float16, "f32": torch.float32}[dtype]
    out = torch.empty((n_rows, stride), dtype=tdt, device=device)
    if stride > vocab:
        out[:, vocab:] = pad_value
    rng = np.random.default_rng(seed ^ 0x5EED)
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) & 0x7FFFFFFFFFFFFFFF)
    # per-row planted structure drawn on the host (tiny)
    if tokens is None:
        tokens = rng.integers(0, vocab, size=n_rows)
    tokens = np.asarray(tokens[:n_rows], np.int64) % vocab
    other = (tokens + rng.integers(1, vocab, size=n_rows)) % vocab
    third = (tokens + rng.integers(1, vocab, size=n_rows)) % vocab
    third = np.where(third == other, (third + 1) % vocab, third)
    third = np.where(third == tokens, (third + 1) % vocab, third)
    third = np.where(third == other, (third + 1) % vocab, third)
    top_is_tok = rng.random(n_rows) < 0.9
    top = np.where(top_is_tok, tokens, other)
    run = np.where(top_is_tok, other, tokens)
    confident = rng.random(n_rows) < 0.7
    gap = np.where(confident, rng.uniform(3, 12, n_rows), rng.uniform(0, 2, n_rows))
    third_off = np.where(confident, np.nan, -rng.uniform(0, 0.5, n_rows))
    kind = rng.random(n_rows)
    if edge_rows:
        gap[kind < 0.01] = 0.0                                  # exact top-1 tie
        third_off[(kind >= 0.01) & (kind < 0.02)] = 0.0         # exact top-2 tie
    sparse = edge_rows & (kind >= 0.02) & (kind < 0.021)        # 20 finite entries
    uniform = edge_rows & (kind >= 0.021) & (kind < 0.022)      # all equal
    for r0 in range(0, n_rows, chunk_rows):
        r1 = min(n_rows, r0 + chunk_rows)
        R = r1 - r0
        bg = torch.randn((R, vocab), generator=g, device=device, dtype=torch.float32)
        bg.mul_(2.5)
        run_v = bg.amax(dim=1) + 3.0                            # runner-up value per row
        rows = torch.arange(R, device=device)
        t_top = torch.as_tensor(top[r0:r1], device=device)
        t_run = torch.as_tensor(run[r0:r1], device=device)
        t_3 = torch.as_tensor(third[r0:r1], device=device)
        off3 = torch.as_tensor(third_off[r0:r1], device=device, dtype=torch.float32)
        has3 = ~torch.isnan(off3)
        bg[rows[has3], t_3[has3]] = (run_v + torch.nan_to_num(off3))[has3]
        bg[rows, t_run] = run_v
        bg[rows, t_top] = run_v + torch.as_tensor(gap[r0:r1], device=device, dtype=torch.float32)
        sp = np.nonzero(sparse[r0:r1])[0]
        for i in sp:
            keep = torch.randperm(vocab, generator=g, device=device)[:20]
            vals = bg[int(i), keep].clone()
            bg[int(i)] = float("-inf")
            bg[int(i), keep] = vals
        un = np.nonzero(uniform[r0:r1])[0]
        if un.size:
            bg[torch.as_tensor(un, device=device)] = 0.0
        out[r0:r1, :vocab] = bg.to(tdt)
        del bg
    return out


def bits_u16(t) -> np.ndarray:
    """A 16-bit torch tensor as its raw uint16 bit patterns (host numpy)."""
    import torch
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)


def host_rows(t, dtype: str) -> np.ndarray:
    """Torch logits -> the host array the oracle takes (uint16 bits or fp32)."""
    return bits_u16(t) if dtype in ("bf16", "f16") else t.detach().cpu().contiguous().numpy()


# --------------------------------------------------------------- configs
CONFIGS = {
    # BASELINE.json configs[0..4]
    "c1": dict(n_traj=1, traj_len=2048, vocab=32000, dtype="f32", n_cues=3, n_pat=3,
               max_len=3),
    "c2": dict(n_traj=1, traj_len=32768, vocab=151936, dtype="bf16", n_cues=8, n_pat=12,
               max_len=3),
    "c3": dict(batch=256, vocab=152064, dtype="bf16", n_cues=8, n_pat=12, max_len=3),
    "c4": dict(n_traj=8, traj_len=32768, vocab=151936, dtype="bf16", n_cues=8, n_pat=12,
               max_len=3),
    "c5": dict(n_traj=64, traj_len=16384, vocab=151936, dtype="bf16", n_cues=32, n_pat=32,
               max_len=6),
}


@dataclass
class ClassCase:
    """A cue set with token-class pattern elements (N4) and a token stream
    planted with class instances and decimal-number triples."""
    cs: CueSet                 # pat_tokens may hold class elements (-1 - class)
    classes: np.ndarray        # uint8 [n_classes, vocab]
    decimal_rule: tuple        # (period, digit_end, digit_start) class ids
    ts: TokenStream


def make_class_case(vocab: int, n_traj: int, traj_len: int, n_cues: int = 6, n_patterns: int = 12,
                    seed: int = BASE_SEED, decimal_rate: float = 0.02) -> ClassCase:
    """Classes: 0 'space-initial' (30% of the ordinary tokens), 1 'period'
    (10 of the 40 terminator ids), 2 'digit-end' / 3 'digit-start' (5% each),
    4 and 5 arbitrary 10% subsets.  Patterns of 1-4 elements, each element a
    class (0, 4 or 5) with probability 0.3, else a cue-pool token.  Tokens:
    make_tokens with every pattern planted through random class members, then
    digit-end / digit-start neighbours put around ``decimal_rate`` of the
    period tokens (and around none of the others)."""
    rng = np.random.default_rng(seed)
    n_cls = 6
    classes = np.zeros((n_cls, vocab), np.uint8)
    ordinary = np.arange(OTHER_BASE, vocab)
    classes[0, ordinary[rng.random(ordinary.size) < 0.3]] = 1
    classes[1, TERMINATOR_IDS[:10]] = 1
    for c, rate in ((2, 0.05), (3, 0.05), (4, 0.1), (5, 0.1)):
        classes[c, ordinary[rng.random(ordinary.size) < rate]] = 1
    pool = np.arange(CUE_TOKEN_BASE, CUE_TOKEN_BASE + 64, dtype=np.int64)
    pats: list[tuple[int, ...]] = []
    cues: list[int] = []
    while len(pats) < n_patterns:
        ln = int(rng.integers(1, 5))
        p = tuple(int(-1 - rng.choice([0, 4, 5])) if (k > 0 and rng.random() < 0.3)
                  else int(rng.choice(pool)) for k in range(ln))
        if p in pats:
            continue
        cues.append(len(pats) if len(pats) < n_cues else int(rng.integers(0, n_cues)))
        pats.append(p)
    offs = np.zeros(len(pats) + 1, np.int32)
    offs[1:] = np.cumsum([len(p) for p in pats])
    term = np.zeros(vocab, np.uint8)
    term[TERMINATOR_IDS[TERMINATOR_IDS < vocab]] = 1
    members = [np.flatnonzero(classes[c]) for c in range(n_cls)]
    # several concrete instances of every pattern for planting
    inst = []
    for p in pats:
        for _ in range(4):
            inst.append(tuple(e if e >= 0 else int(rng.choice(members[-1 - e])) for e in p))
    plant = CueSet(offs.copy(), offs, np.array(cues, np.int32), n_cues, vocab, term, THINK_END, inst)
    ts = make_tokens(n_traj, traj_len, plant, seed=seed + 1)
    toks = ts.tokens
    periods = np.flatnonzero(classes[1][toks] == 1)
    for t in periods:
        if rng.random() < decimal_rate * 25 and 0 < t < toks.size - 1:
            if toks[t - 1] in (THINK_START, THINK_END) or toks[t + 1] in (THINK_START, THINK_END):
                continue
            toks[t - 1] = int(rng.choice(members[2]))
            toks[t + 1] = int(rng.choice(members[3]))
    cs = CueSet(np.array([t for p in pats for t in p], np.int32), offs, np.array(cues, np.int32),
                n_cues, vocab, term, THINK_END, pats)
    return ClassCase(cs, classes, (1, 2, 3), TokenStream(toks, ts.traj_offsets, ts.think_end_pos))
