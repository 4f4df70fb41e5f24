"""Host-side construction of a model pair's cue set (N4, text-faithful cues).

The kernels match token-ID patterns whose elements may be token classes
(relay_cueset_create_ex).  This module turns the paper's text-level cue
descriptions into that form for a given tokenizer:

* ``CUE_POOL`` — the canonical discourse-level cue pool (Appendix A,
  tab:discourse_cue_pool).  "therefore" is listed under two
  categories; it is kept once, under Inference (SPEC design decision).
* ``SWITCH_CUES`` — the model-pair switch-cue sets selected offline
  (tab:switch_cue_sets), as surface strings.
* ``expand_variants`` — capitalisation and punctuation variants of a canonical
  cue ("handled separately during tokenization").
* ``token_classes`` — class bitmaps from the decoded vocabulary: tokens that
  start with a space (for surfaces like "So "), sentence terminators (S:168:
  '.', '!', '?', newline), and the three classes of the decimal-number rule.
* ``build_patterns`` — surface strings -> (pat_tokens, pat_offsets, pat_cue)
  with a trailing space encoded as the SPACE_INITIAL class element.

Plain host logic; nothing here touches the GPU.
"""
from __future__ import annotations

from typing import Callable, Iterable, Sequence

import numpy as np

# tab:discourse_cue_pool, canonical forms by category
CUE_POOL: dict[str, tuple[str, ...]] = {
    "Progression": ("now", "then", "next", "again"),
    "Reconsideration": ("wait", "however", "alternatively", "but", "maybe", "hmm", "oh"),
    "Inference": ("thus", "hence", "therefore", "similarly", "specifically"),
    "Consolidation": ("so", "check", "double-check", "verify"),   # "therefore": Inference
    "Reference": ("another", "other", "any"),
    "Acknowledgement": ("ah",),
}

# tab:switch_cue_sets
SWITCH_CUES: dict[str, tuple[str, ...]] = {
    "Qwen3-32B/Qwen3-1.7B": (
        "Oh,", "another,", "Thus", "Now", "Alternatively", "alternatively,", "Thus,", "Therefore",
        "similarly", "similarly,", "now", "Again", "specifically,", "Again,", "Similarly,", "Now,",
        "Specifically,", "Hence", "Similarly", "Other", "now,", "hence", "Specifically", "So ",
        "Therefore,", "Wait,", "Also", "So,"),
    "R1-Distill-Qwen-32B/R1-Distill-Qwen-1.5B": (
        "Wait", "Thus", "thus", "similarly", "Again,", "Now", "Therefore", "hence", "Hence,",
        "Now,", "Thus,", "Oh,", "Similarly,", "Any", "Therefore,", "Alternatively,", "now,", "So,",
        "now", "verify", "Specifically,", "Alternatively", "Ah,", "wait", "So "),
}

# class ids produced by token_classes (rows of the returned array)
SPACE_INITIAL, PERIOD, DIGIT_END, DIGIT_START = 0, 1, 2, 3
CLASS_NAMES = ("space_initial", "period", "digit_end", "digit_start")
DECIMAL_RULE = (PERIOD, DIGIT_END, DIGIT_START)


def pool_canonicals() -> list[str]:
    """The unique canonical cues of the pool, in table order."""
    seen: list[str] = []
    for cues in CUE_POOL.values():
        seen.extend(c for c in cues if c not in seen)
    return seen


def expand_variants(canonical: str) -> set[str]:
    """{c, C, c",", C",", c" ", C" "} for canonical c (C = first
    letter upper-cased)."""
    if not canonical:
        raise ValueError("empty canonical cue")
    cap = canonical[0].upper() + canonical[1:]
    return {canonical, cap, canonical + ",", cap + ",", canonical + " ", cap + " "}


def canonical_of(surface: str) -> str:
    """The canonical form a surface variant belongs to ("So " -> "so")."""
    return surface.strip().rstrip(",").lower()


def terminator_table(vocab_strings: Sequence[str]) -> np.ndarray:
    """uint8[vocab]: tokens whose text holds a sentence terminator (S:168:
    '.', '!', '?' or a newline)."""
    return np.array([any(ch in t for ch in ".!?\n") for t in vocab_strings], np.uint8)


def token_classes(vocab_strings: Sequence[str]) -> np.ndarray:
    """uint8[4, vocab] class bitmaps (rows SPACE_INITIAL, PERIOD, DIGIT_END,
    DIGIT_START) from the decoded text of every token id."""
    v = len(vocab_strings)
    out = np.zeros((4, v), np.uint8)
    for i, t in enumerate(vocab_strings):
        out[SPACE_INITIAL, i] = len(t) > 0 and t[0] == " "
        out[PERIOD, i] = t == "."
        out[DIGIT_END, i] = len(t) > 0 and t[-1].isdigit()
        out[DIGIT_START, i] = len(t) > 0 and t[0].isdigit()
    return out


def build_patterns(surfaces: Iterable[str], encode: Callable[[str], Sequence[int]],
                   cue_ids: dict[str, int] | None = None):
    """Surface strings -> (pat_tokens, pat_offsets, pat_cue, cue_names).

    ``encode`` maps text to token ids (no special tokens).  A surface ending
    in a space ("So ") is the encoding of its text followed by the
    SPACE_INITIAL class element: the space is carried by the next token in
    BPE vocabularies [R18].  Each surface's cue is its canonical form
    (``cue_ids`` fixes the numbering; default: order of first appearance).
    Duplicate patterns (two surfaces encoding identically) are kept once."""
    cue_ids = dict(cue_ids or {})
    toks: list[int] = []
    offs = [0]
    cues: list[int] = []
    seen: set[tuple[int, ...]] = set()
    for s in surfaces:
        body = s[:-1] if s.endswith(" ") else s
        ids = list(encode(body))
        if s.endswith(" "):
            ids.append(-1 - SPACE_INITIAL)
        if not ids:
            raise ValueError(f"surface {s!r} encodes to no tokens")
        key = tuple(ids)
        if key in seen:
            continue
        seen.add(key)
        c = canonical_of(s)
        if c not in cue_ids:
            cue_ids[c] = len(cue_ids)
        toks.extend(ids)
        offs.append(len(toks))
        cues.append(cue_ids[c])
    names = [None] * len(cue_ids)
    for name, i in cue_ids.items():
        names[i] = name
    return (np.array(toks, np.int32), np.array(offs, np.int32), np.array(cues, np.int32), names)
