"""CPU oracle for the RelayGen (arXiv 2602.06454) hot path — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module.  The product package
``paper_2602_06454_b200`` never imports it and shares no code with it.

This module is argument marshalling over ``relay_oracle.c`` (plain C, fp64, the
paper's definitions written out — see the header of that file for citations).
``build()`` compiles it with gcc (``-O2 -ffp-contract=off``, no fast-math).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "relay_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

DT_BF16, DT_F16, DT_F32 = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile the oracle shared library (host C, no CUDA)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off",
               "-fno-fast-math", "-pthread", "-Wall", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class Summary(C.Structure):
    _fields_ = [("n", C.c_int64), ("mean", C.c_double), ("std", C.c_double),
                ("se", C.c_double), ("token_mean", C.c_double), ("min", C.c_double),
                ("low_frac", C.c_double), ("n_triggers", C.c_int64),
                ("n_invalid", C.c_int64), ("selected", C.c_int32)]


def _load():
    global _lib
    if _lib is None:
        lib = C.CDLL(build())
        P = C.c_void_p
        lib.oracle_margin_row.restype = C.c_int
        lib.oracle_margin_row.argtypes = [P, C.c_int, C.c_int64, C.c_double, P, P, P, P]
        lib.oracle_margin_rows.restype = C.c_int
        lib.oracle_margin_rows.argtypes = [P, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                           C.c_double, C.c_int, P, P, P, P, P]
        lib.oracle_cue_scan_ex.restype = C.c_int64
        lib.oracle_cue_scan_ex.argtypes = [P, C.c_int64, P, C.c_int32, P, P, C.c_int32, P,
                                           C.c_int32, P, C.c_uint32, P, C.c_int32, C.c_int64, P,
                                           P, P, P, C.c_int64]
        lib.oracle_windows.restype = None
        lib.oracle_windows.argtypes = [P, P, C.c_int64, P, C.c_int32, P, C.c_int64, C.c_float,
                                       P, P, P, P, P, P, P]
        lib.oracle_cue_stats.restype = None
        lib.oracle_cue_stats.argtypes = [P, C.c_int64, P, C.c_int32, P, P, P, C.c_int64, P,
                                         C.c_int32, C.c_float, P, P, P, P, P, P, C.c_int64,
                                         C.c_int32, P]
        lib.oracle_sample_row.restype = C.c_int32
        lib.oracle_sample_row.argtypes = [P, C.c_int, C.c_int64, C.c_double, C.c_int32, C.c_double,
                                          C.c_double]
        lib.oracle_offload.restype = None
        lib.oracle_offload.argtypes = [C.c_int64, P, C.c_int32, P, P, P, C.c_int64, P, P, P, P, P]
        lib.oracle_step_one_ex.restype = C.c_int
        lib.oracle_step_one_ex.argtypes = [C.c_int32, C.c_float, P, P, P, P, P, C.c_int32, P, P,
                                           C.c_int64, C.c_int32, C.c_float, C.c_int32, P,
                                           C.c_int32, P]
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _dtype_code(a: np.ndarray, dtype: str | None) -> int:
    if dtype is not None:
        return {"bf16": DT_BF16, "f16": DT_F16, "f32": DT_F32}[dtype]
    if a.dtype == np.float32:
        return DT_F32
    raise ValueError("16-bit rows must be passed as uint16 bit patterns with dtype='bf16'|'f16'")


# --------------------------------------------------------------------- H1
def margin_row(row, dtype: str | None = None, inv_temperature: float = 1.0):
    """One row -> (status, i1, i2, margin, lse) in fp64."""
    a = np.ascontiguousarray(row)
    if a.dtype == np.float64:
        a = a.astype(np.float32)
    code = _dtype_code(a, dtype)
    i1, i2 = C.c_int32(), C.c_int32()
    m, l = C.c_double(), C.c_double()
    st = _load().oracle_margin_row(_p(a), code, a.shape[-1], inv_temperature,
                                   C.byref(i1), C.byref(i2), C.byref(m), C.byref(l))
    if st < 0:
        raise ValueError("vocab < 2")
    return st, i1.value, i2.value, m.value, l.value


def margin_rows(logits: np.ndarray, dtype: str | None = None, vocab: int | None = None,
                inv_temperature: float = 1.0, threads: int = 1):
    """Rows [n, stride] (float32, or uint16 bits with dtype) -> dict of arrays."""
    a = np.ascontiguousarray(logits)
    code = _dtype_code(a, dtype)
    n, stride = a.shape
    vocab = stride if vocab is None else vocab
    out = dict(margin=np.empty(n, np.float64), top1=np.empty(n, np.int32),
               top2=np.empty(n, np.int32), lse=np.empty(n, np.float64),
               status=np.empty(n, np.int8))
    rc = _load().oracle_margin_rows(_p(a), code, n, vocab, stride, inv_temperature, threads,
                                    _p(out["margin"]), _p(out["top1"]), _p(out["top2"]),
                                    _p(out["lse"]), _p(out["status"]))
    if rc < 0:
        raise ValueError("invalid margin_rows arguments")
    return out


# --------------------------------------------------------------------- H2
def _classes(classes, vocab):
    """[n_classes, vocab] 0/1 array (or None) -> (uint8 array, n_classes)."""
    if classes is None:
        return None, 0
    c = np.ascontiguousarray(np.asarray(classes).astype(bool).astype(np.uint8))
    if c.ndim != 2 or c.shape[1] != vocab:
        raise ValueError("classes must be [n_classes, vocab]")
    return c, c.shape[0]


def cue_scan(tokens, traj_offsets, pat_tokens, pat_offsets, pat_cue, n_cues, terminator,
             mode: int = 0, classes=None, decimal_rule=None):
    """Pattern elements < 0 are token classes (row -1-e of ``classes``);
    ``decimal_rule`` = (period, digit_end, digit_start) class ids or None."""
    tokens = np.ascontiguousarray(tokens, np.int32)
    n_tok = tokens.shape[0]
    offs = None if traj_offsets is None else np.ascontiguousarray(traj_offsets, np.int64)
    n_traj = 1 if offs is None else offs.shape[0] - 1
    pt = np.ascontiguousarray(pat_tokens, np.int32)
    po = np.ascontiguousarray(pat_offsets, np.int32)
    pc = np.ascontiguousarray(pat_cue, np.int32)
    term_tab = np.ascontiguousarray(terminator, np.uint8)
    term = np.empty(n_tok, np.uint8)
    lib = _load()
    cap = max(1, n_tok * max(1, n_cues if mode else 1))
    occ_pos = np.empty(cap, np.int32)
    occ_pat = np.empty(cap, np.int32)
    cls, n_cls = _classes(classes, term_tab.shape[0])
    dec = None if decimal_rule is None else np.ascontiguousarray(decimal_rule, np.int32)
    if dec is not None and (cls is None or dec.shape != (3,) or dec.min() < 0 or dec.max() >= n_cls):
        raise ValueError("decimal_rule needs three class ids")
    n = lib.oracle_cue_scan_ex(_p(tokens), n_tok, _p(offs), n_traj, _p(pt), _p(po),
                               po.shape[0] - 1, _p(pc), n_cues, _p(term_tab), mode, _p(cls), n_cls,
                               term_tab.shape[0], _p(dec), _p(term), _p(occ_pos), _p(occ_pat), cap)
    return dict(term=term, occ_pos=occ_pos[:n].copy(), occ_pat=occ_pat[:n].copy())


# --------------------------------------------------------------------- H3
def windows(margin, term, traj_offsets, occ_pos, tau: float):
    margin = np.ascontiguousarray(margin, np.float32)
    term = np.ascontiguousarray(term, np.uint8)
    n_tok = margin.shape[0]
    offs = None if traj_offsets is None else np.ascontiguousarray(traj_offsets, np.int64)
    n_traj = 1 if offs is None else offs.shape[0] - 1
    occ_pos = np.ascontiguousarray(occ_pos, np.int32)
    k = occ_pos.shape[0]
    out = dict(seg_end=np.empty(k, np.int32), seg_mean=np.empty(k), seg_min=np.empty(k),
               seg_lowfrac=np.empty(k), seg_sum=np.empty(k), seg_low=np.empty(k, np.int32),
               seg_invalid=np.empty(k, np.int8))
    _load().oracle_windows(_p(margin), _p(term), n_tok, _p(offs), n_traj, _p(occ_pos), k,
                           tau, _p(out["seg_end"]), _p(out["seg_mean"]), _p(out["seg_min"]),
                           _p(out["seg_lowfrac"]), _p(out["seg_sum"]), _p(out["seg_low"]),
                           _p(out["seg_invalid"]))
    return out


# ------------------------------------------------------------------ H4-H7
def cue_stats(margin, traj_offsets, think_end_pos, occ_pos, occ_pat, pat_cue, n_cues, tau,
              win, min_count: int = 3, rule: int = 0):
    """Per-cue + global summaries (list of dicts, global last)."""
    margin = np.ascontiguousarray(margin, np.float32)
    offs = None if traj_offsets is None else np.ascontiguousarray(traj_offsets, np.int64)
    n_traj = 1 if offs is None else offs.shape[0] - 1
    tep = None if think_end_pos is None else np.ascontiguousarray(think_end_pos, np.int64)
    occ_pos = np.ascontiguousarray(occ_pos, np.int32)
    occ_pat = np.ascontiguousarray(occ_pat, np.int32)
    pc = np.ascontiguousarray(pat_cue, np.int32)
    out = (Summary * (n_cues + 1))()
    _load().oracle_cue_stats(_p(margin), margin.shape[0], _p(offs), n_traj, _p(tep),
                             _p(occ_pos), _p(occ_pat), occ_pos.shape[0], _p(pc), n_cues, tau,
                             _p(win["seg_end"]), _p(win["seg_mean"]), _p(win["seg_min"]),
                             _p(win["seg_sum"]), _p(win["seg_low"]), _p(win["seg_invalid"]),
                             min_count, rule, C.cast(out, C.c_void_p))
    return [{f: getattr(s, f) for f, _ in Summary._fields_} for s in out]


def analyze(margin, tokens, traj_offsets, pat_tokens, pat_offsets, pat_cue, n_cues,
            terminator, tau=0.5, think_end_pos=None, mode=0, min_count=3, rule=0,
            classes=None, decimal_rule=None):
    """H2 -> H3 -> H4..H7 on given margins: the full offline statistics."""
    scan = cue_scan(tokens, traj_offsets, pat_tokens, pat_offsets, pat_cue, n_cues,
                    terminator, mode, classes, decimal_rule)
    win = windows(margin, scan["term"], traj_offsets, scan["occ_pos"], tau)
    summ = cue_stats(margin, traj_offsets, think_end_pos, scan["occ_pos"], scan["occ_pat"],
                     pat_cue, n_cues, tau, win, min_count, rule)
    return scan, win, summ


# --------------------------------------------------------------------- H8
def step_one(tok, margin, state, hist, small_run, pat_tokens, pat_offsets, pat_cue,
             terminator, think_end_token, margin_gate=-1.0, max_small_segment=0, classes=None):
    """One sequence, one decode step.  Returns (flag, cue, state, hist, small_run)."""
    st = np.array([state], np.uint8)
    h = np.ascontiguousarray(np.array(hist, np.int32).copy())
    sr = np.array([small_run], np.int32)
    cue = C.c_int32()
    pt = np.ascontiguousarray(pat_tokens, np.int32)
    po = np.ascontiguousarray(pat_offsets, np.int32)
    pc = np.ascontiguousarray(pat_cue, np.int32)
    term_tab = np.ascontiguousarray(terminator, np.uint8)
    cls, n_cls = _classes(classes, term_tab.shape[0])
    flag = _load().oracle_step_one_ex(int(tok), float(margin), _p(st), _p(h), _p(sr), _p(pt),
                                      _p(po), po.shape[0] - 1, _p(pc), _p(term_tab),
                                      term_tab.shape[0], think_end_token, margin_gate,
                                      max_small_segment, _p(cls), n_cls, C.byref(cue))
    return flag, cue.value, int(st[0]), h, int(sr[0])


# ------------------------------------------------------------------ N2
def sample_rows(logits, u, dtype: str | None = None, vocab: int | None = None,
                temperature: float = 0.6, top_k: int = 20, top_p: float = 0.95):
    """Per row: the token drawn by temperature / top-k / top-p sampling with
    the given uniforms (inverse CDF, R20); -1 for rows with status != 0."""
    a = np.ascontiguousarray(logits)
    code = _dtype_code(a, dtype)
    n, stride = a.shape
    vocab = stride if vocab is None else vocab
    u = np.asarray(u, np.float64)
    lib = _load()
    out = np.empty(n, np.int32)
    for r in range(n):
        out[r] = lib.oracle_sample_row(a[r].ctypes.data_as(C.c_void_p), code, vocab,
                                       1.0 / temperature, top_k, top_p, float(u[r]))
    return out


# ------------------------------------------------------------------ N3
def offload(n_tok, traj_offsets, think_end_pos, occ_pos, occ_pat, seg_end, pat_offsets, pat_cue,
            cue_selected):
    """Per trajectory [large, small_reasoning, answer] token counts (R17)."""
    offs = None if traj_offsets is None else np.ascontiguousarray(traj_offsets, np.int64)
    n_traj = 1 if offs is None else offs.shape[0] - 1
    tep = None if think_end_pos is None else np.ascontiguousarray(think_end_pos, np.int64)
    occ_pos = np.ascontiguousarray(occ_pos, np.int32)
    occ_pat = np.ascontiguousarray(occ_pat, np.int32)
    seg_end = np.ascontiguousarray(seg_end, np.int32)
    po = np.ascontiguousarray(pat_offsets, np.int32)
    pc = np.ascontiguousarray(pat_cue, np.int32)
    sel = np.ascontiguousarray(cue_selected, np.uint8)
    out = np.zeros((n_traj, 3), np.int64)
    _load().oracle_offload(n_tok, _p(offs), n_traj, _p(tep), _p(occ_pos), _p(occ_pat),
                           occ_pos.shape[0], _p(seg_end), _p(po), _p(pc), _p(sel), _p(out))
    return out
