"""RelayGen (arXiv 2602.06454) hot path on B200 — thin Python binding of librelay.so.

Argument marshalling only: every step of the path (margins, cue scan, segment
statistics, decode-step switch) runs in the sm_100a kernels of ``librelay.so``
behind the C ABI declared in ``include/relay.h``.  PyTorch supplies device
memory, streams and process groups.  There is NO CPU fallback: importing this
package without a built ``librelay.so`` raises, and every call raises
``RelayError`` on a non-OK status.

Names follow the C ABI (``relay_margin_rows`` -> ``margin_rows`` ...).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from ._build import LIB_PATH, NVCC_FLAGS  # noqa: E402,F401
from ._build import build_lib as _build_lib  # noqa: E402

DT = {"bf16": 0, "f16": 1, "f32": 2}
FLAG_NONE, FLAG_L2S, FLAG_S2L, FLAG_TO_ANSWER, FLAG_S2L_BUDGET = 0, 1, 2, 3, 4
STAT_FIELDS = 8
F_N, F_SUM_MQ, F_SUM_MQ2, F_SUM_WQ, F_SUM_LEN, F_SUM_LOW, F_TRIG, F_INVALID, F_MIN0 = range(9)
HIST = 7


class RelayError(RuntimeError):
    pass


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile librelay.so for sm_100a with nvcc (works without a GPU)."""
    return _build_lib(force=force, verbose=verbose)


def _load():
    # RELAY_LIB: another build of the same library (A/B tuning tools only)
    path = os.environ.get("RELAY_LIB", LIB_PATH)
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(path)
    P, i32, i64, f32, u32, sz = C.c_void_p, C.c_int32, C.c_int64, C.c_float, C.c_uint32, C.c_size_t
    sig = {
        "relay_version": (C.c_int, []),
        "relay_status_string": (C.c_char_p, [C.c_int]),
        "relay_last_error": (C.c_char_p, []),
        "relay_margin_rows": (C.c_int, [P, C.c_int, i64, i64, i64, f32, P, P, P, P, P, P]),
        "relay_margin_partials": (C.c_int, [P, C.c_int, i64, i64, i64, i64, f32, P, P]),
        "relay_margin_combine": (C.c_int, [P, i32, i64, f32, P, P, P, P, P, P]),
        "relay_cueset_create": (C.c_int, [P, P, i32, P, i32, P, i64, i32, u32, P]),
        "relay_cueset_create_ex": (C.c_int, [P, P, i32, P, i32, P, i64, i32, u32, P, i32, P, P]),
        "relay_cueset_destroy": (C.c_int, [P]),
        "relay_cueset_n_cues": (i32, [P]),
        "relay_workspace_bytes": (sz, [i64, i64, i32]),
        "relay_workspace_init": (C.c_int, [P, sz, i64, i64, i32, P]),
        "relay_workspace_release": (C.c_int, [P]),
        "relay_cue_scan": (C.c_int, [P, P, i64, P, i32, P, P, P, i64, P, P, sz, P]),
        "relay_segment_reduce": (C.c_int, [P, P, i64, P, i32, P, P, P, P, P, i64, f32, P, P, P, P,
                                           P, i32, i32, u32, P, sz, P]),
        "relay_segment_reduce_p2p": (C.c_int, [P, P, P, i64, P, i32, P, P, P, P, P, i64, f32, P, P, P, P,
                                               P, i32, i32, u32, P, sz, P]),
        "relay_stats_init": (C.c_int, [P, i32, i32, i32, P]),
        "relay_stats_init_tables": (C.c_int, [P, i32, i32, i32, i32, P]),
        "relay_stats_merge": (C.c_int, [P, i32, P, i32, i32, i32, P]),
        "relay_stats_allreduce": (C.c_int, [P, P, i32, i32, i32, P]),
        "relay_nccl_version": (C.c_int, [P, P, i32]),
        "relay_nccl_unique_id": (C.c_int, [P]),
        "relay_nccl_comm_init": (C.c_int, [P, i32, i32, P]),
        "relay_nccl_comm_destroy": (C.c_int, [P]),
        "relay_read_probe_words": (i32, []),
        "relay_read_probe": (C.c_int, [P, i64, P, P]),
        "relay_tp_exchange_create": (C.c_int, [i32, i32, i64, P, P]),
        "relay_tp_exchange_connect": (C.c_int, [P, P]),
        "relay_tp_exchange_destroy": (C.c_int, [P]),
        "relay_margin_rows_tp": (C.c_int, [P, P, C.c_int, i64, i64, i64, i64, f32, P, P, P, P, P, P]),
        "relay_stats_allreduce_p2p": (C.c_int, [P, P, i32, i32, i32, P]),
        "relay_offload_estimate": (C.c_int, [P, i64, P, i32, P, P, P, P, i64, P, P, P, P]),
        "relay_stats_words": (sz, [i32, i32]),
        "relay_stats_finalize": (C.c_int, [P, i32, i32, i64, i32, P]),
        "relay_step_switch": (C.c_int, [P, P, C.c_int, i32, i64, i64, f32, P, P, P, P, f32, i32,
                                        P, P, P, P, P, P, sz, P]),
        "relay_step_sample": (C.c_int, [P, P, C.c_int, i32, i64, i64, f32, f32, i32, f32, P, P, P,
                                        P, f32, i32, P, P, P, P, P, P, P, sz, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = _load()
EXPORTS = ("relay_version", "relay_status_string", "relay_last_error", "relay_margin_rows",
           "relay_margin_partials", "relay_margin_combine",
           "relay_cueset_create", "relay_cueset_create_ex", "relay_cueset_destroy", "relay_cueset_n_cues",
           "relay_workspace_bytes", "relay_workspace_init", "relay_workspace_release", "relay_cue_scan",
           "relay_segment_reduce", "relay_stats_init", "relay_stats_init_tables",
           "relay_stats_words", "relay_stats_merge", "relay_stats_allreduce",
           "relay_nccl_version", "relay_nccl_unique_id", "relay_nccl_comm_init", "relay_nccl_comm_destroy",
           "relay_stats_finalize", "relay_step_switch", "relay_offload_estimate",
           "relay_step_sample", "relay_tp_exchange_create", "relay_tp_exchange_connect",
           "relay_tp_exchange_destroy", "relay_margin_rows_tp", "relay_read_probe_words",
           "relay_read_probe", "relay_stats_allreduce_p2p", "relay_segment_reduce_p2p")


def _check(rc: int, what: str):
    if rc != 0:
        msg = _lib.relay_last_error().decode()
        raise RelayError(f"{what}: {_lib.relay_status_string(rc).decode()} ({msg})")


def version() -> int:
    return _lib.relay_version()


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


def _dtype_of(t) -> int:
    import torch
    m = {torch.bfloat16: 0, torch.float16: 1, torch.float32: 2}
    if t.dtype not in m:
        raise RelayError(f"unsupported logits dtype {t.dtype}")
    return m[t.dtype]


def _need_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise RelayError("all tensors must be CUDA tensors (there is no CPU path)")


# ------------------------------------------------------------------- H1
def margin_rows(logits, vocab: int | None = None, inv_temperature: float = 1.0, out=None,
                want_lse: bool = True, stream=None):
    """relay_margin_rows on a [n_rows, row_stride] CUDA tensor (rows contiguous
    in their last dim).  Returns dict(margin, top1, top2, lse, status)."""
    import torch
    _need_cuda(logits)
    if logits.dim() != 2 or logits.stride(1) != 1:
        raise RelayError("logits must be 2-D with unit stride in the vocabulary dim")
    n = logits.shape[0]
    stride = logits.stride(0) if n > 1 else logits.shape[1]
    vocab = logits.shape[1] if vocab is None else vocab
    dev = logits.device
    if out is None:
        out = dict(margin=torch.empty(n, dtype=torch.float32, device=dev),
                   top1=torch.empty(n, dtype=torch.int32, device=dev),
                   top2=torch.empty(n, dtype=torch.int32, device=dev),
                   lse=torch.empty(n, dtype=torch.float32, device=dev) if want_lse else None,
                   status=torch.empty(n, dtype=torch.uint8, device=dev))
    rc = _lib.relay_margin_rows(_ptr(logits), _dtype_of(logits), n, vocab, stride,
                                float(inv_temperature), _ptr(out["margin"]), _ptr(out.get("top1")),
                                _ptr(out.get("top2")), _ptr(out.get("lse")),
                                _ptr(out.get("status")), _stream(stream))
    _check(rc, "relay_margin_rows")
    return out


# ------------------------------------------------- H1 across TP ranks (N1)
PARTIAL_WORDS = 8


def margin_partials(logits_shard, col_offset: int, inv_temperature: float = 1.0, out=None,
                    stream=None):
    """relay_margin_partials: per-row partials [n_rows, 8] of a vocabulary shard
    (columns [col_offset, col_offset + shard width) of the full rows)."""
    import torch
    _need_cuda(logits_shard)
    if logits_shard.dim() != 2 or logits_shard.stride(1) != 1:
        raise RelayError("logits shard must be 2-D with unit stride in the vocabulary dim")
    n = logits_shard.shape[0]
    stride = logits_shard.stride(0) if n > 1 else logits_shard.shape[1]
    if out is None:
        out = torch.empty((n, PARTIAL_WORDS), dtype=torch.float32, device=logits_shard.device)
    rc = _lib.relay_margin_partials(_ptr(logits_shard), _dtype_of(logits_shard), n,
                                    logits_shard.shape[1], stride, int(col_offset),
                                    float(inv_temperature), _ptr(out), _stream(stream))
    _check(rc, "relay_margin_partials")
    return out


def margin_combine(partials, inv_temperature: float = 1.0, out=None, stream=None):
    """relay_margin_combine on stacked partials [n_shards, n_rows, 8]."""
    import torch
    _need_cuda(partials)
    parts = partials.contiguous()
    P, n = parts.shape[0], parts.shape[1]
    dev = parts.device
    if out is None:
        out = dict(margin=torch.empty(n, dtype=torch.float32, device=dev),
                   top1=torch.empty(n, dtype=torch.int32, device=dev),
                   top2=torch.empty(n, dtype=torch.int32, device=dev),
                   lse=torch.empty(n, dtype=torch.float32, device=dev),
                   status=torch.empty(n, dtype=torch.uint8, device=dev))
    rc = _lib.relay_margin_combine(_ptr(parts), P, n, float(inv_temperature), _ptr(out["margin"]),
                                   _ptr(out.get("top1")), _ptr(out.get("top2")),
                                   _ptr(out.get("lse")), _ptr(out.get("status")), _stream(stream))
    _check(rc, "relay_margin_combine")
    return out


def margin_rows_tp(logits_shard, col_offset: int, group=None, inv_temperature: float = 1.0):
    """The margin of rows whose vocabulary is sharded over a tensor-parallel
    group: shard partials (32 B/row) -> one all-gather -> combine, on every rank."""
    import torch
    import torch.distributed as dist
    part = margin_partials(logits_shard, col_offset, inv_temperature)
    world = dist.get_world_size(group)
    gathered = torch.empty((world * part.shape[0], part.shape[1]), dtype=part.dtype,
                           device=part.device)
    dist.all_gather_into_tensor(gathered, part, group=group)   # ranks concatenated on dim 0
    return margin_combine(gathered.view(world, part.shape[0], part.shape[1]), inv_temperature)


def read_probe(buf, out=None, stream=None):
    """relay_read_probe: a read-only stream over ``buf`` (a measurement
    utility: the read-only HBM ceiling bench.py quotes next to K1)."""
    import torch
    _need_cuda(buf)
    if out is None:
        out = torch.zeros(_lib.relay_read_probe_words(), dtype=torch.int32, device=buf.device)
    _check(_lib.relay_read_probe(_ptr(buf), buf.numel() * buf.element_size() // 16 * 16, _ptr(out),
                                 _stream(stream)), "relay_read_probe")
    return out


IPC_HANDLE_BYTES = 64


class TpExchange:
    """relay_tp_exchange_create / connect / destroy: the receive buffers of a
    tensor-parallel group for relay_margin_rows_tp (N1 with the exchange
    fused into the streaming kernel over peer memory).  Collective: every
    rank constructs it; the CUDA IPC handles are gathered over ``group``
    (any torch.distributed backend)."""

    def __init__(self, rows_cap: int, group=None):
        import torch.distributed as dist
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.rows_cap = int(rows_cap)
        h = C.create_string_buffer(IPC_HANDLE_BYTES)
        x = C.c_void_p()
        _check(_lib.relay_tp_exchange_create(self.rank, self.world, self.rows_cap, h, C.byref(x)),
               "relay_tp_exchange_create")
        self._x = x
        handles = [None] * self.world
        dist.all_gather_object(handles, h.raw, group=group)
        buf = C.create_string_buffer(b"".join(handles), IPC_HANDLE_BYTES * self.world)
        _check(_lib.relay_tp_exchange_connect(self._x, buf), "relay_tp_exchange_connect")

    def margin_rows(self, logits_shard, col_offset: int, inv_temperature: float = 1.0, out=None,
                    stream=None):
        """relay_margin_rows_tp: full-row margin / top1 / top2 / lse / status of
        rows whose columns [col_offset, col_offset + width) this rank holds."""
        import torch
        _need_cuda(logits_shard)
        if logits_shard.dim() != 2 or logits_shard.stride(1) != 1:
            raise RelayError("logits shard must be 2-D with unit stride in the vocabulary dim")
        n = logits_shard.shape[0]
        stride = logits_shard.stride(0) if n > 1 else logits_shard.shape[1]
        dev = logits_shard.device
        if out is None:
            out = dict(margin=torch.empty(n, dtype=torch.float32, device=dev),
                       top1=torch.empty(n, dtype=torch.int32, device=dev),
                       top2=torch.empty(n, dtype=torch.int32, device=dev),
                       lse=torch.empty(n, dtype=torch.float32, device=dev),
                       status=torch.empty(n, dtype=torch.uint8, device=dev))
        rc = _lib.relay_margin_rows_tp(self._x, _ptr(logits_shard), _dtype_of(logits_shard), n,
                                       logits_shard.shape[1], stride, int(col_offset), float(inv_temperature),
                                       _ptr(out["margin"]), _ptr(out.get("top1")), _ptr(out.get("top2")),
                                       _ptr(out.get("lse")), _ptr(out.get("status")), _stream(stream))
        _check(rc, "relay_margin_rows_tp")
        return out

    def stats_allreduce(self, stats, n_cues: int, n_tables: int = 1, stream=None):
        """relay_stats_allreduce_p2p: H6 over peer memory (no NCCL); the
        exchange must be sized for the table (``StatsExchange`` does it)."""
        _need_cuda(stats)
        _check(_lib.relay_stats_allreduce_p2p(self._x, _ptr(stats), n_tables, n_cues, self.world,
                                              _stream(stream)), "relay_stats_allreduce_p2p")
        return stats

    def close(self):
        if getattr(self, "_x", None):
            _lib.relay_tp_exchange_destroy(self._x)
            self._x = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def StatsExchange(n_cues: int, n_tables: int = 1, group=None) -> "TpExchange":
    """A peer-memory exchange sized for the statistics table(s) of ``n_cues``
    over ``group`` (collective), for ``TpExchange.stats_allreduce``."""
    import torch.distributed as dist
    words = stats_words(n_cues, dist.get_world_size(group)) * n_tables
    return TpExchange(rows_cap=(words * 8 + 8 + 31) // 32, group=group)


# --------------------------------------------------------------- cue set
class CueSet:
    """relay_cueset_create_ex / destroy.  Host arrays (numpy) in, device copy
    owned.  ``classes`` ([n_classes, vocab] 0/1) makes negative pattern
    elements token classes (N4); ``decimal_rule`` = (period, digit_end,
    digit_start) class ids turns on the decimal-number sentence rule."""

    def __init__(self, pat_tokens, pat_offsets, pat_cue, n_cues: int, terminator, vocab: int,
                 think_end: int = -1, mode: int = 0, classes=None, decimal_rule=None):
        self.pat_tokens = np.ascontiguousarray(pat_tokens, np.int32)
        self.pat_offsets = np.ascontiguousarray(pat_offsets, np.int32)
        self.pat_cue = np.ascontiguousarray(pat_cue, np.int32)
        self.terminator = np.ascontiguousarray(terminator, np.uint8)
        self.n_cues, self.vocab, self.think_end, self.mode = int(n_cues), int(vocab), int(think_end), int(mode)
        if self.terminator.shape[0] < vocab:
            raise RelayError("terminator table shorter than vocab")
        self.classes = None
        n_classes = 0
        if classes is not None:
            self.classes = np.ascontiguousarray(np.asarray(classes).astype(bool).astype(np.uint8))
            if self.classes.ndim != 2 or self.classes.shape[1] != vocab:
                raise RelayError("classes must be [n_classes, vocab]")
            n_classes = self.classes.shape[0]
        self.decimal_rule = None if decimal_rule is None else np.ascontiguousarray(decimal_rule, np.int32)
        if self.decimal_rule is not None and self.decimal_rule.shape != (3,):
            raise RelayError("decimal_rule must hold 3 class ids")
        h = C.c_void_p()
        rc = _lib.relay_cueset_create_ex(self.pat_tokens.ctypes.data_as(C.c_void_p),
                                         self.pat_offsets.ctypes.data_as(C.c_void_p),
                                         self.pat_offsets.shape[0] - 1,
                                         self.pat_cue.ctypes.data_as(C.c_void_p), self.n_cues,
                                         self.terminator.ctypes.data_as(C.c_void_p), self.vocab,
                                         self.think_end, self.mode,
                                         None if self.classes is None else
                                         self.classes.ctypes.data_as(C.c_void_p), n_classes,
                                         None if self.decimal_rule is None else
                                         self.decimal_rule.ctypes.data_as(C.c_void_p), C.byref(h))
        _check(rc, "relay_cueset_create_ex")
        self._h = h

    @classmethod
    def from_synth(cls, cs, mode: int = 0):
        return cls(cs.pat_tokens, cs.pat_offsets, cs.pat_cue, cs.n_cues, cs.terminator, cs.vocab,
                   cs.think_end, mode)

    @property
    def handle(self):
        if self._h is None:
            raise RelayError("cue set destroyed")
        return self._h

    def destroy(self):
        if getattr(self, "_h", None) is not None:
            _lib.relay_cueset_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def workspace_bytes(n_tok: int = 0, occ_capacity: int = 0, batch: int = 0) -> int:
    return int(_lib.relay_workspace_bytes(n_tok, occ_capacity, batch))


def workspace(n_tok: int = 0, occ_capacity: int = 0, batch: int = 0, device="cuda", stream=None):
    """A workspace for up to ``n_tok`` positions / ``occ_capacity`` occurrences
    (cue_scan, segment_reduce) and ``batch`` rows (step_switch, step_sample),
    zeroed and registered with the library (relay_workspace_init); released
    when the tensor is garbage-collected."""
    import weakref

    import torch
    nb = workspace_bytes(n_tok, occ_capacity, batch)
    ws = torch.empty(max(nb, 1), dtype=torch.uint8, device=device)
    _check(_lib.relay_workspace_init(_ptr(ws), ws.numel(), n_tok, occ_capacity, batch, _stream(stream)),
           "relay_workspace_init")
    weakref.finalize(ws, _lib.relay_workspace_release, C.c_void_p(ws.data_ptr()))
    return ws


# ------------------------------------------------------------------- H2
def cue_scan(cs: CueSet, tokens, traj_offsets=None, occ_capacity: int | None = None, ws=None,
             out=None, stream=None):
    import torch
    _need_cuda(tokens, traj_offsets)
    n_tok = tokens.shape[0]
    dev = tokens.device
    cap = n_tok * (cs.n_cues if cs.mode else 1) if occ_capacity is None else occ_capacity
    if ws is None:
        ws = workspace(n_tok, cap, 0, dev, stream)
    if out is None:
        out = dict(term_bits=torch.zeros((n_tok + 31) // 32 + 1, dtype=torch.int32, device=dev),
                   occ_pos=torch.empty(max(cap, 1), dtype=torch.int32, device=dev),
                   occ_pat=torch.empty(max(cap, 1), dtype=torch.int32, device=dev),
                   n_occ=torch.zeros(1, dtype=torch.int64, device=dev))
    n_traj = 1 if traj_offsets is None else traj_offsets.shape[0] - 1
    rc = _lib.relay_cue_scan(cs.handle, _ptr(tokens), n_tok, _ptr(traj_offsets), n_traj,
                             _ptr(out["term_bits"]), _ptr(out["occ_pos"]), _ptr(out["occ_pat"]),
                             cap, _ptr(out["n_occ"]), _ptr(ws), ws.numel(), _stream(stream))
    _check(rc, "relay_cue_scan")
    out["capacity"] = cap
    return out


def stats_words(n_cues: int, world_size: int = 1) -> int:
    return int(_lib.relay_stats_words(n_cues, world_size))


def stats_init(stats, n_cues: int, rank: int = 0, world_size: int = 1, stream=None,
               n_tables: int = 1):
    _check(_lib.relay_stats_init_tables(_ptr(stats), n_tables, n_cues, rank, world_size,
                                        _stream(stream)), "relay_stats_init_tables")
    return stats


def new_stats(n_cues: int, rank: int = 0, world_size: int = 1, device="cuda", stream=None,
              n_tables: int = 1):
    """One table, or ``n_tables`` consecutive ones (per-trajectory tables)."""
    import torch
    st = torch.empty(n_tables * stats_words(n_cues, world_size), dtype=torch.int64, device=device)
    return stats_init(st, n_cues, rank, world_size, stream, n_tables)


def stats_merge(host_tables: np.ndarray, n_cues: int, world_size: int = 1, mask=None, rank: int = 0):
    """Host merge of this rank's per-trajectory tables (``mask``: which ones,
    default all) into one table that ``stats_finalize`` (or, first, the SUM
    all-reduce) takes."""
    words = stats_words(n_cues, world_size)
    ht = np.ascontiguousarray(host_tables).view(np.uint64).reshape(-1)
    if ht.shape[0] % words:
        raise RelayError("tables length is not a multiple of the table size")
    n_tables = ht.shape[0] // words
    m = None
    if mask is not None:
        m = np.ascontiguousarray(np.asarray(mask, dtype=bool).astype(np.uint8))
        if m.shape != (n_tables,):
            raise RelayError("mask must have one entry per table")
    out = np.empty(words, dtype=np.uint64)
    rc = _lib.relay_stats_merge(ht.ctypes.data_as(C.c_void_p), n_tables,
                                None if m is None else m.ctypes.data_as(C.c_void_p), n_cues,
                                rank, world_size, out.ctypes.data_as(C.c_void_p))
    _check(rc, "relay_stats_merge")
    return out


# ------------------------------------------------------------------- H6
def stats_allreduce(comm_ptr: int, stats, n_cues: int, world_size: int, n_tables: int = 1,
                    stream=None):
    """In-place SUM all-reduce of ``n_tables`` stats tables over the NCCL
    communicator ``comm_ptr`` (an ncclComm_t as an int: ``NcclComm.ptr`` or
    torch's ``ProcessGroupNCCL._comm_ptr()``)."""
    _need_cuda(stats)
    if stats.numel() < n_tables * stats_words(n_cues, world_size):
        raise RelayError("stats too short")
    _check(_lib.relay_stats_allreduce(C.c_void_p(comm_ptr), _ptr(stats), n_tables, n_cues,
                                      world_size, _stream(stream)), "relay_stats_allreduce")
    return stats


def nccl_version():
    """(ncclGetVersion code, file) of the NCCL librelay resolved at run time."""
    v = C.c_int32(0)
    buf = C.create_string_buffer(4096)
    _check(_lib.relay_nccl_version(C.byref(v), buf, 4096), "relay_nccl_version")
    return int(v.value), buf.value.decode(errors="replace")


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(_lib.relay_nccl_unique_id(C.cast(buf, C.c_void_p)), "relay_nccl_unique_id")
    return bytes(buf)


class NcclComm:
    """A library-owned NCCL communicator (collective constructor: every rank,
    its CUDA device current).  ``uid`` is rank 0's ``nccl_unique_id()``, sent
    to the others by the caller (``NcclComm.from_group`` does it through
    torch.distributed)."""

    def __init__(self, uid: bytes, world_size: int, rank: int):
        if len(uid) != 128:
            raise RelayError("uid must be 128 bytes")
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        out = C.c_void_p()
        _check(_lib.relay_nccl_comm_init(C.cast(buf, C.c_void_p), world_size, rank, C.byref(out)),
               "relay_nccl_comm_init")
        self.ptr, self.world_size, self.rank = out.value, world_size, rank

    @classmethod
    def from_group(cls, rank: int, world_size: int, group=None):
        import torch.distributed as dist
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls(obj[0], world_size, rank)

    def close(self):
        if self.ptr:
            _check(_lib.relay_nccl_comm_destroy(C.c_void_p(self.ptr)), "relay_nccl_comm_destroy")
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- H3-H5
def segment_reduce(cs: CueSet, margin, scan: dict, traj_offsets=None, think_end_pos=None,
                   tau: float = 0.5, stats=None, rank: int = 0, world_size: int = 1, ws=None,
                   out=None, stream=None, per_trajectory: bool = False, exchange=None):
    """H3-H5.  ``per_trajectory``: one stats table per trajectory (merge with
    ``stats_merge``).  ``exchange`` (a ``StatsExchange``): H6 fused into the
    same kernel — its last CTA all-reduces the finished table(s) over peer
    memory (relay_segment_reduce_p2p; collective over the exchange's group)."""
    import torch
    _need_cuda(margin, traj_offsets, think_end_pos)
    n_tok = margin.shape[0]
    cap = scan["capacity"]
    dev = margin.device
    if ws is None:
        ws = workspace(n_tok, cap, 0, dev, stream)
    n_traj = 1 if traj_offsets is None else traj_offsets.shape[0] - 1
    if stats is None:
        stats = new_stats(cs.n_cues, rank, world_size, dev, stream,
                          n_traj if per_trajectory else 1)
    elif stats.numel() < (n_traj if per_trajectory else 1) * stats_words(cs.n_cues, world_size):
        raise RelayError("stats too short for the table count")
    c1 = max(cap, 1)
    if out is None:
        out = dict(seg_end=torch.empty(c1, dtype=torch.int32, device=dev),
                   seg_mean=torch.empty(c1, dtype=torch.float32, device=dev),
                   seg_min=torch.empty(c1, dtype=torch.float32, device=dev),
                   seg_lowfrac=torch.empty(c1, dtype=torch.float32, device=dev))
    args = (cs.handle, _ptr(margin), n_tok, _ptr(traj_offsets), n_traj, _ptr(think_end_pos),
            _ptr(scan["term_bits"]), _ptr(scan["occ_pos"]), _ptr(scan["occ_pat"]), _ptr(scan["n_occ"]),
            cap, float(tau), _ptr(out["seg_end"]), _ptr(out["seg_mean"]), _ptr(out["seg_min"]),
            _ptr(out["seg_lowfrac"]), _ptr(stats), rank, world_size, 1 if per_trajectory else 0,
            _ptr(ws), ws.numel(), _stream(stream))
    if exchange is not None:
        _check(_lib.relay_segment_reduce_p2p(exchange._x, *args), "relay_segment_reduce_p2p")
    else:
        _check(_lib.relay_segment_reduce(*args), "relay_segment_reduce")
    out["stats"] = stats
    return out


def offload_estimate(cs: CueSet, scan: dict, seg: dict, cue_selected, n_tok: int,
                     traj_offsets=None, think_end_pos=None, stream=None):
    """N3: per-trajectory [large, small_reasoning, answer] token counts of the
    runtime switching replayed with ``cue_selected`` (uint8 CUDA tensor [n_cues])."""
    import torch
    _need_cuda(cue_selected, traj_offsets, think_end_pos)
    n_traj = 1 if traj_offsets is None else traj_offsets.shape[0] - 1
    out = torch.empty((n_traj, 3), dtype=torch.int64, device=cue_selected.device)
    rc = _lib.relay_offload_estimate(cs.handle, n_tok, _ptr(traj_offsets), n_traj,
                                     _ptr(think_end_pos), _ptr(scan["occ_pos"]), _ptr(scan["occ_pat"]),
                                     _ptr(scan["n_occ"]), scan["capacity"], _ptr(seg["seg_end"]),
                                     _ptr(cue_selected), _ptr(out), _stream(stream))
    _check(rc, "relay_offload_estimate")
    return out


class Summary(C.Structure):
    _fields_ = [("n", C.c_int64), ("mean", C.c_double), ("std", C.c_double), ("se", C.c_double),
                ("token_mean", C.c_double), ("min", C.c_double), ("low_frac", C.c_double),
                ("n_triggers", C.c_int64), ("n_invalid", C.c_int64), ("selected", C.c_int32)]


def stats_finalize(host_stats: np.ndarray, n_cues: int, world_size: int = 1, min_count: int = 3,
                   rule: int = 0):
    """H7 on the host: list of per-cue dicts, global row last."""
    hs = np.ascontiguousarray(host_stats).view(np.uint64)
    if hs.shape[0] < stats_words(n_cues, world_size):
        raise RelayError("stats table too short")
    out = (Summary * (n_cues + 1))()
    rc = _lib.relay_stats_finalize(hs.ctypes.data_as(C.c_void_p), n_cues, world_size, min_count,
                                   rule, C.cast(out, C.c_void_p))
    _check(rc, "relay_stats_finalize")
    return [{f: getattr(s, f) for f, _ in Summary._fields_} for s in out]


# ------------------------------------------------------------------- H8
def step_switch(cs: CueSet, logits, state, hist, small_run=None, sampled=None, vocab=None,
                inv_temperature: float = 1.0, margin_gate: float = -1.0,
                max_small_segment: int = 0, ws=None, out=None, stream=None):
    import torch
    _need_cuda(logits, state, hist, small_run, sampled)
    B = logits.shape[0]
    stride = logits.stride(0) if B > 1 else logits.shape[1]
    vocab = logits.shape[1] if vocab is None else vocab
    dev = logits.device
    if ws is None:
        ws = workspace(0, 0, B, dev, stream)
    if out is None:
        out = dict(margin=torch.empty(B, dtype=torch.float32, device=dev),
                   top1=torch.empty(B, dtype=torch.int32, device=dev),
                   top2=torch.empty(B, dtype=torch.int32, device=dev),
                   flag=torch.empty(B, dtype=torch.uint8, device=dev),
                   cue_id=torch.empty(B, dtype=torch.int16, device=dev))
    rc = _lib.relay_step_switch(cs.handle, _ptr(logits), _dtype_of(logits), B, vocab, stride,
                                float(inv_temperature), _ptr(sampled), _ptr(state), _ptr(hist),
                                _ptr(small_run), float(margin_gate), int(max_small_segment),
                                _ptr(out["margin"]), _ptr(out.get("top1")), _ptr(out.get("top2")),
                                _ptr(out["flag"]), _ptr(out["cue_id"]), _ptr(ws), ws.numel(),
                                _stream(stream))
    _check(rc, "relay_step_switch")
    return out


# ------------------------------------------------------------------- N2
def step_sample(cs: CueSet, logits, uniform, state, hist, small_run=None, temperature: float = 0.6,
                top_k: int = 20, top_p: float = 0.95, vocab=None, inv_temperature: float = 1.0,
                margin_gate: float = -1.0, max_small_segment: int = 0, ws=None, out=None,
                stream=None):
    """One decode step with the token drawn on the device (temperature / top-k /
    top-p, inverse CDF with the caller's ``uniform`` [B] in [0, 1)), then the
    switch on the drawn token.  ``out`` gains ``sampled`` (int32 [B])."""
    import torch
    _need_cuda(logits, uniform, state, hist, small_run)
    B = logits.shape[0]
    stride = logits.stride(0) if B > 1 else logits.shape[1]
    vocab = logits.shape[1] if vocab is None else vocab
    dev = logits.device
    if ws is None:
        ws = workspace(0, 0, B, dev, stream)
    if out is None:
        out = dict(margin=torch.empty(B, dtype=torch.float32, device=dev),
                   top1=torch.empty(B, dtype=torch.int32, device=dev),
                   top2=torch.empty(B, dtype=torch.int32, device=dev),
                   sampled=torch.empty(B, dtype=torch.int32, device=dev),
                   flag=torch.empty(B, dtype=torch.uint8, device=dev),
                   cue_id=torch.empty(B, dtype=torch.int16, device=dev))
    rc = _lib.relay_step_sample(cs.handle, _ptr(logits), _dtype_of(logits), B, vocab, stride,
                                float(inv_temperature), float(temperature), int(top_k),
                                float(top_p), _ptr(uniform), _ptr(state), _ptr(hist),
                                _ptr(small_run), float(margin_gate), int(max_small_segment),
                                _ptr(out["margin"]), _ptr(out.get("top1")), _ptr(out.get("top2")),
                                _ptr(out["sampled"]), _ptr(out["flag"]), _ptr(out["cue_id"]),
                                _ptr(ws), ws.numel(), _stream(stream))
    _check(rc, "relay_step_sample")
    return out


# ------------------------------------------------------- whole offline pass
class Analyzer:
    """The full offline hot path for one shard: H1 margins -> H2 cue scan ->
    H3-H5 segment statistics into a uint64 table (-> H6 all-reduce -> H7 on
    the host).  Buffers are allocated once; ``run`` only launches kernels."""

    def __init__(self, cs: CueSet, n_tok: int, vocab: int, device="cuda", occ_capacity=None,
                 tau: float = 0.5, rank: int = 0, world_size: int = 1, inv_temperature=1.0,
                 overlap_scan: bool = True, per_trajectory_tables: int = 0, exchange=None):
        """``per_trajectory_tables`` = n_traj keeps one stats table per
        trajectory (``stats_merge`` any subset on the host); 0 = one table."""
        import torch
        self.cs, self.n_tok, self.vocab, self.tau = cs, n_tok, vocab, tau
        self.rank, self.world_size, self.iota = rank, world_size, inv_temperature
        self.overlap_scan = overlap_scan
        self.exchange = exchange          # StatsExchange: H6 fused into K3 (peer memory)
        self.device = torch.device(device)
        self.cap = (n_tok * (cs.n_cues if cs.mode else 1)) if occ_capacity is None else occ_capacity
        d = self.device
        self.ws = workspace(n_tok, self.cap, 0, d)
        self.rows = dict(margin=torch.empty(n_tok, dtype=torch.float32, device=d),
                         top1=torch.empty(n_tok, dtype=torch.int32, device=d),
                         top2=torch.empty(n_tok, dtype=torch.int32, device=d),
                         lse=torch.empty(n_tok, dtype=torch.float32, device=d),
                         status=torch.empty(n_tok, dtype=torch.uint8, device=d))
        c1 = max(self.cap, 1)
        self.scan = dict(term_bits=torch.zeros((n_tok + 31) // 32 + 1, dtype=torch.int32, device=d),
                         occ_pos=torch.empty(c1, dtype=torch.int32, device=d),
                         occ_pat=torch.empty(c1, dtype=torch.int32, device=d),
                         n_occ=torch.zeros(1, dtype=torch.int64, device=d), capacity=self.cap)
        self.seg = dict(seg_end=torch.empty(c1, dtype=torch.int32, device=d),
                        seg_mean=torch.empty(c1, dtype=torch.float32, device=d),
                        seg_min=torch.empty(c1, dtype=torch.float32, device=d),
                        seg_lowfrac=torch.empty(c1, dtype=torch.float32, device=d))
        self.n_tables = max(1, per_trajectory_tables)
        self.per_traj = per_trajectory_tables > 0
        self.stats = torch.empty(self.n_tables * stats_words(cs.n_cues, world_size),
                                 dtype=torch.int64, device=d)
        self._side = None

    def run(self, logits, tokens, traj_offsets=None, think_end_pos=None, stream=None,
            vocab=None, k1_events=None):
        """Launch one pass.  K2 (tokens only) runs on a side stream concurrently
        with K1; K3 joins both.  Stream-ordered, no host synchronisation."""
        import torch
        s = torch.cuda.current_stream() if stream is None else stream
        if not self.overlap_scan:
            cue_scan(self.cs, tokens, traj_offsets, self.cap, self.ws, self.scan, s)
            stats_init(self.stats, self.cs.n_cues, self.rank, self.world_size, s, self.n_tables)
        else:
            if self._side is None:
                self._side = torch.cuda.Stream(device=self.device)
                self._fork = torch.cuda.Event()
                self._join = torch.cuda.Event()
            self._fork.record(s)
            self._side.wait_event(self._fork)
            # the table reset and K2 both run beside K1 (K3 joins them)
            stats_init(self.stats, self.cs.n_cues, self.rank, self.world_size, self._side, self.n_tables)
            cue_scan(self.cs, tokens, traj_offsets, self.cap, self.ws, self.scan, self._side)
            self._join.record(self._side)
        if k1_events:
            k1_events[0].record(s)
        margin_rows(logits, vocab=vocab or self.vocab, inv_temperature=self.iota, out=self.rows,
                    stream=s)
        if k1_events:
            k1_events[1].record(s)
        if self.overlap_scan:
            s.wait_event(self._join)
        segment_reduce(self.cs, self.rows["margin"], self.scan, traj_offsets, think_end_pos,
                       self.tau, self.stats, self.rank, self.world_size, self.ws, self.seg, s,
                       per_trajectory=self.per_traj, exchange=self.exchange)
        return self.stats

    def run_streamed(self, chunks, tokens, traj_offsets=None, think_end_pos=None, stream=None,
                     vocab=None, k1_events=None):
        """The same pass with the logits streamed in row chunks (configs[4]: a
        corpus larger than HBM).  ``chunks`` yields (first_row, logits[R, V]);
        each chunk's margins land at their row offset, then H2-H5 run once over
        the whole token stream.  The caller may refill a chunk buffer as soon as
        the stream has moved past its relay_margin_rows launch."""
        import torch
        s = torch.cuda.current_stream() if stream is None else stream
        if self._side is None:
            self._side = torch.cuda.Stream(device=self.device)
            self._fork = torch.cuda.Event()
            self._join = torch.cuda.Event()
        self._fork.record(s)
        self._side.wait_event(self._fork)
        stats_init(self.stats, self.cs.n_cues, self.rank, self.world_size, self._side, self.n_tables)
        cue_scan(self.cs, tokens, traj_offsets, self.cap, self.ws, self.scan, self._side)
        self._join.record(self._side)
        if k1_events:
            k1_events[0].record(s)
        for r0, chunk in chunks:
            r1 = r0 + chunk.shape[0]
            out = {k: (v[r0:r1] if v is not None else None) for k, v in self.rows.items()}
            margin_rows(chunk, vocab=vocab or self.vocab, inv_temperature=self.iota, out=out,
                        stream=s)
        if k1_events:
            k1_events[1].record(s)
        s.wait_event(self._join)
        segment_reduce(self.cs, self.rows["margin"], self.scan, traj_offsets, think_end_pos,
                       self.tau, self.stats, self.rank, self.world_size, self.ws, self.seg, s,
                       per_trajectory=self.per_traj, exchange=self.exchange)
        return self.stats

    def capture(self, logits, tokens, traj_offsets=None, think_end_pos=None, host_stats=None,
                vocab=None):
        """A CUDA graph of one device-side pass (+ the stats table copied to the
        pinned ``host_stats`` when given).  ``graph.replay()`` re-runs it on the
        same buffers; the inputs may be refilled in place between replays."""
        import torch
        self.run(logits, tokens, traj_offsets, think_end_pos, vocab=vocab)   # warm-up
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(device=self.device)
        with torch.cuda.stream(cap):
            with torch.cuda.graph(g, stream=cap):
                self.run(logits, tokens, traj_offsets, think_end_pos, stream=cap, vocab=vocab)
                if host_stats is not None:
                    host_stats.copy_(self.stats, non_blocking=True)
        torch.cuda.synchronize(self.device)
        return g

    def n_launches(self) -> int:
        """Kernels launched by one run(): stats_init 1 + K1 1 + K2 1 + K3 1."""
        return 4
