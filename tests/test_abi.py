"""No-GPU tests of the boundary: librelay.so loads, exports every symbol that
include/relay.h declares, rejects bad arguments on the host before any device
work, and finalizes an integer stats table (H7, host code) to the values of
the hand-traced golden fixture."""
import ctypes as C
import json
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def relay():
    import __graft_entry__
    __graft_entry__._build_lib()
    import paper_2602_06454_b200 as r
    return r


def test_exports_match_header(relay):
    hdr = open(os.path.join(ROOT, "include", "relay.h")).read()
    declared = set(re.findall(r"\b(relay_[a-z0-9_]+)\s*\(", hdr))
    lib = C.CDLL(relay.LIB_PATH)
    missing = [n for n in sorted(declared) if not hasattr(lib, n)]
    assert not missing, missing
    assert declared == set(relay.EXPORTS)
    assert relay.version() == 1


def test_library_is_sm100a_only(relay):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", relay.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out and "sm_90" not in out


def test_host_validation_without_device(relay):
    lib = relay._lib
    P = C.c_void_p
    ptr = P(16)        # never dereferenced: validation fails first
    # vocab < 2
    assert lib.relay_margin_rows(ptr, 0, 4, 1, 1, 1.0, ptr, None, None, None, None, None) == 1
    assert b"vocab" in lib.relay_last_error()
    # row_stride < vocab
    assert lib.relay_margin_rows(ptr, 0, 4, 8, 7, 1.0, ptr, None, None, None, None, None) == 1
    # bad dtype / temperature / n_rows
    assert lib.relay_margin_rows(ptr, 9, 4, 8, 8, 1.0, ptr, None, None, None, None, None) == 1
    assert lib.relay_margin_rows(ptr, 0, 4, 8, 8, 0.0, ptr, None, None, None, None, None) == 1
    assert lib.relay_margin_rows(ptr, 0, -1, 8, 8, 1.0, ptr, None, None, None, None, None) == 1
    # n_rows == 0 is a no-op
    assert lib.relay_margin_rows(None, 0, 0, 8, 8, 1.0, None, None, None, None, None, None) == 0
    # cue set validation happens before any allocation
    out = P()
    term = np.zeros(16, np.uint8)
    t = lambda a: np.ascontiguousarray(a, np.int32).ctypes.data_as(P)  # noqa: E731
    keep = [np.array([1, 2, 1, 2], np.int32), np.array([0, 2, 4], np.int32), np.array([0, 0], np.int32)]
    assert lib.relay_cueset_create(keep[0].ctypes.data_as(P), keep[1].ctypes.data_as(P), 2,
                                   keep[2].ctypes.data_as(P), 1, term.ctypes.data_as(P), 16, -1, 0,
                                   C.byref(out)) == 1
    assert b"identical" in lib.relay_last_error()
    bad = [np.array([1, 99], np.int32), np.array([0, 2], np.int32), np.array([0], np.int32)]
    assert lib.relay_cueset_create(bad[0].ctypes.data_as(P), bad[1].ctypes.data_as(P), 1,
                                   bad[2].ctypes.data_as(P), 1, term.ctypes.data_as(P), 16, -1, 0,
                                   C.byref(out)) == 1
    assert lib.relay_cueset_create(bad[0].ctypes.data_as(P), bad[1].ctypes.data_as(P), 1,
                                   bad[2].ctypes.data_as(P), 1, term.ctypes.data_as(P), 16, -1, 2,
                                   C.byref(out)) == 1
    # workspace checks
    assert lib.relay_cue_scan(None, ptr, 10, None, 1, ptr, ptr, ptr, 4, ptr, ptr, 0, None) == 1
    assert lib.relay_stats_init(ptr, 3, 2, 2, None) == 1            # rank >= world
    assert lib.relay_stats_finalize(None, 3, 1, 3, 0, None) == 1
    del t


def test_workspace_registry_without_device(relay):
    """Workspace calls are checked against the registry before any launch:
    an unregistered workspace, NULL, or bad capacities fail on the host."""
    lib = relay._lib
    P = C.c_void_p
    ptr = P(4096)
    cs = P(64)      # never dereferenced: the workspace check fails first
    # cue_scan with a workspace that relay_workspace_init never saw
    n_occ = np.zeros(1, np.int64)
    assert lib.relay_cue_scan(cs, ptr, 10, None, 1, ptr, ptr, ptr, 4, n_occ.ctypes.data_as(P), ptr,
                              1 << 20, None) == 7
    assert b"relay_workspace_init" in lib.relay_last_error()
    assert lib.relay_workspace_init(None, 16, 10, 10, 0, None) == 1
    assert lib.relay_workspace_init(ptr, 1 << 20, -1, 0, 0, None) == 1
    need = relay.workspace_bytes(100000, 1000, 64)
    assert lib.relay_workspace_init(ptr, need - 1, 100000, 1000, 64, None) == 7
    assert lib.relay_workspace_release(ptr) == 0
    # one workspace serves both regions: the size is the sum
    step64 = relay.workspace_bytes(0, 0, 64) - relay.workspace_bytes(0, 0, 0)
    assert step64 > 0 and need == relay.workspace_bytes(100000, 1000, 0) + step64


def test_nccl_version_is_torchs(relay):
    """relay_nccl_version reports the NCCL librelay resolves at run time; the
    binding hands torch's communicator to it only when it is torch's library
    (dist.torch_comm_compatible)."""
    import torch
    try:
        code, path = relay.nccl_version()
    except relay.RelayError:
        pytest.skip("no libnccl.so.2 resolvable here")
    tv = torch.cuda.nccl.version()
    tv = tv if isinstance(tv, int) else tv[0] * 10000 + tv[1] * 100 + (tv[2] if len(tv) > 2 else 0)
    assert code > 20000 and path.endswith(".so.2") or "libnccl" in path
    from paper_2602_06454_b200 import dist as rdist
    ok, why = rdist.torch_comm_compatible()
    assert ok == (code == tv and path and __import__("os").path.realpath(path) in rdist._loaded_nccl_files()
                  and len(rdist._loaded_nccl_files()) == 1), why


def test_workspace_sizes_are_monotone(relay):
    a = relay.workspace_bytes(1000, 10, 0)
    b = relay.workspace_bytes(100000, 1000, 0)
    c = relay.workspace_bytes(0, 0, 256)
    assert 0 < a < b and c > 0
    assert relay.stats_words(8, 1) == 9 * 9 and relay.stats_words(8, 4) == 9 * 12


def _q20(x: float) -> int:
    # round-half-even of the fp32 value times 2^20 (exact in Python)
    return int(round(float(np.float32(x)) * (1 << 20)))


def test_finalize_golden_trace(relay):
    """Build the uint64 table by integer arithmetic from the golden fixture's
    windows (hand-traced ends), finalize on the host, compare to the golden
    per-cue and global numbers (within the Q20 error, 1e-5)."""
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "trace_fixture.json")))
    m = g["margins"]
    nf = 9
    tab = np.zeros((3, nf), np.uint64)
    tab[:, 8] = 0x7F800000
    pat_cue = g["pat_cue"]
    for k, o in enumerate(g["occurrences"]):
        c = pat_cue[o["pat"]]
        w = [_q20(x) for x in m[o["s"]:o["e"] + 1]]
        ln = len(w)
        sq = sum(w)
        mq = (2 * sq + ln) // (2 * ln)
        prev = [p for p in g["occurrences"][:k] if p["s"] < o["s"]]
        trig = 1 if not prev or prev[-1]["e"] != o["e"] else 0
        row = tab[c]
        row[0] += 1; row[1] += mq; row[2] += mq * mq; row[3] += sq; row[4] += ln
        row[5] += sum(1 for x in m[o["s"]:o["e"] + 1] if np.float32(x) < np.float32(g["tau"]))
        row[6] += trig
        row[8] = min(int(row[8]), int(np.float32(o["min"]).view(np.uint32)))
    q = [_q20(x) for x in m]
    gr = tab[2]
    gr[0] = len(q); gr[1] = sum(q); gr[2] = sum(x * x for x in q); gr[3] = sum(q); gr[4] = len(q)
    gr[5] = sum(1 for x in m if np.float32(x) < np.float32(g["tau"]))
    gr[8] = int(np.float32(min(m)).view(np.uint32))
    fin = relay.stats_finalize(tab.reshape(-1).view(np.int64), 2, 1, min_count=1)
    for c, e in enumerate(g["cues"]):
        assert fin[c]["n"] == e["n"] and fin[c]["n_triggers"] == e["n_triggers"]
        for f in ("mean", "std", "se", "token_mean", "min", "low_frac"):
            assert abs(fin[c][f] - e[f]) < 1e-5, (c, f)
    for f in ("mean", "std", "se", "min", "low_frac"):
        assert abs(fin[2][f] - g["global"][f]) < 1e-5, f
    assert [f["selected"] for f in fin[:2]] == g["selected_rule0_min_count_1"]
    fin3 = relay.stats_finalize(tab.reshape(-1).view(np.int64), 2, 1, min_count=5)
    assert [f["selected"] for f in fin3[:2]] == [0, 0]


def test_finalize_rules_and_small_n(relay):
    nf = 9
    tab = np.zeros((2, nf), np.uint64)
    Q = 1 << 20
    # global: margins {0.25, 0.75} -> mu .5, sigma .25, SE .25/sqrt2
    tab[1, 0] = 2; tab[1, 1] = Q // 4 + 3 * Q // 4; tab[1, 2] = (Q // 4) ** 2 + (3 * Q // 4) ** 2
    tab[1, 4] = 2
    # cue: one window of mean 0.6
    tab[0, 0] = 1; tab[0, 1] = int(0.6 * Q); tab[0, 2] = int(0.6 * Q) ** 2; tab[0, 4] = 1
    f0 = relay.stats_finalize(tab.reshape(-1).view(np.int64), 1, 1, 1, rule=0)
    f1 = relay.stats_finalize(tab.reshape(-1).view(np.int64), 1, 1, 1, rule=1)
    f2 = relay.stats_finalize(tab.reshape(-1).view(np.int64), 1, 1, 1, rule=2)
    assert abs(f0[1]["se"] - 0.25 / np.sqrt(2)) < 1e-12
    assert (f0[0]["selected"], f1[0]["selected"], f2[0]["selected"]) == (0, 1, 1)
    tab[1, 0] = 1
    f = relay.stats_finalize(tab.reshape(-1).view(np.int64), 1, 1, 1, rule=2)
    assert np.isnan(f[1]["se"]) and f[0]["selected"] == 0


def test_plain_c_consumer(relay, tmp_path):
    """include/relay.h is a self-contained C header: a plain C program links
    librelay.so and runs host-side calls without torch or CUDA headers."""
    import subprocess
    exe = str(tmp_path / "abi_host")
    lib_dir = os.path.dirname(relay.LIB_PATH)
    subprocess.check_call(["gcc", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "c", "abi_host.c"), "-o", exe,
                           "-L", lib_dir, "-Wl,-rpath," + lib_dir, "-l:librelay.so", "-lm"])
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0 and "c abi ok" in r.stdout, (r.returncode, r.stdout, r.stderr)


def test_stats_merge_host(relay):
    """relay_stats_merge (host): fields 0-7 add, the rank's own min slot takes
    the minimum (every slot with rank -1, after the all-reduce), the mask
    picks tables, and summing the per-rank merges equals merging the summed
    tables (each rank's min slot is +inf-initialised only on that rank, 0
    elsewhere), also when a rank merges nothing (an empty merge
    must leave the other ranks' slots 0, or the SUM corrupts their minima)."""
    rng = np.random.default_rng(7)
    n_cues, world, n_tab = 5, 2, 6
    nf = 8 + world
    words = relay.stats_words(n_cues, world)
    assert words == (n_cues + 1) * nf
    per_rank = []
    for r in range(world):
        t = rng.integers(0, 1 << 40, size=(n_tab, n_cues + 1, nf), dtype=np.uint64)
        mins = np.float32(rng.random((n_tab, n_cues + 1))).view(np.uint32).astype(np.uint64)
        mins[rng.random(mins.shape) < 0.3] = 0x7F800000          # empty rows keep +inf
        t[:, :, 8:] = 0
        t[:, :, 8 + r] = mins
        per_rank.append(t)
    mask = np.array([1, 0, 1, 1, 0, 1], bool)
    for r, t in enumerate(per_rank):
        got = relay.stats_merge(t, n_cues, world, mask, rank=r).reshape(n_cues + 1, nf)
        sel = t[mask]
        np.testing.assert_array_equal(got[:, :8], sel[:, :, :8].sum(axis=0))
        np.testing.assert_array_equal(got[:, 8 + r], sel[:, :, 8 + r].min(axis=0))
        assert not np.delete(got[:, 8:], r, axis=1).any()
    # merge(sum over ranks) == sum over ranks(merge), for any selection
    summed = per_rank[0] + per_rank[1]
    for m in (mask, np.zeros(n_tab, bool), np.ones(n_tab, bool)):
        a = relay.stats_merge(summed, n_cues, world, m, rank=-1)
        b = relay.stats_merge(per_rank[0], n_cues, world, m, rank=0) + \
            relay.stats_merge(per_rank[1], n_cues, world, m, rank=1)
        np.testing.assert_array_equal(a, b)
    # empty selection on one rank: exactly an initialised table of that rank
    e = relay.stats_merge(per_rank[1], n_cues, world, np.zeros(n_tab, bool), rank=1).reshape(n_cues + 1, nf)
    assert not e[:, :9].any() and (e[:, 9] == 0x7F800000).all()
    with pytest.raises(relay.RelayError):
        relay.stats_merge(per_rank[0].reshape(-1)[:-1], n_cues, world)
    with pytest.raises(relay.RelayError):
        relay.stats_merge(per_rank[0], n_cues, world, rank=world)
    lib = C.CDLL(relay.LIB_PATH)
    assert lib.relay_stats_merge(None, 1, None, 3, 0, 1, None) == 1


def test_nccl_entry_points_host(relay):
    """H6 boundary without a GPU: NCCL resolves at run time (a unique id is
    host-only), and bad arguments fail before any NCCL call."""
    uid = relay.nccl_unique_id()
    assert len(uid) == 128 and any(uid)
    lib = C.CDLL(relay.LIB_PATH)
    lib.relay_stats_allreduce.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                          C.c_void_p]
    assert lib.relay_stats_allreduce(None, None, 1, 3, 1, None) == 1
    assert lib.relay_stats_allreduce(C.c_void_p(8), C.c_void_p(8), 0, 3, 1, None) == 1
    assert lib.relay_stats_allreduce(C.c_void_p(8), C.c_void_p(8), 1, 0, 1, None) == 1
    lib.relay_nccl_comm_init.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]
    out = C.c_void_p()
    buf = (C.c_uint8 * 128)()
    assert lib.relay_nccl_comm_init(C.cast(buf, C.c_void_p), 2, 2, C.byref(out)) == 1
    assert lib.relay_nccl_comm_destroy(None) == 0
    assert relay.version() >= 1 and lib.relay_status_string(3)


def test_cueset_create_ex_validation(relay):
    """N4 argument checks happen on the host before any device work."""
    V = 32
    term = np.zeros(V, np.uint8)
    classes = np.zeros((2, V), np.uint8)
    ok = dict(pat_tokens=[1, -1], pat_offsets=[0, 2], pat_cue=[0], n_cues=1, terminator=term, vocab=V)
    with pytest.raises(relay.RelayError):          # class element -3 with only 2 classes
        relay.CueSet([1, -3], [0, 2], [0], 1, term, V, classes=classes)
    with pytest.raises(relay.RelayError):          # class element without classes
        relay.CueSet(**ok)
    with pytest.raises(relay.RelayError):          # decimal rule naming a missing class
        relay.CueSet(**ok, classes=classes, decimal_rule=(0, 1, 2))
    with pytest.raises(relay.RelayError):          # too many classes
        relay.CueSet(**ok, classes=np.zeros((9, V), np.uint8))
    lib = C.CDLL(relay.LIB_PATH)
    out = C.c_void_p()
    P = C.c_void_p
    keep = [np.array([1], np.int32), np.array([0, 1], np.int32), np.array([0], np.int32)]
    lib.relay_cueset_create_ex.argtypes = [P, P, C.c_int32, P, C.c_int32, P, C.c_int64, C.c_int32,
                                           C.c_uint32, P, C.c_int32, P, P]
    assert lib.relay_cueset_create_ex(keep[0].ctypes.data_as(P), keep[1].ctypes.data_as(P), 1,
                                      keep[2].ctypes.data_as(P), 1, term.ctypes.data_as(P), V, -1,
                                      0, None, 1, None, C.byref(out)) == 1   # classes NULL, n=1


def test_tp_exchange_validation_host(relay):
    """N1 fused exchange: bad arguments fail on the host before any CUDA call."""
    lib = C.CDLL(relay.LIB_PATH)
    P = C.c_void_p
    lib.relay_tp_exchange_create.argtypes = [C.c_int32, C.c_int32, C.c_int64, P, P]
    lib.relay_tp_exchange_connect.argtypes = [P, P]
    lib.relay_tp_exchange_destroy.argtypes = [P]
    lib.relay_margin_rows_tp.argtypes = [P, P, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                         C.c_float, P, P, P, P, P, P]
    h = (C.c_uint8 * relay.IPC_HANDLE_BYTES)()
    out = C.c_void_p()
    assert lib.relay_tp_exchange_create(0, 9, 16, h, C.byref(out)) == 1     # world > 8
    assert lib.relay_tp_exchange_create(2, 2, 16, h, C.byref(out)) == 1     # rank >= world
    assert lib.relay_tp_exchange_create(0, 2, 0, h, C.byref(out)) == 1      # rows_cap < 1
    assert lib.relay_tp_exchange_create(0, 2, 16, None, C.byref(out)) == 1  # no handle buffer
    assert lib.relay_tp_exchange_connect(None, h) == 1
    assert lib.relay_tp_exchange_destroy(None) == 0
    assert lib.relay_margin_rows_tp(None, None, 0, 4, 8, 8, 0, 1.0, None, None, None, None, None,
                                    None) == 1


def test_read_probe_validation_host(relay):
    """The read-probe measurement utility rejects bad arguments on the host."""
    lib = C.CDLL(relay.LIB_PATH)
    lib.relay_read_probe.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
    assert lib.relay_read_probe(None, 64, C.c_void_p(16), None) == 1
    assert lib.relay_read_probe(C.c_void_p(16), 15, C.c_void_p(16), None) == 1
    assert lib.relay_read_probe(C.c_void_p(24), 64, C.c_void_p(16), None) == 1   # misaligned
    assert lib.relay_read_probe_words() > 0
