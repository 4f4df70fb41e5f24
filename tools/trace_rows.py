"""Timeline of the row kernel (K4 decode step by default) from a traced build:
    python tools/trace_rows.py build     # librelay with -DRELAY_TRACE into build/trace/
    python tools/trace_rows.py run       # one graph-free step on cuda:0, per-CTA stamps (us)
Stamps: 0 entry, 1 first stage landed (consumer warp 0), 2.. consumer item ends,
10.. epilogue item ends, 15 consumer exit."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.environ.get("RELAY_TRACE_LIB", os.path.join(ROOT, "build", "trace", "librelay.so"))
def _builder():
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_relay_build", os.path.join(ROOT, "paper_2602_06454_b200", "_build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def build(*extra):
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    _builder().build_lib(OUT, defines=["RELAY_TRACE", *extra])


def run(mode="step"):
    import numpy as np
    import torch
    import paper_2602_06454_b200 as relay
    relay.LIB_PATH = OUT
    relay._lib = relay._load()
    import synth
    dev = torch.device("cuda:0")
    B = int(os.environ.get("TRACE_BATCH", "256" if mode == "step" else "444"))
    V = 152064
    h = synth.make_cueset(V, 8, 12, max_len=3)
    cs = relay.CueSet.from_synth(h)
    L = synth.make_logits(B, V, "bf16", device=dev)
    state = torch.zeros(B, dtype=torch.uint8, device=dev)
    hist = torch.full((B, 7), -1, dtype=torch.int32, device=dev)
    ws = relay.workspace(0, 0, B, dev)
    small = torch.zeros(B, dtype=torch.int32, device=dev)
    uni = torch.rand(B, device=dev)

    def sample_step():
        relay.step_sample(cs, L, uni, state, hist, small, temperature=0.6, top_k=20, top_p=0.95, ws=ws)
    for _ in range(3):
        if mode == "step":
            relay.step_switch(cs, L, state, hist, ws=ws)
        elif mode == "sample":
            sample_step()
        else:
            relay.margin_rows(L)
    torch.cuda.synchronize()
    n = 444
    S = 32
    lib0 = C.CDLL(OUT)
    zero = np.zeros((n, S), np.uint64)
    lib0.relay_debug_trace_reset.argtypes = [C.c_void_p, C.c_int]
    if mode == "step":
        assert lib0.relay_debug_trace_reset(zero.ctypes.data_as(C.c_void_p), n) == 0
        relay.step_switch(cs, L, state, hist, ws=ws)
    elif mode == "sample":
        assert lib0.relay_debug_trace_reset(zero.ctypes.data_as(C.c_void_p), n) == 0
        sample_step()
    else:
        assert lib0.relay_debug_trace_reset(zero.ctypes.data_as(C.c_void_p), n) == 0
        relay.margin_rows(L)
    torch.cuda.synchronize()
    buf = np.zeros((n, S), np.uint64)
    lib = C.CDLL(OUT)
    lib.relay_debug_trace_copy.argtypes = [C.c_void_p, C.c_int]
    assert lib.relay_debug_trace_copy(buf.ctypes.data_as(C.c_void_p), n) == 0
    print("CTAs with an entry stamp:", int((buf[:, 0] > 0).sum()), " RELAY_K4_MODE =",
          os.environ.get("RELAY_K4_MODE", "(default)"))
    t0 = int(buf[:, 0][buf[:, 0] > 0].min())
    rel = np.where(buf > 0, (buf.astype(np.int64) - t0) / 1e3, np.nan)
    np.set_printoptions(linewidth=250, precision=1, suppress=True)
    print("per CTA: entry, first TMA issued | stage 1..10 landed | item-1 fetched, rempty passed, "
          "probe barrier passed, first stage consumed | consumer item ends | epilogue item ends | exit "
          "(us from the first CTA entry)")
    for b in list(range(0, n, 37)) + [n - 1]:
        r = rel[b]
        print(f"{b:4d} {r[0]:5.1f} {r[15]:5.1f} |", r[1:11], "|", r[11:15], "|", r[16:20], "|",
              r[24:28], "|", f"{r[31]:5.1f}")
    st = rel[:, 1:11]
    gaps = np.diff(st, axis=1)
    print("stage-1 landed: min %.1f med %.1f max %.1f" % tuple(np.nanpercentile(st[:, 0], [0, 50, 100])))
    print("stage gap (us): p10 %.2f med %.2f p90 %.2f max %.2f" %
          tuple(np.nanpercentile(gaps, [10, 50, 90, 100])))
    print("consumer exit: min %.1f med %.1f max %.1f" % tuple(np.nanpercentile(rel[:, 31], [0, 50, 100])))
    print("max epilogue", np.nanmax(rel[:, 24:31]))
    lag = rel[:, 24:28] - rel[:, 16:20]  # epilogue item end - consumer item end
    if np.isfinite(lag).any():
        print("epilogue lag per item (us): p50 %.2f p90 %.2f max %.2f" %
              tuple(np.nanpercentile(lag, [50, 90, 100])))
        last_c = np.nanmax(rel[:, 16:24], axis=1)
        last_e = np.nanmax(rel[:, 24:31], axis=1)
        if mode == "step" and os.environ.get("RELAY_K4_MODE", "strided") == "strided":
            # item 0's epilogue: consumers' barrier passed (20), partials merged (21),
            # before finish (22), after finish + switch (24); from consumer warp 0's end (16)
            d = rel[:, [20, 21, 22, 24]] - rel[:, [16]]
            print("strided epilogue after consumer warp 0 (us) p50/p90: barrier %.2f/%.2f merged %.2f/%.2f "
                  "pre-finish %.2f/%.2f done %.2f/%.2f" % tuple(x for k in range(4)
                                                              for x in np.nanpercentile(d[:, k], [50, 90])))
        if mode == "step":
            sm = buf[:, 29].astype(np.int64) - 1
            end_c = rel[:, 31]
            from collections import defaultdict
            per = defaultdict(list)
            for b in range(n):
                if sm[b] >= 0 and np.isfinite(end_c[b]):
                    per[int(sm[b])].append(end_c[b])
            one = [v[0] for v in per.values() if len(v) == 1]
            two = [sorted(v) for v in per.values() if len(v) == 2]
            if one:
                print("SMs with one CTA: %d, consumer exit p50 %.1f max %.1f" % (len(one), np.median(one), max(one)))
            if two:
                t = np.array(two)
                print("SMs with two CTAs: %d, first exit p50 %.1f max %.1f, second exit p50 %.1f max %.1f" %
                      (len(two), np.median(t[:, 0]), t[:, 0].max(), np.median(t[:, 1]), t[:, 1].max()))
        if mode == "sample":
            d = rel[:, [1, 11, 14, 16, 20, 21, 22, 23, 24]]
            names = ["stage1", "bound", "stage1 done", "cons end", "epi barrier", "merged", "pre-finish",
                     "drawn", "epi end"]
            print("sample-mode stamps p50 (us):", ", ".join("%s %.2f" % (nm, np.nanmedian(d[:, k]))
                                                          for k, nm in enumerate(names)))
        print("last consumer item end: p50 %.1f p90 %.1f max %.1f | last epilogue end: p50 %.1f p90 %.1f max %.1f"
              % (*np.nanpercentile(last_c, [50, 90, 100]), *np.nanpercentile(last_e, [50, 90, 100])))


if __name__ == "__main__":
    build(*sys.argv[2:]) if sys.argv[1] == "build" else run(*(sys.argv[2:3] or ["step"]))
