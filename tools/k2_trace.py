"""K2 (relay_cue_scan) timeline from a traced build (tools/trace_rows.py build
writes build/trace/librelay.so with -DRELAY_TRACE): per-tile stamps, thread 0:
0 entry, 1 patterns staged, 2 phase 1 (match + counts) done, 3 look-back done,
4 writes issued.  python tools/k2_trace.py [n_tok]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.environ.get("RELAY_TRACE_LIB", os.path.join(ROOT, "build", "trace", "librelay.so"))


def main():
    import numpy as np
    import torch
    import paper_2602_06454_b200 as relay
    relay.LIB_PATH = OUT
    relay._lib = relay._load()
    import synth
    n_tok = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    V = 151936
    h = synth.make_cueset(V, 8, 12, max_len=3)
    cs = relay.CueSet.from_synth(h)
    ts = synth.make_tokens(1, n_tok, h)
    dev = torch.device("cuda:0")
    tok = torch.as_tensor(ts.tokens, device=dev)
    offs = torch.as_tensor(ts.traj_offsets, device=dev)
    for _ in range(3):
        relay.cue_scan(cs, tok, offs)
    torch.cuda.synchronize()
    relay.cue_scan(cs, tok, offs)
    torch.cuda.synchronize()
    n = (n_tok + 255) // 256
    buf = np.zeros((n, 16), np.uint64)
    lib = C.CDLL(OUT)
    lib.relay_debug_trace2_copy.argtypes = [C.c_void_p, C.c_int]
    assert lib.relay_debug_trace2_copy(buf.ctypes.data_as(C.c_void_p), n) == 0
    t0 = int(buf[:, 0].min())
    rel = (buf[:, :5].astype(np.int64) - t0) / 1e3
    names = ["entry", "patterns staged", "phase 1 done", "look-back done", "writes issued"]
    for k in range(5):
        print("%-16s p0 %6.2f p50 %6.2f p100 %6.2f us" % (names[k], *np.percentile(rel[:, k], [0, 50, 100])))
    has = buf[:, 5] > 0
    if has.any():
        r5 = (buf[has, 5].astype(np.int64) - t0) / 1e3
        r6 = (buf[has, 6].astype(np.int64) - t0) / 1e3
        print("first window loaded (after first use) p50 %.2f | window complete p50 %.2f max %.2f | spins p50 %d max %d"
              % (np.median(r5), np.median(r6), r6.max(), np.median(buf[has, 7]), buf[has, 7].max()))
    if (buf[:, 10] > 0).any():
        ph = [(buf[:, k].astype(np.int64) - t0) / 1e3 for k in (10, 11, 12)]
        print("warp 0 phase 1: terms done p50 %.2f | ballot words p50 %.2f | patterns p50 %.2f us"
              % tuple(np.median(x) for x in ph))
    pub = (buf[1:, 8].astype(np.int64) - t0) / 1e3
    print("agg published p50 %.2f max %.2f (tile %d)" % (np.median(pub), pub.max(), 1 + int(np.argmax(pub))))
    last_pending = buf[:, 9].astype(np.int64) - 1
    vals, cnts = np.unique(last_pending[last_pending >= 0], return_counts=True)
    print("last pending predecessor seen (tile: count):", dict(zip(vals.tolist()[:10], cnts.tolist()[:10])))
    d = np.diff(rel, axis=1)
    for k in range(4):
        print("%-16s -> %-16s p50 %5.2f max %5.2f us" % (names[k], names[k + 1], np.median(d[:, k]), d[:, k].max()))


if __name__ == "__main__":
    main()
