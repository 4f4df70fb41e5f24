"""K3 (relay_segment_reduce) timeline from a traced build (tools/trace_rows.py
build): per-tile stamps by thread 0: entry, positions loaded, moments added,
carry known, occurrences gathered, exit.   python tools/k3_trace.py [n_tok]"""
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
    h = synth.make_cueset(151936, 8, 12, max_len=3)
    cs = relay.CueSet.from_synth(h)
    ts = synth.make_tokens(1, n_tok, h)
    dev = torch.device("cuda:0")
    tok = torch.as_tensor(ts.tokens, device=dev)
    offs = torch.as_tensor(ts.traj_offsets, device=dev)
    m = torch.as_tensor(synth.make_margins(n_tok, seed=5), device=dev)
    ws = relay.workspace(n_tok, n_tok, 0, dev)
    scan = relay.cue_scan(cs, tok, offs, n_tok, ws=ws)
    out = relay.segment_reduce(cs, m, scan, offs, ws=ws)
    for _ in range(3):
        relay.segment_reduce(cs, m, scan, offs, stats=out["stats"], ws=ws, out=out)
    torch.cuda.synchronize()
    n = (n_tok + 2047) // 2048
    buf = np.zeros((n, 8), np.uint64)
    lib = C.CDLL(OUT)
    lib.relay_debug_trace3_copy.argtypes = [C.c_void_p, C.c_int]
    assert lib.relay_debug_trace3_copy(buf.ctypes.data_as(C.c_void_p), n) == 0
    t0 = int(buf[:, 0].min())
    rel = (buf[:, :6].astype(np.int64) - t0) / 1e3
    names = ["entry", "positions", "moments", "carry", "gathered", "exit"]
    for k in range(6):
        print("%-10s p0 %6.2f p50 %6.2f p100 %6.2f us" % (names[k], *np.percentile(rel[:, k], [0, 50, 100])))


if __name__ == "__main__":
    main()
