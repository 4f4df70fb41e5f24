"""K3 relay_segment_reduce alone (serialised, device-timed) at configs[1]
(32,768 tokens, 8 cues / 12 patterns) and configs[4]'s per-rank / corpus
streams:  python tools/k3_time.py"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2602_06454_b200 as relay  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
for name, (nt, L, V, nc, npat, ml) in {"c2": (1, 32768, 151936, 8, 12, 3), "c5_rank": (8, 16384, 151936, 32, 32, 6),
                                       "c5_corpus": (64, 16384, 151936, 32, 32, 6)}.items():
    h = synth.make_cueset(V, nc, npat, max_len=ml, min_len=1)
    ts = synth.make_tokens(nt, L, h)
    n = ts.tokens.shape[0]
    cs = relay.CueSet.from_synth(h)
    tok = torch.as_tensor(ts.tokens, device=dev)
    offs = torch.as_tensor(ts.traj_offsets, device=dev)
    m = torch.as_tensor(synth.make_margins(n, seed=5), device=dev)
    ws = relay.workspace(n, n, 0, dev)
    scan = relay.cue_scan(cs, tok, offs, n, ws=ws)
    out = relay.segment_reduce(cs, m, scan, offs, ws=ws)
    torch.cuda.synchronize()
    ts_ = []
    for _ in range(30):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        relay.segment_reduce(cs, m, scan, offs, stats=out["stats"], ws=ws, out=out)
        e1.record()
        torch.cuda.synchronize()
        ts_.append(e0.elapsed_time(e1) * 1e3)
    print("%-10s n_tok %8d: K3 %7.2f us (min %.2f), n_occ %d" % (name, n, statistics.median(ts_), min(ts_),
                                                            int(scan["n_occ"].item())))
    cs.destroy()
