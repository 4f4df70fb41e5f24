"""K2 relay_cue_scan alone (serialised, device-timed) at configs[1] (32,768
tokens, 8 cues / 12 patterns) and configs[4]'s per-rank stream (8 x 16,384 and
the 1M-token 64 x 16,384 corpus, 32 patterns of length 1-6), both modes.
    python tools/k2_time.py"""
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
    tok = torch.as_tensor(ts.tokens, device=dev)
    offs = torch.as_tensor(ts.traj_offsets, device=dev)
    for mode in (0, 1):
        cs = relay.CueSet.from_synth(h, mode=mode) if mode else relay.CueSet.from_synth(h)
        n = ts.tokens.shape[0]
        cap = n * (nc if mode else 1)
        ws = relay.workspace(n, cap, 0, dev)
        out = relay.cue_scan(cs, tok, offs, cap, ws=ws)
        for _ in range(5):
            relay.cue_scan(cs, tok, offs, cap, ws=ws, out=out)
        # device time: 20 launches captured in a CUDA graph (no host launch gaps)
        torch.cuda.synchronize()   # one workspace: no two launches may overlap across streams
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            relay.cue_scan(cs, tok, offs, cap, ws=ws, out=out, stream=s)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                for _ in range(20):
                    relay.cue_scan(cs, tok, offs, cap, ws=ws, out=out, stream=s)
        g.replay()
        torch.cuda.synchronize()
        ts_ = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts_.append(e0.elapsed_time(e1) * 1e3 / 20)
        print(f"{name:10s} n_tok {n:8d} mode {'ALL' if mode else 'LONGEST'}: K2 {statistics.median(ts_):7.2f} us "
              f"(min {min(ts_):.2f}), n_occ {int(out['n_occ'].item())}")
        cs.destroy()
