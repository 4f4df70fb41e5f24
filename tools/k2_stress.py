"""K2 stress: many back-to-back relay_cue_scan launches on a 1M-token stream
(2,048 tiles > resident CTAs), eager and in a CUDA graph, checking n_occ."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2602_06454_b200 as relay  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
nt = int(sys.argv[1]) if len(sys.argv) > 1 else 64
h = synth.make_cueset(151936, 32, 32, max_len=6, min_len=1)
ts = synth.make_tokens(nt, 16384, h)
tok = torch.as_tensor(ts.tokens, device=dev)
offs = torch.as_tensor(ts.traj_offsets, device=dev)
cs = relay.CueSet.from_synth(h)
n = ts.tokens.shape[0]
ws = relay.workspace(n, n, 0, dev)
out = relay.cue_scan(cs, tok, offs, n, ws=ws)
torch.cuda.synchronize()
ref = int(out["n_occ"].item())
print("first", ref, flush=True)
for i in range(50):
    relay.cue_scan(cs, tok, offs, n, ws=ws, out=out)
t0 = time.time()
torch.cuda.synchronize()
print("eager x50 ok", int(out["n_occ"].item()) == ref, time.time() - t0, flush=True)
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    relay.cue_scan(cs, tok, offs, n, ws=ws, out=out, stream=s)
    torch.cuda.synchronize()
    print("side stream ok", flush=True)
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            relay.cue_scan(cs, tok, offs, n, ws=ws, out=out, stream=s)
print("captured", flush=True)
g.replay()
torch.cuda.synchronize()
print("graph ok", int(out["n_occ"].item()) == ref, flush=True)
