"""A few eager relay_step_sample launches on configs[2] inputs (for ncu):
    ncu --set full -k regex:sample_switch --launch-skip 3 -c 1 python tools/k5_once.py [--edge] [--no-top-k]
(--edge: the synthetic edge rows, incl. constant rows; --no-top-k: the
R1-Distill setting, K5 + the nucleus kernel K6)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2602_06454_b200 as relay  # noqa: E402
import synth  # noqa: E402

B, V = int(os.environ.get("K5_BATCH", "256")), 152064
dev = torch.device("cuda:0")
h = synth.make_cueset(V, 8, 12, max_len=3)
cs = relay.CueSet.from_synth(h)
edge = "--edge" in sys.argv
bufs = [synth.make_logits(B, V, "bf16", seed=100 + i, device=dev, edge_rows=edge) for i in range(4)]
state = torch.zeros(B, dtype=torch.uint8, device=dev)
hist = torch.full((B, 7), -1, dtype=torch.int32, device=dev)
small = torch.zeros(B, dtype=torch.int32, device=dev)
uni = torch.rand(B, device=dev)
ws = relay.workspace(0, 0, B, dev)
top_k = 0 if "--no-top-k" in sys.argv else 20
out = relay.step_sample(cs, bufs[0], uni, state, hist, small, top_k=top_k, ws=ws)
for i in range(6):
    relay.step_sample(cs, bufs[i % 4], uni, state, hist, small, top_k=top_k, ws=ws, out=out)
torch.cuda.synchronize()
cs.destroy()
