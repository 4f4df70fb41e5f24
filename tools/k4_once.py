"""A few eager K4 (relay_step_switch) launches on configs[2] inputs, for ncu:
    ncu --set full -k regex:rows_kernel --launch-skip 3 -c 1 python tools/k4_once.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2602_06454_b200 as relay  # noqa: E402
import synth  # noqa: E402

B, V = 256, 152064
dev = torch.device("cuda:0")
h = synth.make_cueset(V, 8, 12, max_len=3)
cs = relay.CueSet.from_synth(h)
bufs = [synth.make_logits(B, V, "bf16", seed=100 + i, device=dev) for i in range(4)]
state = torch.zeros(B, dtype=torch.uint8, device=dev)
hist = torch.full((B, 7), -1, dtype=torch.int32, device=dev)
small = torch.zeros(B, dtype=torch.int32, device=dev)
samp = torch.randint(3000, V, (B,), dtype=torch.int32, device=dev)
ws = relay.workspace(0, 0, B, dev)
out = relay.step_switch(cs, bufs[0], state, hist, small, samp, ws=ws)
for i in range(6):
    relay.step_switch(cs, bufs[i % 4], state, hist, small, samp, ws=ws, out=out)
torch.cuda.synchronize()
cs.destroy()
