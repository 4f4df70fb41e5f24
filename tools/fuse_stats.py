"""Fused top-k draw statistics (traced build, build/trace/librelay.so): rows
K4 drew itself vs rows handed to K5, mean candidates per row, on configs[2]
rows.   python tools/fuse_stats.py"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.environ.get("RELAY_TRACE_LIB", os.path.join(ROOT, "build", "trace", "librelay.so"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_06454_b200 as relay  # noqa: E402

relay.LIB_PATH = OUT
relay._lib = relay._load()
import synth  # noqa: E402

B, V = 256, 152064
dev = torch.device("cuda:0")
cs = relay.CueSet.from_synth(synth.make_cueset(V, 8, 12, max_len=3))
L = synth.make_logits(B, V, "bf16", seed=100, device=dev)
state = torch.zeros(B, dtype=torch.uint8, device=dev)
hist = torch.full((B, 7), -1, dtype=torch.int32, device=dev)
small = torch.zeros(B, dtype=torch.int32, device=dev)
uni = torch.rand(B, device=dev)
ws = relay.workspace(0, 0, B, dev)
lib = C.CDLL(OUT)
buf = np.zeros(4, np.uint64)
lib.relay_debug_fuse_stats(buf.ctypes.data_as(C.c_void_p), 1)
for top_k in (20, 64):
    relay.step_sample(cs, L, uni, state, hist, small, temperature=0.6, top_k=top_k, top_p=0.95, ws=ws)
    torch.cuda.synchronize()
    lib.relay_debug_fuse_stats(buf.ctypes.data_as(C.c_void_p), 1)
    print("top_k %d: drawn in K4 %d, to K5 %d, candidates per row %.1f" %
          (top_k, buf[0], buf[1], buf[2] / max(1, buf[0] + buf[1])))
