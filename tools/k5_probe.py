"""Per-buffer timing of relay_step_sample on configs[2] inputs, with and without
the synthetic edge rows, and how many rows leave the top-64 fast path of the
no-top-k (nucleus) mode (tuning only).

    python tools/k5_probe.py [--top-k K] [--top-p P]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2602_06454_b200 as relay  # noqa: E402
import synth  # noqa: E402

if os.environ.get("RELAY_LIB"):  # A/B runs against another build of the library
    relay.LIB_PATH = os.environ["RELAY_LIB"]
    relay._lib = relay._load()

ap = argparse.ArgumentParser()
ap.add_argument("--top-k", type=int, default=0)
ap.add_argument("--top-p", type=float, default=0.95)
ap.add_argument("--temperature", type=float, default=0.6)
ap.add_argument("--n-bufs", type=int, default=7)
args = ap.parse_args()

B, V = 256, 152064
dev = torch.device("cuda:0")
h = synth.make_cueset(V, 8, 12, max_len=3)
cs = relay.CueSet.from_synth(h)
state = torch.zeros(B, dtype=torch.uint8, device=dev)
hist = torch.full((B, 7), -1, dtype=torch.int32, device=dev)
small = torch.zeros(B, dtype=torch.int32, device=dev)
uni = torch.rand(B, device=dev, generator=torch.Generator(device=dev).manual_seed(5))
ws = relay.workspace(0, 0, B, dev)


def run(x, out=None):
    return relay.step_sample(cs, x, uni, state, hist, small, temperature=args.temperature,
                             top_k=args.top_k, top_p=args.top_p, ws=ws, out=out)


for edge in (False, True):
    for i in range(args.n_bufs):
        x = synth.make_logits(B, V, "bf16", seed=100 + i, device=dev, edge_rows=edge)
        # rows whose top-64 hold < top_p of the mass at the sampling temperature
        z = x.float()
        w = torch.exp((z - z.amax(dim=1, keepdim=True)) / args.temperature)
        top = torch.topk(w, 64, dim=1).values.sum(dim=1)
        slow = int((top < args.top_p * w.sum(dim=1)).sum())
        const = int((z.amin(dim=1) == z.amax(dim=1)).sum())
        out = run(x)
        torch.cuda.synchronize()
        for _ in range(3):
            run(x, out)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            run(x, out)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 100
        print(f"edge={int(edge)} buf={i} us/step={us:9.1f} slow_rows={slow} const_rows={const}", flush=True)

# isolate one pathological row in an otherwise plain batch
if True:
    base = synth.make_logits(B, V, "bf16", seed=100, device=dev, edge_rows=False)
    cases = {"plain": lambda x: None,
             "const": lambda x: x[0].fill_(1.25),
             "const_neg": lambda x: x[0].fill_(-3.0),
             "sparse20": lambda x: (x[0].fill_(float("-inf")), x[0, :20].normal_()),
             "flat": lambda x: x[0].normal_(0, 0.05)}
    for name, mod in cases.items():
        x = base.clone()
        mod(x)
        out = run(x)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            run(x, out)
        e1.record()
        torch.cuda.synchronize()
        print(f"row0={name:10s} us/step={e0.elapsed_time(e1) * 100:9.1f}", flush=True)
cs.destroy()
