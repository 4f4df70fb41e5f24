"""Randomised parity sweep of relay_step_sample against the oracle sampler
(evidence for the sampler's exact paths; tests/ holds the fixed cases):
random batch / vocab / dtype / temperature / top-k / top-p and row types
(normal, flat, constant, tied blocks, sparse -inf, small/large offsets).
    python tools/sample_fuzz.py [n_cases] [seed]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2602_06454_b200 as relay  # noqa: E402
import synth  # noqa: E402

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 30
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
dev = torch.device("cuda:0")
bad_total = 0
for case in range(n_cases):
    B = int(rng.choice([3, 17, 64, 150]))
    V = int(rng.choice([40, 1000, 5003, 32000, 152064]))
    dtype = str(rng.choice(["bf16", "bf16", "f16", "f32"]))
    T = float(rng.choice([0.3, 0.6, 1.0, 1.7]))
    k = int(rng.choice([0, 0, 1, 5, 20, 64]))
    p = float(rng.choice([0.3, 0.9, 0.95, 1.0]))
    rows = rng.normal(0, rng.choice([0.05, 0.5, 2.5]), (B, V)) + rng.choice([-20.0, 0.0, 8.0, 30.0])
    for b in range(B):
        kind = rng.random()
        if kind < 0.05:
            rows[b] = rng.normal()                                   # constant
        elif kind < 0.10:
            blk = max(1, V // 50)
            rows[b] = np.repeat(rng.normal(0, 1, V // blk + 1), blk)[:V]  # tied blocks
        elif kind < 0.13:
            rows[b, rng.integers(1, V):] = -np.inf                  # sparse
    tdt = {"bf16": torch.bfloat16, "f16": torch.float16, "f32": torch.float32}[dtype]
    L = torch.as_tensor(rows.astype(np.float32), device=dev).to(tdt)
    host = synth.host_rows(L, dtype)
    u = rng.random(B).astype(np.float32)
    term = np.zeros(V, np.uint8)
    term[min(3, V - 1)] = 1
    h = synth.CueSet(np.array([1], np.int32), np.array([0, 1], np.int32), np.array([0], np.int32), 1, V, term,
                     V - 1, [(1,)])
    cs = relay.CueSet.from_synth(h)
    st = torch.zeros(B, dtype=torch.uint8, device=dev)
    hi = torch.full((B, 7), -1, dtype=torch.int32, device=dev)
    out = relay.step_sample(cs, L, torch.as_tensor(u, device=dev), st, hi, temperature=T, top_k=k, top_p=p)
    torch.cuda.synchronize()
    got = out["sampled"].cpu().numpy()
    want = oracle.sample_rows(host, u.astype(np.float64), dtype=dtype, vocab=V, temperature=T, top_k=k, top_p=p)
    bad = []
    for b in np.flatnonzero(want != got):
        alts = set()
        for du in (-1e-5, 1e-5):
            for dp in (0.0, -1e-5, 1e-5):
                uu = min(max(float(u[b]) + du, 0.0), 1 - 1e-12)
                pp = min(max(p + dp, 1e-9), 1.0)
                alts.add(int(oracle.sample_rows(host[b:b + 1], [uu], dtype=dtype, vocab=V, temperature=T,
                                                top_k=k, top_p=pp)[0]))
        if int(got[b]) not in alts:
            bad.append((int(b), int(got[b]), int(want[b])))
    bad_total += len(bad)
    print(f"case {case:3d} B={B:4d} V={V:6d} {dtype:4s} T={T} k={k:2d} p={p}: mismatches {len(bad)} {bad[:3]}",
          flush=True)
    cs.destroy()
print("TOTAL mismatches beyond CDF edges:", bad_total)
