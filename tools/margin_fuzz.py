"""Randomised parity sweep of relay_margin_rows (K1) and relay_step_switch's
margins (K4, every work split) against the oracle: random row counts, vocab
sizes, strides, misaligned bases, dtypes and edge rows (evidence; tests/
holds the fixed cases).   python tools/margin_fuzz.py [n_cases] [seed]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2602_06454_b200 as relay  # noqa: E402
import synth  # noqa: E402

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 3)
dev = torch.device("cuda:0")
fails = 0
for case in range(n_cases):
    n = int(rng.choice([1, 7, 150, 600, 2000]))
    V = int(rng.choice([2, 3, 17, 1000, 4099, 32000, 151936]))
    pad = int(rng.choice([0, 1, 5, 64]))
    off = int(rng.choice([0, 1, 3]))
    dtype = str(rng.choice(["bf16", "f16", "f32"]))
    tdt = {"bf16": torch.bfloat16, "f16": torch.float16, "f32": torch.float32}[dtype]
    rows = rng.normal(0, rng.choice([0.01, 1.0, 3.0]), (n, V)) * rng.choice([1, 1000])
    for b in range(n):
        r = rng.random()
        if r < 0.03: rows[b] = rng.normal()                         # constant
        elif r < 0.05: rows[b, rng.integers(0, V)] = np.nan
        elif r < 0.07: rows[b, :] = -np.inf; rows[b, rng.integers(0, V)] = 1.0
        elif r < 0.08: rows[b, :] = -np.inf
        elif r < 0.10: rows[b, rng.integers(0, V)] = np.inf
        elif r < 0.13: rows[b] = np.sort(rows[b])                   # ascending: the slow top-2 path
    big = torch.full((n * (V + pad) + off + 8,), float("nan"), dtype=tdt, device=dev)
    view = big[off:off + n * (V + pad)].view(n, V + pad)
    view[:, :V] = torch.as_tensor(rows.astype(np.float32), device=dev).to(tdt)
    L = view[:, :V]
    host = synth.host_rows(L.contiguous(), dtype)
    ref = oracle.margin_rows(host, dtype=dtype, vocab=V)
    got = relay.margin_rows(L)
    torch.cuda.synchronize()
    ok = (np.array_equal(got["top1"].cpu().numpy(), ref["top1"]) and
          np.array_equal(got["top2"].cpu().numpy(), ref["top2"]) and
          np.array_equal(got["status"].cpu().numpy(), ref["status"].astype(np.uint8)))
    s0 = ref["status"] == 0
    err = float(np.abs(got["margin"].cpu().numpy()[s0] - ref["margin"][s0]).max()) if s0.any() else 0.0
    ok = ok and err < 1e-5
    # K4 on the same rows, every work split (margins, top-2 and status of the decode step)
    if V >= 2 and n <= 2000:
        term = np.zeros(V, np.uint8)
        h = synth.CueSet(np.array([V - 1], np.int32), np.array([0, 1], np.int32), np.array([0], np.int32), 1, V,
                         term, -1, [(V - 1,)])
        cs = relay.CueSet.from_synth(h)
        for mode in ("strided", "flat", "dynamic", "cluster"):
            os.environ["RELAY_K4_MODE"] = mode
            st = torch.zeros(n, dtype=torch.uint8, device=dev)
            hist = torch.full((n, 7), -1, dtype=torch.int32, device=dev)
            o4 = relay.step_switch(cs, L, st, hist)
            torch.cuda.synchronize()
            ok = ok and np.array_equal(o4["top1"].cpu().numpy(), ref["top1"]) and \
                np.array_equal(o4["top2"].cpu().numpy(), ref["top2"])
            if s0.any():
                ok = ok and float(np.abs(o4["margin"].cpu().numpy()[s0] - ref["margin"][s0]).max()) < 1e-5
        os.environ.pop("RELAY_K4_MODE")
        cs.destroy()
    fails += not ok
    print(f"case {case:3d} n={n:5d} V={V:6d} pad={pad:2d} off={off} {dtype:4s}: {'ok' if ok else 'FAIL'} "
          f"max|dm|={err:.2e}", flush=True)
print("FAILURES:", fails)
