"""K1 per-element cost with the rows L2-resident (hot: the same 444 rows,
135 MB, relaunched back to back) vs streamed from HBM (configs[1]), per
library build: separates the compute side from the memory side.
    python tools/k1_hot.py a.so [b.so ...]"""
import ctypes as C
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402

V = 151936
big = synth.make_logits(32768, V, "bf16", device="cuda:0", chunk_rows=2048)
P = C.c_void_p
out = {k: torch.empty(32768, dtype=d, device="cuda:0") for k, d in
       (("margin", torch.float32), ("top1", torch.int32), ("top2", torch.int32), ("lse", torch.float32),
        ("status", torch.uint8))}


def run(lib, L, n, reps):
    a = (L.data_ptr(), 0, n, V, V, 1.0, out["margin"].data_ptr(), out["top1"].data_ptr(), out["top2"].data_ptr(),
         out["lse"].data_ptr(), out["status"].data_ptr(), torch.cuda.current_stream().cuda_stream)
    for _ in range(3):
        lib.relay_margin_rows(*a)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        lib.relay_margin_rows(*a)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for p in sys.argv[1:]:
    lib = C.CDLL(p)
    lib.relay_margin_rows.argtypes = [P, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_float, P, P, P, P, P, P]
    res = []
    for _ in range(3):
        hot = run(lib, big, 444, 200)
        cold = run(lib, big, 32768, 5)
        res.append((hot, cold))
    hot = statistics.median(r[0] for r in res)
    cold = statistics.median(r[1] for r in res)
    print(f"{os.path.basename(p):24s} hot 444 rows {hot * 1e3:8.1f} us = {444 * V / hot / 1e6:.3f} Gelem/ms"
          f"  cold 32768 rows {cold:.4f} ms = {32768 * V / cold / 1e9:.3f} Gelem/ms")
