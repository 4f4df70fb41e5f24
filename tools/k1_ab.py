"""A/B of K1 (relay_margin_rows on configs[1]) between builds of the
library, interleaved in one process so clocks and thermals are shared:
    python tools/k1_ab.py path/to/librelay_a.so path/to/librelay_b.so [...] [rounds]"""
import ctypes as C
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2602_06454_b200 as relay  # noqa: E402
import synth  # noqa: E402

paths = [a for a in sys.argv[1:] if a.endswith(".so")]
rounds = int(sys.argv[-1]) if not sys.argv[-1].endswith(".so") else 8
libs = [C.CDLL(p) for p in paths]
T, V = 32768, 151936
L = synth.make_logits(T, V, "bf16", device="cuda:0", chunk_rows=2048)
out = {k: torch.empty(T, dtype=d, device="cuda:0") for k, d in
       (("margin", torch.float32), ("top1", torch.int32), ("top2", torch.int32), ("lse", torch.float32),
        ("status", torch.uint8))}
P = C.c_void_p
for lib in libs:
    lib.relay_margin_rows.argtypes = [P, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_float, P, P, P, P, P, P]
args = (L.data_ptr(), 0, T, V, V, 1.0, out["margin"].data_ptr(), out["top1"].data_ptr(), out["top2"].data_ptr(),
        out["lse"].data_ptr(), out["status"].data_ptr(), torch.cuda.current_stream().cuda_stream)
res = [[] for _ in libs]
for _ in range(rounds):
    for k, lib in enumerate(libs):
        for _ in range(2):
            lib.relay_margin_rows(*args)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            lib.relay_margin_rows(*args)
        e1.record()
        torch.cuda.synchronize()
        res[k].append(e0.elapsed_time(e1) / 5)
for k in range(len(libs)):
    print(f"{os.path.basename(paths[k])}: median {statistics.median(res[k]):.4f} ms  min {min(res[k]):.4f}")
