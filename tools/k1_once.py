"""One configs[1] K1 launch (relay_margin_rows) from a given library build,
for ncu:  python tools/k1_once.py [path/to/librelay.so] [launches]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2602_06454_b200 as relay  # noqa: E402
import synth  # noqa: E402

lib = C.CDLL(sys.argv[1]) if len(sys.argv) > 1 else relay._lib
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1
T, V = 32768, 151936
L = synth.make_logits(T, V, "bf16", device="cuda:0", chunk_rows=2048)
out = {k: torch.empty(T, dtype=d, device="cuda:0") for k, d in
       (("margin", torch.float32), ("top1", torch.int32), ("top2", torch.int32), ("lse", torch.float32),
        ("status", torch.uint8))}
P = C.c_void_p
lib.relay_margin_rows.argtypes = [P, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_float, P, P, P, P, P, P]
args = (L.data_ptr(), 0, T, V, V, 1.0, out["margin"].data_ptr(), out["top1"].data_ptr(), out["top2"].data_ptr(),
        out["lse"].data_ptr(), out["status"].data_ptr(), torch.cuda.current_stream().cuda_stream)
for _ in range(n):
    assert lib.relay_margin_rows(*args) == 0
torch.cuda.synchronize()
print("ok", float(out["margin"].float().mean()))
