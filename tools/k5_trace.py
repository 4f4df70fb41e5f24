"""Timeline of K5 (the sampling kernel of relay_step_sample) from a traced
build, for a batch whose row 0 is pathological (tuning only):
    python tools/k5_trace.py build
    python tools/k5_trace.py run [const|flat|plain] [top_k]
Stamps (us from the CTA's row start): 1 candidates collected, 2 top list,
3 mass / fast-path test, 4 level-1 histogram, 5 total, 6-7 level-2 pass
(cut), 8-9 draw bin, 10 level-2 pass (draw), 11-12 tie index, 15 row done.
Value-bin path (f16/f32): 6 level 1 built, 7 cut selected, 10 draw selected."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "build", "trace", "librelay.so")


def build():
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_relay_build", os.path.join(ROOT, "paper_2602_06454_b200", "_build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    mod.build_lib(OUT, defines=["RELAY_TRACE"])


def run(kind="const", top_k=0, dtype="bf16"):
    import numpy as np
    import torch
    import paper_2602_06454_b200 as relay
    relay.LIB_PATH = OUT
    relay._lib = relay._load()
    import synth
    dev = torch.device("cuda:0")
    B, V = 256, 152064
    h = synth.make_cueset(V, 8, 12, max_len=3)
    cs = relay.CueSet.from_synth(h)
    x = synth.make_logits(B, V, dtype, seed=100, device=dev, edge_rows=False)
    if kind == "const":
        x[0].fill_(1.25)
    elif kind == "flat":
        x[0].normal_(0, 0.05)
    state = torch.zeros(B, dtype=torch.uint8, device=dev)
    hist = torch.full((B, 7), -1, dtype=torch.int32, device=dev)
    uni = torch.full((B,), 0.5, device=dev)
    ws = relay.workspace(0, 0, B, dev)
    lib = relay._lib
    lib.relay_debug_trace5_copy.argtypes = [C.c_void_p, C.c_int]
    for _ in range(3):
        relay.step_sample(cs, x, uni, state.zero_(), hist.fill_(-1), top_k=top_k, ws=ws)
    torch.cuda.synchronize()
    buf = np.zeros((B, 16), np.uint64)
    lib.relay_debug_trace5_copy(buf.ctypes.data, B)
    t = buf.astype(np.int64)
    t0 = t[:, 0:1]
    rel = np.where(t > 0, (t - t0) / 1e3, np.nan)
    print(f"row0 ({kind}, {dtype}, top_k={top_k}):", " ".join(f"{k}:{rel[0, k]:.1f}" for k in range(16) if t[0, k] > 0))
    med = np.nanmedian(rel[1:], axis=0)
    print("median other rows:", " ".join(f"{k}:{med[k]:.1f}" for k in range(16) if not np.isnan(med[k])))
    print("CTA start spread (us):", (t0.max() - t0.min()) / 1e3)
    cs.destroy()


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    else:
        run(sys.argv[2] if len(sys.argv) > 2 else "const", int(sys.argv[3]) if len(sys.argv) > 3 else 0,
            sys.argv[4] if len(sys.argv) > 4 else "bf16")
