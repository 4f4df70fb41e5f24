"""Timeline of the row kernel (K4 decode step by default) from a traced build:
    python tools/trace_rows.py build     # librelay with -DRELAY_TRACE into build/trace/
    python tools/trace_rows.py run       # one graph-free step on cuda:0, per-CTA stamps (us)
Stamps: 0 entry, 1 first stage landed (consumer warp 0), 2.. consumer item ends,
10.. epilogue item ends, 15 consumer exit."""
import ctypes as C
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "build", "trace", "librelay.so")
SRC = [os.path.join(ROOT, "paper_2602_06454_b200", "csrc", f)
       for f in ("margin_kernels.cu", "scan_kernels.cu", "relay_api.cu")]


def build():
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                           "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
                           "-DRELAY_TRACE", "-o", OUT] + SRC)


def run(mode="step"):
    import numpy as np
    import torch
    import paper_2602_06454_b200 as relay
    relay.LIB_PATH = OUT
    relay._lib = relay._load()
    import synth
    dev = torch.device("cuda:0")
    B, V = (256, 152064) if mode == "step" else (444, 152064)
    h = synth.make_cueset(V, 8, 12, max_len=3)
    cs = relay.CueSet.from_synth(h)
    L = synth.make_logits(B, V, "bf16", device=dev)
    state = torch.zeros(B, dtype=torch.uint8, device=dev)
    hist = torch.full((B, 7), -1, dtype=torch.int32, device=dev)
    ws = relay.workspace(0, 0, B, dev)
    for _ in range(3):
        if mode == "step":
            relay.step_switch(cs, L, state, hist, ws=ws)
        else:
            relay.margin_rows(L)
    torch.cuda.synchronize()
    n = 444
    buf = np.zeros((n, 16), np.uint64)
    lib = C.CDLL(OUT)
    lib.relay_debug_trace_copy.argtypes = [C.c_void_p, C.c_int]
    assert lib.relay_debug_trace_copy(buf.ctypes.data_as(C.c_void_p), n) == 0
    t0 = int(buf[:, 0][buf[:, 0] > 0].min())
    rel = np.where(buf > 0, (buf.astype(np.int64) - t0) / 1e3, np.nan)
    np.set_printoptions(linewidth=200, precision=1, suppress=True)
    cols = [0, 1, 2, 3, 4, 10, 11, 12, 15]
    print("cols", cols)
    for b in list(range(0, n, 37)) + [n - 1]:
        print(b, rel[b, cols])
    print("max entry", np.nanmax(rel[:, 0]), "max consumer exit", np.nanmax(rel[:, 15]),
          "max epilogue", np.nanmax(rel[:, 10:15]))


if __name__ == "__main__":
    build() if sys.argv[1] == "build" else run(*(sys.argv[2:3] or ["step"]))
