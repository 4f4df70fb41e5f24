"""Global timeline of one relay_step_sample step (K4 margin pass + K5 sampler)
at configs[2] from a traced build (tuning only):
    python tools/k45_timeline.py build     # librelay with -DRELAY_TRACE into build/trace/
    python tools/k45_timeline.py run [top_k]
Prints percentiles (us from the first K4 CTA entry) of K4 CTA entry / row
done / exit and K5 CTA entry / row ready / candidates / ranked / done."""
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


def run(top_k=20):
    import numpy as np
    os.environ["RELAY_LIB"] = OUT
    import torch
    import paper_2602_06454_b200 as relay
    import synth
    dev = torch.device("cuda:0")
    B, V = 256, 152064
    h = synth.make_cueset(V, 8, 12, max_len=3)
    cs = relay.CueSet.from_synth(h)
    L = synth.make_logits(B, V, "bf16", seed=100, device=dev)
    state = torch.zeros(B, dtype=torch.uint8, device=dev)
    hist = torch.full((B, 7), -1, dtype=torch.int32, device=dev)
    uni = torch.rand(B, device=dev)
    ws = relay.workspace(0, 0, B, dev)
    for _ in range(3):
        relay.step_sample(cs, L, uni, state, hist, temperature=0.6, top_k=top_k, top_p=0.95, ws=ws)
    torch.cuda.synchronize()
    lib = C.CDLL(OUT)
    z = np.zeros((4096, 32), np.uint64)
    lib.relay_debug_trace_reset.argtypes = [C.c_void_p, C.c_int]
    assert lib.relay_debug_trace_reset(z.ctypes.data_as(C.c_void_p), 4096) == 0
    relay.step_sample(cs, L, uni, state, hist, temperature=0.6, top_k=top_k, top_p=0.95, ws=ws)
    torch.cuda.synchronize()
    k4 = np.zeros((4096, 32), np.uint64)
    k5 = np.zeros((1024, 16), np.uint64)
    lib.relay_debug_trace_copy.argtypes = [C.c_void_p, C.c_int]
    lib.relay_debug_trace5_copy.argtypes = [C.c_void_p, C.c_int]
    lib.relay_debug_trace_copy(k4.ctypes.data_as(C.c_void_p), 4096)
    lib.relay_debug_trace5_copy(k5.ctypes.data_as(C.c_void_p), 1024)
    t0 = int(k4[:, 0][k4[:, 0] > 0].min())

    def pct(name, col):
        v = col[col > 0].astype(np.int64)
        if v.size == 0:
            return
        v = (v - t0) / 1e3
        print(f"{name:28s} n {v.size:4d}  min {v.min():6.1f}  p10 {np.percentile(v, 10):6.1f}  med {np.median(v):6.1f}"
              f"  p90 {np.percentile(v, 90):6.1f}  max {v.max():6.1f}")
    pct("K4 CTA entry", k4[:, 0])
    pct("K4 first stage landed", k4[:, 1])
    pct("K4 consumer row done", k4[:, 16])
    pct("K4 epilogue row done", k4[:, 24])
    pct("K4 exit (consumer 0)", k4[:, 31])
    pct("K5 CTA entry", k5[:, 13])
    pct("K5 row taken (ready)", k5[:, 14])
    pct("K5 candidates", k5[:, 1])
    pct("K5 ranked", k5[:, 2])
    pct("K5 row done", k5[:, 15])


if __name__ == "__main__":
    build() if sys.argv[1] == "build" else run(*(int(x) for x in sys.argv[2:3]))
