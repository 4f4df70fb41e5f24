"""Tuning sweep for K1 (relay_margin_rows): build librelay variants with
different launch shapes (tools/k1_sweep.py build, on any host with nvcc) and
time them on one GPU on the configs[1] workload (tools/k1_sweep.py run).
Reports GB/s of algorithmic bytes and the fraction of MEASURED_PEAKS hbm_gbs."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "build", "k1_sweep")
VARIANTS = [  # (ncw, stages, uv, minb, extra): stage bytes = uv * ncw * 32 * 16
    (8, 4, 4, 3, ""), (8, 6, 2, 4, ""), (8, 4, 2, 4, ""), (12, 4, 2, 3, ""),
    (6, 6, 2, 5, ""), (16, 3, 2, 2, ""), (8, 6, 4, 2, ""), (8, 5, 4, 2, ""),
    (8, 4, 4, 3, "NULL"),
]


def name(v):
    return "w%d_s%d_u%d_m%d" % v[:4] + (("_" + v[4]) if v[4] else "")


def _builder():
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_relay_build", os.path.join(ROOT, "paper_2602_06454_b200", "_build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def defines(v):
    d = ["RELAY_K1_NCW=%d" % v[0], "RELAY_K1_STAGES=%d" % v[1], "RELAY_K1_UV=%d" % v[2],
         "RELAY_K1_MINB=%d" % v[3]]
    if v[4] == "NULL":
        d.append("RELAY_K1_NULL")
    elif v[4].startswith("S"):
        d.append("RELAY_PRODUCER_SLEEP_NS=%s" % v[4][1:])
    return d


def build():
    os.makedirs(OUT, exist_ok=True)
    b = _builder()
    for v in VARIANTS:
        so = os.path.join(OUT, "librelay_%s.so" % name(v))
        b.build_lib(so, defines=defines(v))
        print("built", so)


def run(cfg="c2", reps=20):
    import torch
    import synth
    c = synth.CONFIGS[cfg]
    T, V, dt = c["traj_len"], c["vocab"], c["dtype"]
    ts = synth.make_tokens(1, T, synth.make_cueset(V, c["n_cues"], c["n_pat"], max_len=c["max_len"]))
    L = synth.make_logits(T, V, dt, tokens=ts.tokens, device="cuda", chunk_rows=2048)
    esz = 2 if dt != "f32" else 4
    nbytes = T * (V * esz + 17)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0)
    outs = [torch.empty(T, dtype=d, device="cuda") for d in (torch.float32, torch.int32, torch.int32,
                                                                torch.float32, torch.uint8)]
    P = C.c_void_p
    res = {}
    for v in VARIANTS:
        so = os.path.join(OUT, "librelay_%s.so" % name(v))
        if not os.path.exists(so):
            continue
        lib = C.CDLL(so)
        f = lib.relay_margin_rows
        f.restype = C.c_int
        f.argtypes = [P, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_float, P, P, P, P, P, P]
        s = torch.cuda.current_stream()
        call = lambda: f(P(L.data_ptr()), {"bf16": 0, "f16": 1, "f32": 2}[dt], T, V, V, 1.0,
                         *[P(o.data_ptr()) for o in outs], P(s.cuda_stream))  # noqa: E731
        for _ in range(3):
            assert call() == 0
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
        for i in range(reps):
            ev[2 * i].record(s)
            call()
            ev[2 * i + 1].record(s)
        torch.cuda.synchronize()
        ms = sorted(ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(reps))
        med = ms[reps // 2]
        gbs = nbytes / (med / 1e3) / 1e9
        res[name(v)] = dict(ms_median=med, ms_best=ms[0], gbs=gbs, frac=gbs / peak)
        print(json.dumps({name(v): res[name(v)]}), flush=True)
    return res


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    else:
        run(*(sys.argv[2:3] or ["c2"]))
