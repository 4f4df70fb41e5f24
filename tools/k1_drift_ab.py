"""Sustained-load A/B of K1 builds: blocks of back-to-back configs[1] launches
(default 1200 = ~2 s each), alternating libraries, so each block runs at the
clock the box settles at under that kernel's own power draw.  Reports per block
the mean K1 time over its last 2/3 and the SM clock / power sampled during it.
    python tools/k1_drift_ab.py a.so b.so [...] [--blocks 2] [--n 1200]"""
import argparse
import ctypes as C
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs="+")
ap.add_argument("--blocks", type=int, default=2)
ap.add_argument("--n", type=int, default=1200)
args = ap.parse_args()
T, V = 32768, 151936
L = synth.make_logits(T, V, "bf16", device="cuda:0", chunk_rows=2048)
out = {k: torch.empty(T, dtype=d, device="cuda:0") for k, d in
       (("margin", torch.float32), ("top1", torch.int32), ("top2", torch.int32), ("lse", torch.float32),
        ("status", torch.uint8))}
P = C.c_void_p
libs = []
for p in args.libs:
    lib = C.CDLL(p)
    lib.relay_margin_rows.argtypes = [P, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_float, P, P, P, P, P, P]
    libs.append(lib)
cargs = (L.data_ptr(), 0, T, V, V, 1.0, out["margin"].data_ptr(), out["top1"].data_ptr(), out["top2"].data_ptr(),
         out["lse"].data_ptr(), out["status"].data_ptr(), torch.cuda.current_stream().cuda_stream)


def sampler(stop, acc):
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                           capture_output=True, text=True).stdout.strip().split(",")
        try:
            acc.append((float(r[0]), float(r[1])))
        except (ValueError, IndexError):
            pass
        time.sleep(0.1)


for b in range(args.blocks):
    for k, lib in enumerate(libs):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.n)]
        stop, acc = threading.Event(), []
        th = threading.Thread(target=sampler, args=(stop, acc))
        th.start()
        for e0, e1 in evs:
            e0.record()
            lib.relay_margin_rows(*cargs)
            e1.record()
        torch.cuda.synchronize()
        stop.set()
        th.join()
        ms = [e0.elapsed_time(e1) for e0, e1 in evs][args.n // 3:]
        clk = statistics.median(a[0] for a in acc) if acc else float("nan")
        pw = statistics.median(a[1] for a in acc) if acc else float("nan")
        gbs = T * (V * 2 + 17) / statistics.mean(ms) / 1e6
        print(f"block {b} {os.path.basename(args.libs[k]):24s} K1 {statistics.mean(ms):.4f} ms  {gbs:7.1f} GB/s  "
              f"sm {clk:.0f} MHz  {pw:.0f} W  ({len(acc)} samples)", flush=True)
