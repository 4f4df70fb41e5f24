"""Decode-step switch (K4 relay_step_switch) timing on configs[2]: batch 256
live sequences x 152,064-vocab bf16 logits per step.  Rotates through enough
distinct logits buffers (>= 4 x L2) that every step streams from HBM ("cold"),
and also times the L2-resident case ("hot", as right after the LM head).
Prints one JSON line: us/step, rows/s, GB/s of algorithmic bytes, fraction of
MEASURED_PEAKS hbm_gbs."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_06454_b200 as relay  # noqa: E402
import synth  # noqa: E402


def main(B=256, V=152064, steps=200, graph=True, sample=False, top_k=20):
    dev = torch.device("cuda:0")
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    nbuf = max(2, int(np.ceil(4 * l2 / (B * V * 2))))
    h = synth.make_cueset(V, 8, 12, max_len=3)
    cs = relay.CueSet.from_synth(h)
    bufs = [synth.make_logits(B, V, "bf16", seed=100 + i, device=dev) for i in range(nbuf)]
    state = torch.zeros(B, dtype=torch.uint8, device=dev)
    hist = torch.full((B, 7), -1, dtype=torch.int32, device=dev)
    small = torch.zeros(B, dtype=torch.int32, device=dev)
    samp = torch.randint(3000, V, (B,), dtype=torch.int32, device=dev)
    ws = relay.workspace(0, 0, B, dev)
    uni = torch.rand(B, device=dev)

    def step(x, out=None):
        if sample:   # N2: the paper's Qwen3 sampling (T 0.6, top-p 0.95, top-k 20)
            return relay.step_sample(cs, x, uni, state, hist, small, temperature=0.6, top_k=top_k,
                                     top_p=0.95, ws=ws, out=out)
        return relay.step_switch(cs, x, state, hist, small, samp, ws=ws, out=out)
    out = step(bufs[0])
    torch.cuda.synchronize()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0)
    res = {}
    # steps are captured in one CUDA graph (as a serving engine would run the
    # decode step), so the number is device time, not Python launch overhead
    reps = max(1, steps // nbuf)
    for mode in ("cold", "hot"):
        seq = [bufs[i % nbuf] if mode == "cold" else bufs[0] for i in range(nbuf)]
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            for x in seq:                     # warm-up on the capture stream
                step(x, out)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                for x in seq:
                    step(x, out)
        torch.cuda.synchronize()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (reps * nbuf)
        gbs = B * (V * 2 + 12) / (us * 1e-6) / 1e9
        res[mode] = dict(us_per_step=us, rows_per_s=B / (us * 1e-6), gbs=gbs, frac=gbs / peak)
    # host cost of one eager Python call (argument marshalling + launch)
    torch.cuda.synchronize()
    import time
    t0 = time.perf_counter()
    for _ in range(100):
        step(bufs[0], out)
    res["eager_host_us_per_call"] = (time.perf_counter() - t0) * 1e4
    torch.cuda.synchronize()
    print(json.dumps({"kernel": "relay_step_sample (K4 + K5)" if sample else "relay_step_switch (K4)",
                      "batch": B, "vocab": V, "buffers": nbuf,
                      "l2_bytes": l2, **res}), flush=True)
    cs.destroy()


if __name__ == "__main__":
    main(sample="--sample" in sys.argv, top_k=0 if "--no-topk" in sys.argv else 20)
