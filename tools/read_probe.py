"""Reference points for the decode-step kernel (K4) on configs[2]-sized
buffers (256 x 152,064 bf16 = 77.9 MB): how long do plain library reductions
over the same bytes take inside a CUDA graph, rotating 7 buffers (> 4 x L2)?"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402


def timeit(fns, reps=30):
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        for f in fns:
            f()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for f in fns:
                f()
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
    return e0.elapsed_time(e1) * 1e3 / (reps * len(fns))


def main(B=256, V=152064):
    dev = torch.device("cuda:0")
    bufs = [synth.make_logits(B, V, "bf16", seed=100 + i, device=dev) for i in range(7)]
    out = torch.empty(B, dtype=torch.bfloat16, device=dev)
    tiny = torch.zeros(1, device=dev)
    res = {}
    res["empty_kernel_us"] = timeit([lambda: tiny.add_(1)] * 7)
    res["amax_rows_us"] = timeit([lambda b=b: torch.amax(b, dim=1, out=out) for b in bufs])
    res["sum_all_us"] = timeit([lambda b=b: b.sum() for b in bufs])
    flat = [b.view(-1) for b in bufs]
    o2 = torch.empty_like(flat[0])
    res["copy_us(2x bytes)"] = timeit([lambda b=b: o2.copy_(b) for b in flat])
    res["bytes"] = B * V * 2
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
