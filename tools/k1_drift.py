"""K1 time per step over a long run of the configs[1] pass (does the rate
drift with sustained load?).  Prints per-decile means and the SM clock."""
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2602_06454_b200 as relay  # noqa: E402
import synth  # noqa: E402

T, V, N = 32768, 151936, int(sys.argv[1]) if len(sys.argv) > 1 else 300
dev = torch.device("cuda:0")
L = synth.make_logits(T, V, "bf16", device=dev, chunk_rows=2048)
out = relay.margin_rows(L)
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(N)]
torch.cuda.synchronize()
for a, b in evs:
    a.record()
    relay.margin_rows(L, out=out)
    b.record()
torch.cuda.synchronize()
ms = [a.elapsed_time(b) for a, b in evs]
k = N // 10
for i in range(10):
    print(f"steps {i * k:4d}-{(i + 1) * k - 1:4d}: K1 {statistics.mean(ms[i * k:(i + 1) * k]):.4f} ms")
print(subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,temperature.gpu,temperature.memory,power.draw",
                      "--format=csv"], capture_output=True, text=True).stdout)
