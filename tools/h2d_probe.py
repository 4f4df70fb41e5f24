"""Host->device copy bandwidth from pinned memory with 1, 2 and 4 concurrent
streams (tuning the e2e path; evidence only)."""
import torch

n = 4 * 1024 ** 3
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda:0")
for k in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    part = n // k
    for _ in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i, s in enumerate(streams):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
        for s in streams:
            e1.wait_stream(s) if hasattr(e1, "wait_stream") else torch.cuda.current_stream().wait_stream(s)
        torch.cuda.current_stream().wait_stream(streams[0])
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
    print(f"{k} stream(s): {n / (e0.elapsed_time(e1) / 1e3) / 1e9:.1f} GB/s", flush=True)
