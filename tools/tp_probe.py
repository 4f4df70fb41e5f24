"""Single-GPU timing of the N1 paths on configs[1]-shaped rows (tuning /
evidence only): relay_margin_rows on the full rows vs the fused TP path
(relay_margin_rows_tp, world 1: the partial-mode stream kernel storing its
per-row partials through the exchange buffer + the combine kernel) vs the
unfused partials + combine.  With one rank no bytes cross NVLink; the point
is the cost the fused exchange adds to the stream kernel.
    python tools/tp_probe.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2602_06454_b200 as relay  # noqa: E402
import synth  # noqa: E402


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:29533", rank=0, world_size=1)
    T, V = 32768, 151936
    L = synth.make_logits(T, V, "bf16", device="cuda:0", chunk_rows=2048)
    x = relay.TpExchange(rows_cap=T)
    full = relay.margin_rows(L)
    fused = x.margin_rows(L, 0)
    part = relay.margin_partials(L, 0)
    comb = relay.margin_combine(part.view(1, T, 8))
    bytes_ = T * V * 2
    for name, fn in (("margin_rows", lambda: relay.margin_rows(L, out=full)),
                     ("margin_rows_tp (fused, world 1)", lambda: x.margin_rows(L, 0, out=fused)),
                     ("partials + combine", lambda: relay.margin_combine(relay.margin_partials(L, 0, out=part)
                                                                         .view(1, T, 8), out=comb))):
        ms = timed(fn)
        print(f"{name:34s} {ms:7.3f} ms  {bytes_ / ms / 1e6:7.0f} GB/s", flush=True)
    torch.cuda.synchronize()
    assert torch.equal(fused["top1"], full["top1"]) and torch.equal(fused["top2"], full["top2"])
    x.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
