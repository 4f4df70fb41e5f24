import sys, json, torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2602_06454_b200 as relay, synth
B, V = 256, 152064
dev = torch.device('cuda:0')
bufs = [synth.make_logits(B, V, 'bf16', seed=100 + i, device=dev) for i in range(7)]
outs = relay.margin_rows(bufs[0])
def timeit(fn, n=7, reps=30):
    s = torch.cuda.Stream(); g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        for i in range(n): fn(i)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for i in range(n): fn(i)
    torch.cuda.synchronize()
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): g.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * n)
print("K1 on 256 rows (one row per CTA): us", timeit(lambda i: relay.margin_rows(bufs[i % 7], out=outs)))
for rows in (444, 888, 1776, 4096):
    big = synth.make_logits(rows, V, 'bf16', seed=7, device=dev)
    ob = relay.margin_rows(big)
    t = timeit(lambda i: relay.margin_rows(big, out=ob), n=3, reps=20)
    print(f"K1 on {rows} rows: us {t:.1f}  GB/s {rows*V*2/t/1e3:.0f}")
