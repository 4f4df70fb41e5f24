"""Small end-to-end run of every kernel (K1 all dtypes, K2 both modes, K3 incl.
per-trajectory tables, K4 in every work split, K5 sampler incl. the overflow
fallback, N1 partials/combine, N4 class patterns + decimal rule) for
compute-sanitizer: python tools/sanitize_smoke.py (under
compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_06454_b200 as relay  # noqa: E402
import synth  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    for dt, V, stride in (("bf16", 4099, 4107), ("f16", 3000, 3000), ("f32", 2053, 2060)):
        L = synth.make_logits(37, V, dt, row_stride=stride, device=dev)
        relay.margin_rows(L, vocab=V)
    h = synth.make_cueset(8192, 4, 6, max_len=3, seed=3)
    ts = synth.make_tokens(3, 3000, h, seed=4)
    n = ts.tokens.shape[0]
    tok = torch.as_tensor(ts.tokens, device=dev)
    offs = torch.as_tensor(ts.traj_offsets, device=dev)
    tep = torch.as_tensor(ts.think_end_pos, device=dev)
    for mode in (0, 1):
        cs = relay.CueSet.from_synth(h, mode=mode)
        L = synth.make_logits(n, 8192, "bf16", tokens=ts.tokens, device=dev)
        an = relay.Analyzer(cs, n, 8192, dev)
        an.run(L, tok, offs, tep)
        torch.cuda.synchronize()
        B = 48
        lg = synth.make_logits(B, 8192, "bf16", device=dev)
        st = torch.zeros(B, dtype=torch.uint8, device=dev)
        hist = torch.full((B, 7), -1, dtype=torch.int32, device=dev)
        sr = torch.zeros(B, dtype=torch.int32, device=dev)
        samp = torch.as_tensor(np.random.default_rng(5).integers(0, 8192, B).astype(np.int32), device=dev)
        for mode_k4 in ("strided", "flat", "dynamic"):
            os.environ["RELAY_K4_MODE"] = mode_k4
            for _ in range(2):
                relay.step_switch(cs, lg, st, hist, sr, samp, max_small_segment=4)
        os.environ.pop("RELAY_K4_MODE")
        uni = torch.rand(B, device=dev)
        lg[0] = 1.0                                   # a constant row: the exact fallback
        for _ in range(2):
            relay.step_sample(cs, lg, uni, st, hist, sr, top_k=20, top_p=0.95)
        # no top-k: K6 on bf16 (exact value counts), flat and tied rows, and f32 (value bins)
        lg[1] = torch.randn(8192, device=dev) * 0.05
        lg[2] = torch.arange(8192, device=dev).float().div(64).floor().neg()
        for p in (0.95, 1.0):
            relay.step_sample(cs, lg, uni, st, hist, sr, top_k=0, top_p=p)
            relay.step_sample(cs, lg.float(), uni, st, hist, sr, top_k=0, top_p=p)
        relay.segment_reduce(cs, an.rows["margin"], an.scan, offs, tep, per_trajectory=True)
        torch.cuda.synchronize()
        cs.destroy()
    # N1: vocabulary shards
    L = synth.make_logits(40, 6000, "bf16", device=dev)
    parts = [relay.margin_partials(L[:, i * 2000:(i + 1) * 2000], col_offset=i * 2000) for i in range(3)]
    relay.margin_combine(torch.stack(parts))
    # N4: class patterns and the decimal rule
    cc = synth.make_class_case(8192, 3, 2000, seed=6)
    cs = relay.CueSet(cc.cs.pat_tokens, cc.cs.pat_offsets, cc.cs.pat_cue, cc.cs.n_cues, cc.cs.terminator,
                      cc.cs.vocab, cc.cs.think_end, 0, cc.classes, cc.decimal_rule)
    tok = torch.as_tensor(cc.ts.tokens, device=dev)
    offs = torch.as_tensor(cc.ts.traj_offsets, device=dev)
    scan = relay.cue_scan(cs, tok, offs)
    m = torch.as_tensor(synth.make_margins(cc.ts.tokens.shape[0], seed=7), device=dev)
    relay.segment_reduce(cs, m, scan, offs)
    torch.cuda.synchronize()
    cs.destroy()
    print("sanitize smoke done")


if __name__ == "__main__":
    main()
