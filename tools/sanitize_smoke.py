"""Small end-to-end run of every kernel (K1 all dtypes, K2 both modes, K3, K4)
for compute-sanitizer: python tools/sanitize_smoke.py (under
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
        for _ in range(3):
            relay.step_switch(cs, lg, st, hist, sr, samp, max_small_segment=4)
        torch.cuda.synchronize()
        cs.destroy()
    print("sanitize smoke done")


if __name__ == "__main__":
    main()
