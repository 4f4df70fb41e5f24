"""Randomised parity sweep of K2 (relay_cue_scan) + K3 (relay_segment_reduce)
against the oracle: random trajectory counts and lengths (incl. tiny ones),
cue sets (1-32 patterns of length 1-6, both match modes), cue densities,
think-end restriction, NaN margins and tau (evidence; tests/ holds the fixed
cases).   python tools/segment_fuzz.py [n_cases] [seed]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2602_06454_b200 as relay  # noqa: E402
import synth  # noqa: E402
from test_gpu_parity import _compare_segments  # noqa: E402

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 4)
dev = torch.device("cuda:0")
fails = 0
for case in range(n_cases):
    V = 151936
    n_cues = int(rng.integers(1, 9))
    n_pat = int(rng.integers(n_cues, min(32, 4 * n_cues) + 1))
    max_len = int(rng.integers(1, 7))
    mode = int(rng.integers(0, 2))
    h = synth.make_cueset(V, n_cues, n_pat, max_len=max_len, seed=int(rng.integers(1 << 30)))
    cs = relay.CueSet.from_synth(h, mode=mode)
    n_traj = int(rng.choice([1, 3, 9, 40]))
    L = int(rng.choice([1, 5, 300, 2048, 5000]))
    ts = synth.make_tokens(n_traj, L, h, seed=int(rng.integers(1 << 30)), cue_rate=float(rng.choice([0.1, 0.5, 0.9])))
    tau = float(rng.choice([0.1, 0.5, 0.9]))
    think = bool(rng.integers(0, 2))
    m = synth.make_margins(ts.tokens.shape[0], seed=int(rng.integers(1 << 30)),
                           nan_rate=float(rng.choice([0.0, 0.0, 0.01])), tau=tau)
    tok = torch.as_tensor(ts.tokens, device=dev)
    offs = torch.as_tensor(ts.traj_offsets, device=dev)
    tep = torch.as_tensor(ts.think_end_pos, device=dev) if think else None
    try:
        scan = relay.cue_scan(cs, tok, offs)
        seg = relay.segment_reduce(cs, torch.as_tensor(m, device=dev), scan, offs, tep, tau=tau)
        torch.cuda.synchronize()
        o_scan, o_win, o_sum = oracle.analyze(m, ts.tokens, ts.traj_offsets, h.pat_tokens, h.pat_offsets,
                                              h.pat_cue, h.n_cues, h.terminator, tau=tau,
                                              think_end_pos=ts.think_end_pos if think else None, mode=mode,
                                              min_count=1)
        n = int(scan["n_occ"].item())
        assert np.array_equal(scan["occ_pos"][:n].cpu().numpy(), o_scan["occ_pos"])
        _compare_segments(relay, h, scan, seg, o_scan, o_win, o_sum)
        ok, msg = True, f"{n} occurrences"
    except AssertionError as e:
        ok, msg = False, repr(e)[:200]
    fails += not ok
    print(f"case {case:3d} traj={n_traj:3d}x{L:5d} cues={n_cues} pats={n_pat:2d} len<={max_len} mode={mode} "
          f"think={int(think)} tau={tau}: {'ok' if ok else 'FAIL'} {msg}", flush=True)
    cs.destroy()
print("FAILURES:", fails)
