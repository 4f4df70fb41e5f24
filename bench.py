#!/usr/bin/env python
"""Benchmark of the RelayGen hot path on B200 (BASELINE.json metric).

One step = one pass of the whole offline hot path over a
batch of synthetic input resident in HBM: stats init, K1 relay_margin_rows
over every logit row, K2 relay_cue_scan, K3 relay_segment_reduce, (N>1) the
NCCL sum all-reduce of the uint64 statistics table (H6), the 4 KB table read
back and relay_stats_finalize on the host (H7).

Workload per rank (weak scaling, default --config c2): one Qwen3-32B-shaped
reasoning trajectory of 32,768 tokens x 151,936-vocab bf16 logits with 8
switch cues (configs[1]).  --config c4 is configs[3] as stated: the FIXED
corpus of 8 x 32,768-token trajectories sharded by trajectory over the N
ranks (strong scaling; N = 1 holds all 79.7 GB), so T(1)/T(8) is read off
directly.  Inputs (>= 9.96 GB of logits per rank) are far larger than the
126 MB L2, so no flush is needed between steps.  Every line also carries a
"sustained" sub-record: ~3 s of back-to-back steps with the clocks sampled
(the rate once the SM clock has settled under the 1,000 W power cap).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl relay|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "logit rows/sec and HBM GB/s (fraction of ~8 TB/s) for margin+segment pass, 1/2/4/8 GPU"
UNIT = "rows/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="relay", choices=["relay", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c4", "c5"],
                    help="c2 (default, the metric's workload): one 32,768-token trajectory per rank "
                         "(weak scaling); c4: the FIXED corpus of 8 x 32,768-token trajectories sharded "
                         "by trajectory over the ranks (strong scaling; N = 1 holds all 79.7 GB); c1; "
                         "c5: the cue-set sweep corpus (8 x 16,384-token trajectories per rank, 32 patterns "
                         "of length 1-6, logits streamed in --chunk-rows chunks from a ~10 GB buffer pool)")
    ap.add_argument("--sustained-s", type=float, default=3.0,
                    help="after the timed steps, back-to-back steps for this many seconds with the clocks "
                         "sampled (the 'sustained' sub-record: the rate at the clock the box settles at "
                         "under this kernel's own power draw); 0 = off")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--chunk-rows", type=int, default=8192, help="c5: logit rows per streamed chunk")
    ap.add_argument("--shard", default="trajectory", choices=["trajectory", "rows"],
                    help="trajectory: one trajectory per rank (weak scaling, the default); rows: ONE "
                         "trajectory split over the ranks at safe cuts (strong scaling, dist.safe_cuts)")
    ap.add_argument("--no-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-decode", action="store_true", help="skip the decode-step (configs[2]) line")
    ap.add_argument("--profile", action="store_true", help="minimal run for ncu (no clocks/e2e/baseline)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--allreduce", default="nccl", choices=["nccl", "p2p"],
                    help="H6 over NCCL (relay_stats_allreduce) or fused into K3 over peer memory "
                         "(relay_segment_reduce_p2p)")
    ap.add_argument("--serial-scan", action="store_true",
                    help="run K2 before K1 on the main stream instead of on a side stream")
    return ap.parse_args()


class Clocks:
    """nvidia-smi sampling during the timed region (the recipe's clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if len(r) >= 6 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 6 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 6 for i in range(4)
                          if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def workload(cfg: str):
    import synth
    c = synth.CONFIGS[cfg]
    return c


def oracle_pass(rows_host, dtype, vocab, tokens, offs, cs_h, threads):
    """The whole hot path in the oracle: margins, scan, windows, stats."""
    import oracle
    ref = oracle.margin_rows(rows_host, dtype=dtype, vocab=vocab, threads=threads)
    m32 = ref["margin"].astype(np.float32)
    oracle.analyze(m32, tokens, offs, cs_h.pat_tokens, cs_h.pat_offsets, cs_h.pat_cue, cs_h.n_cues,
                   cs_h.terminator)


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args):
    """--impl reference: the oracle, as it stands, on this box's host cores,
    each step a contiguous sub-trajectory sample of the same workload."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import synth
    c = workload(args.config)
    vocab, dtype = c["vocab"], c["dtype"]
    cs_h = synth.make_cueset(vocab, c["n_cues"], c["n_pat"], max_len=c["max_len"])
    ts = synth.make_tokens(1, c["traj_len"], cs_h)
    threads = cpu_threads()
    # size the sample so a step takes ~1 s on this host (whole run: a few minutes)
    probe = synth.make_logits(8, vocab, dtype, tokens=ts.tokens[:8], device="cpu")
    host = synth.host_rows(probe, dtype)
    t0 = time.perf_counter()
    oracle_pass(host, dtype, vocab, ts.tokens[:8], None, cs_h, 1)
    per_row = (time.perf_counter() - t0) / 8
    budget = min(1.5, 150.0 / max(1, args.steps + args.warmup))
    S = int(max(threads, min(c["traj_len"], budget * threads / max(per_row, 1e-9))))
    S = max(threads, S // threads * threads)
    L = synth.make_logits(S, vocab, dtype, tokens=ts.tokens[:S], device="cpu")
    host = synth.host_rows(L, dtype)
    toks = np.ascontiguousarray(ts.tokens[:S])
    for _ in range(args.warmup):
        oracle_pass(host, dtype, vocab, toks, None, cs_h, threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle_pass(host, dtype, vocab, toks, None, cs_h, threads)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = S * args.steps / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{args.config}: oracle on a {S}-row contiguous sample of the "
                   f"{c['traj_len']}-token x {vocab}-vocab {dtype} trajectory per step",
                   "rows_per_step": S},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": f"{S} rows per step (plain C fp64 oracle, {threads} threads)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.config == "c5":
        run_c5(args)
        return
    import torch
    import torch.distributed as dist

    import paper_2602_06454_b200 as relay
    import synth
    from paper_2602_06454_b200.dist import allreduce_stats

    rank, world, local = dist_env()
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N>1 must be launched with torchrun (one process per GPU)")
    # RELAY_BENCH_SAME_DEVICE=1: every rank on cuda:0 (a 1-GPU functional check of the
    # multi-rank path with --dist-backend gloo; its timings are not a scaling result)
    if os.environ.get("RELAY_BENCH_SAME_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)
    c = workload(args.config)
    vocab, dtype, T = c["vocab"], c["dtype"], c["traj_len"]
    cs_h = synth.make_cueset(vocab, c["n_cues"], c["n_pat"], max_len=c["max_len"])
    cs = relay.CueSet.from_synth(cs_h)
    T_job = T * world   # rows of the whole job (weak scaling: one trajectory per rank)
    n_my = 1            # trajectories of this rank
    if args.config == "c4":
        # the fixed corpus: global trajectory g (tokens seed BASE+g, logits seed BASE+17g,
        # the same for every world size) -> rank g*world//8; T_job = 8 x 32,768 rows
        if args.shard == "rows":
            raise SystemExit("--config c4 shards by trajectory")
        NT = c["n_traj"]
        if world > NT:
            raise SystemExit(f"--config c4 has {NT} trajectories: at most {NT} ranks")
        mine = list(range(rank * NT // world, (rank + 1) * NT // world))
        n_my = len(mine)
        parts = [synth.make_tokens(1, T, cs_h, seed=synth.BASE_SEED + g) for g in mine]
        toks = np.concatenate([p.tokens for p in parts]).astype(np.int32)
        offs_np = np.arange(n_my + 1, dtype=np.int64) * T
        tep_np = np.array([p.think_end_pos[0] + k * T for k, p in enumerate(parts)], np.int64)
        ts = synth.TokenStream(toks, offs_np, tep_np)
        T_job = NT * T
        logits = torch.empty((n_my * T, vocab), dtype=torch.bfloat16 if dtype == "bf16" else torch.float32,
                             device=dev)
        for k, g in enumerate(mine):
            logits[k * T:(k + 1) * T] = synth.make_logits(T, vocab, dtype, tokens=parts[k].tokens,
                                                          seed=synth.BASE_SEED + 17 * g, device=dev,
                                                          chunk_rows=2048)
        T = n_my * T
    elif args.shard == "rows":
        # strong scaling: one trajectory (the same on every rank), split at safe cuts
        from paper_2602_06454_b200.dist import range_view, safe_cuts
        full = synth.make_tokens(1, T, cs_h, seed=synth.BASE_SEED)
        cuts = safe_cuts(full.tokens, full.traj_offsets, cs_h.terminator, world, cs_h.pat_tokens)
        lo, hi = int(cuts[rank]), int(cuts[rank + 1])
        t_np, o_np, te_np = range_view(full.tokens, full.traj_offsets, full.think_end_pos, lo, hi)
        ts = synth.TokenStream(t_np.astype(np.int32), o_np, te_np)
        T, T_job = hi - lo, T
    else:
        ts = synth.make_tokens(1, T, cs_h, seed=synth.BASE_SEED + rank)
    if args.config != "c4":
        logits = synth.make_logits(max(T, 1), vocab, dtype, tokens=ts.tokens, seed=synth.BASE_SEED + 17 * rank,
                                   device=dev, chunk_rows=2048)[:T]
    tok = torch.as_tensor(ts.tokens, device=dev)
    offs = torch.as_tensor(ts.traj_offsets, device=dev)
    tep = torch.as_tensor(ts.think_end_pos, device=dev)
    # inputs smaller than 4 x L2 (c1: 262 MB): rotate through enough distinct
    # copies that every step streams from HBM (the same logits, other addresses)
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    in_bytes = logits.numel() * logits.element_size()
    n_rot = max(1, -(-4 * l2_bytes // max(in_bytes, 1)))
    rot = [logits] + [logits.clone() for _ in range(n_rot - 1)]
    # --allreduce p2p: H6 fused into K3 over peer memory (relay_segment_reduce_p2p)
    xchg = relay.StatsExchange(cs.n_cues) if (world > 1 and args.allreduce == "p2p") else None
    an = relay.Analyzer(cs, T, vocab, dev, rank=rank, world_size=world,
                        overlap_scan=not args.serial_scan, exchange=xchg)
    stream = torch.cuda.current_stream()
    # two pinned host tables: step i's table is finalized on the host while the
    # GPU already runs step i+1 (the work per step is unchanged)
    host_stats = [torch.empty(an.stats.shape, dtype=torch.int64, pin_memory=True) for _ in range(2)]
    done = [torch.cuda.Event(), torch.cuda.Event()]
    k1_ev = []
    results = []

    def h6(stats):
        if xchg is None:                                # (p2p: already summed by K3's last CTA)
            allreduce_stats(stats, cs.n_cues, world)    # H6: relay_stats_allreduce (NCCL)

    def launch(i, timed=False):
        """Device side of step i: H1-H5 (K1 timed with events on its stream), H6, D2H."""
        e0 = e1 = None
        if timed:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
        an.run(rot[i % n_rot], tok, offs, tep, k1_events=(e0, e1) if timed else None)
        if timed:
            k1_ev.append((e0, e1))
        if world > 1:
            h6(an.stats)
        host_stats[i % 2].copy_(an.stats, non_blocking=True)
        done[i % 2].record(stream)

    def finish(i):
        done[i % 2].synchronize()
        results.append(relay.stats_finalize(host_stats[i % 2].numpy(), cs.n_cues, world))   # H7

    def run_steps(n, timed=False):
        for i in range(n):
            launch(i, timed)
            if i > 0:
                finish(i - 1)
        finish(n - 1)

    run_steps(args.warmup)
    clocks = Clocks(local)
    if not args.profile:
        clocks.start()
        time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    run_steps(args.steps, timed=True)
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ck = clocks.stop() if not args.profile else None
    ms = t0.elapsed_time(t1)
    k1_ms = statistics.mean(a.elapsed_time(b) for a, b in k1_ev)
    if world > 1:
        t = torch.tensor([ms, k1_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, k1_ms = float(t[0]), float(t[1])
    sustained = None
    if args.sustained_s > 0 and not args.profile:
        sustained = measure_sustained(args, ms / args.steps, run_steps, k1_ev, local, world, dev, T, T_job,
                                      vocab, {"bf16": 2, "f16": 2, "f32": 4}[dtype])
    rows_total = T_job * args.steps
    value = rows_total / (ms / 1e3)
    esz = {"bf16": 2, "f16": 2, "f32": 4}[dtype]
    k1_bytes = T * (vocab * esz + 17)      # logits read + margin/top1/top2/lse/status written
    achieved = k1_bytes / (k1_ms / 1e3) / 1e9
    pk = peaks()
    peak = pk.get("hbm_gbs") or 6650.0
    traffic, traffic_src = None, None
    tf = os.path.join(ROOT, "profiles", "k1_traffic.json")
    if os.path.exists(tf):
        try:
            tj = json.load(open(tf))
            rec = tj.get(args.config, {})
            traffic = rec.get("dram_bytes_per_launch")
            if traffic is not None and args.config == "c4":
                traffic = None   # profiled at configs[1]; per-launch bytes scale with the rows
            traffic_src = (f"profiled offline, not this run: {rec.get('profile', tj.get('_source'))} "
                           f"(kernel {rec.get('kernel')}, source commit {rec.get('commit', 'n/a')})"
                           if traffic is not None else None)
        except Exception:
            traffic = None

    # read-only HBM ceiling of this box over the same buffer (relay_read_probe,
    # a measurement utility): K1's fraction is also quoted against it
    read_gbs = None
    if not args.profile:
        probe_out = relay.read_probe(logits)
        for _ in range(2):
            relay.read_probe(logits, out=probe_out)
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0.record(stream)
        for _ in range(5):
            relay.read_probe(logits, out=probe_out)
        r1.record(stream)
        torch.cuda.synchronize()
        read_gbs = logits.numel() * logits.element_size() // 16 * 16 * 5 / (r0.elapsed_time(r1) / 1e3) / 1e9
        if world > 1:
            t = torch.tensor([read_gbs], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            read_gbs = float(t[0])

    e2e = None
    if not args.no_e2e and not args.profile:
        e2e = measure_e2e(args, relay, an, cs, logits, ts, dev, world, rank, h6, T_job,
                          traj_rows=(T // n_my) if args.config == "c4" else None)
    cpu = None
    if rank == 0 and not args.no_baseline and not args.profile:
        cpu = cpu_baseline(logits, ts, cs_h, dtype, vocab)
    decode = None
    if rank == 0 and not args.no_decode and not args.profile:
        decode = measure_decode(relay, synth, dev, peak)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if (args.shard == "rows" or args.config == "c4") else "weak",
            "vs_baseline": None, "dtype": dtype,
            "data": "synthetic",
            "config": {"workload": (f"{args.config}: one {T_job}-token trajectory split at safe cuts over {world} "
                                    f"ranks x {vocab}-vocab " if args.shard == "rows" else
                                    f"c4: the fixed corpus of {T_job // (T // n_my)} trajectories x {T // n_my} "
                                    f"tokens ({T_job} rows) sharded by trajectory over {world} ranks x {vocab}-vocab "
                                    if args.config == "c4" else
                                    f"{args.config}: {world} x one {T}-token trajectory x {vocab}-vocab ") +
                       f"{dtype} logits (Qwen3-32B shape), {c['n_cues']} cues / {c['n_pat']} patterns, "
                       "margin+cue-scan+segment-reduce+stats (H1-H7)" +
                       (", row ranges at sentence starts" if args.shard == "rows" else
                        f", {n_my} trajectories on rank 0" if args.config == "c4" else ", one trajectory per rank"),
                       "rows_per_rank": T, "vocab": vocab,
                       "l2": (f"inputs {T * (vocab * esz) / 1e9:.2f} GB/rank >> 126 MB L2, no flush" if n_rot == 1 else
                              f"inputs {in_bytes / 1e9:.3f} GB/rank < 4 x L2: {n_rot} rotating copies "
                              f"({n_rot * in_bytes / 1e9:.2f} GB), a different one each step"),
                       "parallelism": f"dp{world} " + ("(one trajectory, row-range-sharded at safe cuts)"
                                                      if args.shard == "rows" else "(trajectory-sharded)"),
                       "allreduce": (args.allreduce if world > 1 else None)},
            "hbm_gbs_step": (T_job * (vocab * esz + 17)) / (ms / 1e3 / args.steps) / 1e9 / world,
            "roofline": {"kernel": "relay_margin_rows (K1)", "bound": "hbm", "achieved": achieved,
                         "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "traffic_source": traffic_src,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)" if pk.get("hbm_gbs") else "fallback",
                         "peak_note": ("the copy peak counts the read and the write bytes of a device-to-device "
                                       "copy; K1 only reads, so it can exceed it (frac > 1): frac_of_read_peak is "
                                       "against the read-only ceiling measured in this run"),
                         "frac_of_8TBs": achieved / 8000.0, "k1_ms": k1_ms,
                         "k1_share_of_step": k1_ms / (ms / args.steps),
                         "algorithmic_bytes_per_launch": k1_bytes,
                         "read_peak_gbs": read_gbs,
                         "frac_of_read_peak": (achieved / read_gbs) if read_gbs else None,
                         "read_peak_source": "relay_read_probe (TMA bulk copies into a 3 x 32 KB ring, "
                                             "2 CTAs per SM, no compute) over this run's logits buffer, 5 passes"},
            "gpu_launches": an.n_launches() * args.steps,
            "clocks": ck,
            "sustained": sustained,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "decode_step": decode,
        }
        print(json.dumps(line), flush=True)
    if xchg is not None:
        dist.barrier()
        xchg.close()
    cs.destroy()
    if world > 1:
        dist.destroy_process_group()


def run_c5(args):
    """configs[4]: per rank 8 trajectories x 16,384 tokens (64 at N = 8), 32
    cue patterns of length 1-6; each step streams the 131,072 logit rows in
    --chunk-rows chunks from a ~10 GB pool of pre-generated chunk buffers (>>
    L2: every chunk streams from HBM; the 318 GB corpus never exists at once)
    through Analyzer.run_streamed (K1 per chunk, K2 on a side stream, K3 +
    H6 once), then the table to the host and H7."""
    import torch
    import torch.distributed as dist

    import paper_2602_06454_b200 as relay
    import synth
    from paper_2602_06454_b200.dist import allreduce_stats
    rank, world, local = dist_env()
    if os.environ.get("RELAY_BENCH_SAME_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)
    c = synth.CONFIGS["c5"]
    V, L, NT = c["vocab"], c["traj_len"], 8
    R = args.chunk_rows                                   # rows per chunk (divides 8 x 16,384)
    K = max(2, int(10e9 // (R * V * 2)))                  # pool of ~10 GB >> L2
    cs_h = synth.make_cueset(V, c["n_cues"], c["n_pat"], max_len=c["max_len"], min_len=1)
    cs = relay.CueSet.from_synth(cs_h)
    ts = synth.make_tokens(NT, L, cs_h, seed=synth.BASE_SEED + 5 + rank)
    n = ts.tokens.shape[0]
    pool = [synth.make_logits(R, V, "bf16", seed=synth.BASE_SEED + 1000 * rank + i, device=dev) for i in range(K)]
    tok = torch.as_tensor(ts.tokens, device=dev)
    offs = torch.as_tensor(ts.traj_offsets, device=dev)
    tep = torch.as_tensor(ts.think_end_pos, device=dev)
    xchg = relay.StatsExchange(cs.n_cues) if (world > 1 and args.allreduce == "p2p") else None
    an = relay.Analyzer(cs, n, V, dev, rank=rank, world_size=world, exchange=xchg)
    stream = torch.cuda.current_stream()
    host_stats = torch.empty(an.stats.shape, dtype=torch.int64, pin_memory=True)
    k1_ev = []

    def step(timed=False):
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) if timed else None
        an.run_streamed(((i * R, pool[i % K]) for i in range(n // R)), tok, offs, tep, k1_events=ev)
        if timed:
            k1_ev.append(ev)
        if world > 1 and xchg is None:
            allreduce_stats(an.stats, cs.n_cues, world)
        host_stats.copy_(an.stats, non_blocking=True)
        stream.synchronize()
        relay.stats_finalize(host_stats.numpy(), cs.n_cues, world)

    for _ in range(args.warmup):
        step()
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        step(timed=True)
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ck = clocks.stop()
    ms = t0.elapsed_time(t1)
    k1_ms = statistics.mean(a.elapsed_time(b) for a, b in k1_ev)
    if world > 1:
        t = torch.tensor([ms, k1_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, k1_ms = float(t[0]), float(t[1])
    pk = peaks()
    peak = pk.get("hbm_gbs") or 6650.0
    k1_bytes = n * (V * 2 + 17)
    achieved = k1_bytes / (k1_ms / 1e3) / 1e9
    cpu = None
    if rank == 0 and not args.no_baseline:
        cpu = cpu_baseline(pool[0], ts, cs_h, "bf16", V)   # chunk 0 = pool[0] = rows 0..R-1
    if rank == 0:
        line = {
            "metric": METRIC, "value": n * world * args.steps / (ms / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic",
            "config": {"workload": f"c5: {world} x {NT} trajectories x {L} tokens x {V}-vocab bf16 logits streamed "
                                   f"in {R}-row chunks from a {K}-buffer pool, {c['n_cues']} cues / "
                                   f"{c['n_pat']} patterns of length 1-{c['max_len']}, H1-H7",
                       "rows_per_rank": n, "vocab": V,
                       "l2": f"chunk pool {K * R * V * 2 / 1e9:.1f} GB >> 126 MB L2, no flush",
                       "parallelism": f"dp{world} (trajectory-sharded)",
                       "allreduce": (args.allreduce if world > 1 else None)},
            "roofline": {"kernel": "relay_margin_rows (K1), all chunks of a step", "bound": "hbm",
                         "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": None, "k1_ms": k1_ms, "k1_share_of_step": k1_ms / (ms / args.steps),
                         "algorithmic_bytes_per_launch": k1_bytes // (n // R),
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)" if pk.get("hbm_gbs") else "fallback"},
            "gpu_launches": (n // R + 4) * args.steps,
            "clocks": ck,
            "e2e": None,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if xchg is not None:
        dist.barrier()
        xchg.close()
    cs.destroy()
    if world > 1:
        dist.destroy_process_group()


def measure_decode(relay, synth, dev, peak, B=256, V=152064, reps=30):
    """H8 on configs[2] (256 live rows x 152,064 bf16 per step): relay_step_switch
    (K4) and relay_step_sample (K4 + K5, T 0.6 / top-p 0.95 / top-k 20; and
    without top-k, + K6), each as a CUDA graph over 7 rotating logits buffers
    (> 4 x L2), device-timed; "hot" repeats one buffer (L2-resident)."""
    import torch
    h = synth.make_cueset(V, 8, 12, max_len=3)
    cs = relay.CueSet.from_synth(h)
    bufs = [synth.make_logits(B, V, "bf16", seed=100 + i, device=dev) for i in range(7)]
    state = torch.zeros(B, dtype=torch.uint8, device=dev)
    hist = torch.full((B, 7), -1, dtype=torch.int32, device=dev)
    small = torch.zeros(B, dtype=torch.int32, device=dev)
    samp = torch.randint(3000, V, (B,), dtype=torch.int32, device=dev)
    uni = torch.rand(B, device=dev)
    ws = relay.workspace(0, 0, B, dev)
    res = {"workload": f"configs[2]: {B} live rows x {V} bf16 per step, 7 rotating buffers",
           "bytes_per_step": B * (V * 2 + 12)}
    for name, fn in (("switch", lambda x, o: relay.step_switch(cs, x, state, hist, small, samp, ws=ws, out=o)),
                     ("sample", lambda x, o: relay.step_sample(cs, x, uni, state, hist, small, ws=ws, out=o)),
                     ("sample_no_top_k", lambda x, o: relay.step_sample(cs, x, uni, state, hist, small, top_k=0,
                                                                         ws=ws, out=o))):
        out = fn(bufs[0], None)
        s = torch.cuda.Stream(device=dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            for x in bufs:
                fn(x, out)
            torch.cuda.synchronize(dev)
            with torch.cuda.graph(g, stream=s):
                for x in bufs:
                    fn(x, out)
        torch.cuda.synchronize(dev)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize(dev)
        us = e0.elapsed_time(e1) * 1e3 / (reps * len(bufs))
        gbs = res["bytes_per_step"] / (us * 1e-6) / 1e9
        # "hot": the same buffer every step (L2-resident, as right after the LM-head GEMM)
        gh = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(gh, stream=s):
                for _ in bufs:
                    fn(bufs[0], out)
        torch.cuda.synchronize(dev)
        gh.replay()
        torch.cuda.synchronize(dev)
        e0.record()
        for _ in range(reps):
            gh.replay()
        e1.record()
        torch.cuda.synchronize(dev)
        us_hot = e0.elapsed_time(e1) * 1e3 / (reps * len(bufs))
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        mufu_peak = 16 * sms * 1.965e9          # MUFU.EX2 per second at the max SM clock
        res[name] = {"us_per_step": us, "rows_per_s": B / (us * 1e-6), "gbs": gbs, "frac": gbs / peak,
                     "us_per_step_hot": us_hot,
                     # K4 needs one exp per element: the SFU (MUFU) roofline of the margin pass
                     "mufu": {"bound": "alu", "achieved_gexp_s": B * V / (us * 1e-6) / 1e9,
                              "peak_gexp_s": mufu_peak / 1e9, "frac": B * V / (us * 1e-6) / mufu_peak,
                              "peak_source": "16 MUFU.EX2/clk/SM x SMs x 1965 MHz (guide unit counts)"},
                     "kernels": "K4" if name == "switch" else "K4 + K5",
                     "sampling": {"switch": "token given", "sample": "T 0.6, top-p 0.95, top-k 20 (Qwen3)",
                                  "sample_no_top_k": "T 0.6, top-p 0.95 (R1-Distill)"}[name]}
    del bufs
    cs.destroy()
    return res


def measure_e2e(args, relay, an, cs, logits, ts, dev, world, rank, h6, rows_job, traj_rows=None):
    """Same metric through the public API with HOST inputs: every step copies the
    step's logits + tokens from pinned host memory, runs the pass, and reads the
    statistics table back.  With more than one trajectory per rank (c4) the
    logits are streamed from the host one trajectory at a time (a one-
    trajectory pinned buffer sent for each of the rank's trajectories, K1 per
    trajectory through Analyzer.run_streamed): host memory holds 10 GB, not
    the rank's whole shard."""
    import torch
    import torch.distributed as dist

    T, V = logits.shape
    if traj_rows and T > traj_rows:
        return measure_e2e_streamed(args, relay, an, cs, logits, ts, dev, world, h6, rows_job, traj_rows)
    pinned = True
    try:
        h_logits = torch.empty((T, V), dtype=logits.dtype, pin_memory=True)
    except RuntimeError:   # pinned host memory exhausted (e.g. 8 ranks x 10 GB): pageable copies
        pinned = False
        h_logits = torch.empty((T, V), dtype=logits.dtype)
    h_logits.copy_(logits)
    h_tok = torch.from_numpy(ts.tokens.copy()).pin_memory()
    h_offs = torch.from_numpy(ts.traj_offsets.copy()).pin_memory()
    d_logits = torch.empty_like(logits)
    d_tok = torch.empty(T, dtype=torch.int32, device=dev)
    d_offs = torch.empty(h_offs.shape, dtype=torch.int64, device=dev)
    host_stats = torch.empty(an.stats.shape, dtype=torch.int64, pin_memory=True)
    stream = torch.cuda.current_stream()

    def step():
        d_logits.copy_(h_logits, non_blocking=True)
        d_tok.copy_(h_tok, non_blocking=True)
        d_offs.copy_(h_offs, non_blocking=True)
        an.run(d_logits, d_tok, d_offs)
        if world > 1:
            h6(an.stats)
        host_stats.copy_(an.stats, non_blocking=True)
        stream.synchronize()
        relay.stats_finalize(host_stats.numpy(), cs.n_cues, world)

    step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.e2e_steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
    bi = h_logits.numel() * h_logits.element_size() + h_tok.numel() * 4 + h_offs.numel() * 8
    bo = host_stats.numel() * 8
    del h_logits, d_logits
    torch.cuda.empty_cache()
    return {"value": rows_job * args.e2e_steps / (ms / 1e3), "unit": UNIT,
            "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo, "steps": args.e2e_steps,
            "pinned": pinned,
            "path": "host logits+tokens -> H2D -> Analyzer.run (C ABI) -> D2H stats -> finalize"}


def measure_e2e_streamed(args, relay, an, cs, logits, ts, dev, world, h6, rows_job, R):
    import torch
    import torch.distributed as dist
    T, V = logits.shape
    pinned = True
    try:
        h_chunk = torch.empty((R, V), dtype=logits.dtype, pin_memory=True)
    except RuntimeError:
        pinned = False
        h_chunk = torch.empty((R, V), dtype=logits.dtype)
    h_chunk.copy_(logits[:R])
    h_tok = torch.from_numpy(ts.tokens.copy()).pin_memory()
    h_offs = torch.from_numpy(ts.traj_offsets.copy()).pin_memory()
    h_tep = torch.from_numpy(ts.think_end_pos.copy()).pin_memory()
    d_buf = [torch.empty((R, V), dtype=logits.dtype, device=dev) for _ in range(2)]
    d_tok = torch.empty(T, dtype=torch.int32, device=dev)
    d_offs = torch.empty(h_offs.shape, dtype=torch.int64, device=dev)
    d_tep = torch.empty(h_tep.shape, dtype=torch.int64, device=dev)
    host_stats = torch.empty(an.stats.shape, dtype=torch.int64, pin_memory=True)
    stream = torch.cuda.current_stream()

    def chunks():
        for k in range(T // R):
            d_buf[k % 2].copy_(h_chunk, non_blocking=True)
            yield k * R, d_buf[k % 2]

    def step():
        d_tok.copy_(h_tok, non_blocking=True)
        d_offs.copy_(h_offs, non_blocking=True)
        d_tep.copy_(h_tep, non_blocking=True)
        an.run_streamed(chunks(), d_tok, d_offs, d_tep)
        if world > 1:
            h6(an.stats)
        host_stats.copy_(an.stats, non_blocking=True)
        stream.synchronize()
        relay.stats_finalize(host_stats.numpy(), cs.n_cues, world)

    step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.e2e_steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
    bi = (T // R) * h_chunk.numel() * h_chunk.element_size() + h_tok.numel() * 4 + h_offs.numel() * 8 + \
        h_tep.numel() * 8
    bo = host_stats.numel() * 8
    del h_chunk, d_buf
    torch.cuda.empty_cache()
    return {"value": rows_job * args.e2e_steps / (ms / 1e3), "unit": UNIT,
            "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo, "steps": args.e2e_steps, "pinned": pinned,
            "path": "host logits (one pinned trajectory buffer, sent once per trajectory of the shard) + "
                    "tokens -> H2D -> Analyzer.run_streamed (C ABI, K1 per trajectory) -> D2H stats -> finalize"}


def measure_sustained(args, step_ms, run_steps, k1_ev, local, world, dev, T, T_job, vocab, esz):
    """Back-to-back steps for ~args.sustained_s seconds after the timed region,
    clocks sampled throughout: the rate once the SM clock has settled under
    the kernel's own power draw (the driver's burst line is ~30 ms)."""
    import torch
    import torch.distributed as dist
    n = max(3, int(args.sustained_s * 1e3 / max(step_ms, 1e-3)))
    if world > 1:
        t = torch.tensor([n], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        n = int(t[0])
    k1_ev.clear()
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.2)
    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    run_steps(n, timed=True)
    t1.record(stream)
    torch.cuda.synchronize()
    ck = clocks.stop()
    ms = t0.elapsed_time(t1)
    # the settled part: the last half of the launches
    k1 = [a.elapsed_time(b) for a, b in k1_ev]
    k1_ms = statistics.mean(k1[len(k1) // 2:])
    if world > 1:
        t = torch.tensor([ms, k1_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, k1_ms = float(t[0]), float(t[1])
    gbs = T * (vocab * esz + 17) / (k1_ms / 1e3) / 1e9
    return {"seconds": ms / 1e3, "steps": n, "value": T_job * n / (ms / 1e3), "unit": UNIT,
            "k1_ms_settled": k1_ms, "k1_gbs_settled": gbs, "k1_frac_of_8TBs": gbs / 8000.0,
            "clocks": ck,
            "note": "K1 mean over the second half of the launches; clocks sampled over the whole run"}


def cpu_baseline(logits, ts, cs_h, dtype, vocab):
    """The oracle as it stands on this host's cores, on a bounded contiguous
    sample of the same workload (~10-20 s of CPU work)."""
    import synth
    threads = cpu_threads()
    host8 = synth.host_rows(logits[:8], dtype)
    t0 = time.perf_counter()
    oracle_pass(host8, dtype, vocab, ts.tokens[:8], None, cs_h, 1)
    per_row = (time.perf_counter() - t0) / 8
    S = int(min(logits.shape[0], max(threads, 12.0 * threads / max(per_row, 1e-9))))
    host = synth.host_rows(logits[:S], dtype)
    toks = np.ascontiguousarray(ts.tokens[:S])
    t0 = time.perf_counter()
    oracle_pass(host, dtype, vocab, toks, None, cs_h, threads)
    dt = time.perf_counter() - t0
    return {"value": S / dt, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"first {S} rows (+ their tokens) of the rank-0 trajectory, full H1-H7 oracle pass, "
                      f"{dt:.1f} s"}


if __name__ == "__main__":
    main()
