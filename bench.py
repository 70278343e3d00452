"""Benchmark: resampled tokens/s and HBM roofline fraction of the fused
logits-cache re-sampling path (lookup -> step-wise speculative resample ->
accept), vs the reference CPU path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

N > 1 runs under torchrun, one process per GPU (weak scaling: every rank owns
its own requests/trees and cache shard; NCCL only reduces statistics after the
timed region).  Default workload = BASELINE.json configs[1] (C2):
Best-of-N re-sampling, V = 32000, 256 requests x N = 32 branches,
temperature 0.6 + top-p 0.9, bf16 rows, one 500-row cached trajectory per
request (8.2 GB slab, larger than L2, so no flush is needed between steps).
A step = for every request: hash lookup, resample of every cached position
for all 32 branches (u = RngStream(branch seed) at draw number = position,
engine.py:301-310), and the step-wise acceptance.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs, as resample workloads over HBM-resident cached trajectories:
    # n_req entries (tree nodes / requests), R cached rows each, nb draws per row (siblings)
    "c1": dict(V=32000, n_req=120, nb=1, R=500, T=0.6, k=0, p=1.0, dtype="float32", scaling="weak",
               desc="ToT re-sampling, vocab 32000, 16 branches x depth 8 (120 revisits x 500 cached rows), "
                    "fp32, T 0.6, top-p 1"),
    "c2": dict(V=32000, n_req=256, nb=32, R=500, T=0.6, k=0, p=0.9, dtype="bfloat16", scaling="weak",
               desc="Best-of-N re-sampling, vocab 32000, 256 requests x N=32, T 0.6 + top-p 0.9, bf16"),
    "c3": dict(V=151936, n_req=1024, nb=1, R=16, T=0.6, k=50, p=0.95, dtype="bfloat16", scaling="weak",
               desc="vocab 151936, 1024 concurrent branches (16-row entries, all hits), top-k 50 + top-p 0.95, bf16"),
    "c5": dict(V=151936, n_req=8 * 512, nb=1, R=4, T=0.6, k=50, p=0.95, dtype="bfloat16", scaling="strong",
               desc="multi-agent: 8 trees x 512 branches (4 cached rows each), vocab 151936, top-k 50 + "
                    "top-p 0.95, bf16; trees sharded tree i -> GPU i mod G"),
    "c4": dict(V=128256, keys=1 << 20, entries=400_000, batch=8192, ins_frac=0.9, dtype="bfloat16",
               scaling="weak", desc="cache capacity/eviction stress: 1M prefix digests (tree expansion), one "
                                    "V=128256 bf16 row per entry, slab of up to 400k rows, 90% insert / "
                                    "10% lookup batches"),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------------ our arm


def setup_workload(cfg, dev, rank, world=1):
    import torch

    import paper_2604_17353_b200 as lcb
    from paper_2604_17353_b200 import _capi, _dev
    from paper_2604_17353_b200.mixing import mix2

    V, n_req, nb, R = cfg["V"], cfg["n_req"], cfg["nb"], cfg["R"]
    bf16 = cfg["dtype"] == "bfloat16"
    slab_bytes = n_req * R * V * (2 if bf16 else 4)
    budget = n_req * R * (V * 4 + 8) + 1024
    cache = lcb.LogitsCache(budget, vocab=V, dtype=cfg["dtype"], key_capacity=n_req + 64, page_rows=min(R, 16),
                            max_rows=R, device=dev)
    # prompts: one per request (tree root), digests from the GPU hasher
    prompts = [[rank % 256, r % 256, r // 256] + [(rank * 7919 + r * 31 + i) % 256 for i in range(46 + r % 32)]
               for r in range(n_req)]  # unique per (rank, request)
    digests = lcb.hash_prompts(prompts, dev=dev)
    # synthetic rows from the reference producer (model seed 7, conc 2.5, range 5), per request chunk
    chunk = max(1, (1 << 30) // (R * V * (2 if bf16 else 4)))
    tdt = torch.bfloat16 if bf16 else torch.float32
    ws = lcb.sampling.Workspace(dev)
    for r0 in range(0, n_req, chunk):
        rn = min(chunk, n_req - r0)
        states = lcb._dev.u64_tensor([mix2(7, (rank << 40) + (r0 + i) * R + t) for i in range(rn) for t in range(R)],
                                     dev)
        rows = torch.empty((rn * R, V), dtype=tdt, device=dev)
        _capi.check(_capi.lib.lc_fill_logits(states.data_ptr(), rn * R, V, 2.5, 5.0,
                                             _capi.LC_BF16 if bf16 else _capi.LC_F32, rows.data_ptr(), V,
                                             _dev.stream_ptr(dev)))
        # the cached continuation = one sampled trajectory of these rows (first branch's seed family)
        tasks = lcb.make_tasks(row=np.arange(rn * R), pos=np.tile(np.arange(R), rn), temperature=cfg["T"],
                               top_k=cfg["k"], top_p=cfg["p"], draw_begin=np.arange(rn * R),
                               draw_end=np.arange(rn * R) + 1, seed_base=np.repeat(np.arange(rn), R))
        seeds0 = lcb._dev.u64_tensor([mix2(99, (rank << 32) + r0 + i) for i in range(rn)], dev)
        tok, _ = lcb.resample(rows, tasks, seeds=seeds0, n_draws=rn * R)
        lens = torch.full((rn,), R, dtype=torch.int32, device=dev)
        vocs = torch.full((rn,), V, dtype=torch.int32, device=dev)
        offs = torch.arange(rn, dtype=torch.int64, device=dev) * R
        cache.insert_batch(digests[r0:r0 + rn], lens, vocs, rows, offs, tok.contiguous(), R)
        del rows
    torch.cuda.synchronize(dev)
    st = cache._stats()
    assert st.entries == n_req, (st.entries, n_req)
    seeds = lcb._dev.u64_tensor([mix2(1, (rank << 32) + b) for b in range(n_req * nb)], dev)
    T = torch.full((n_req,), cfg["T"], dtype=torch.float64, device=dev)
    K = torch.full((n_req,), cfg["k"], dtype=torch.int32, device=dev)
    P = torch.full((n_req,), cfg["p"], dtype=torch.float64, device=dev)
    return dict(cache=cache, prompts=prompts, digests=digests, seeds=seeds, T=T, K=K, P=P, slab_bytes=slab_bytes,
                bufs={})


def workload_config(args, cfg, world):
    """The ``config`` object of a resample bench line -- identical for our arm and the
    reference arm (same workload, same keys)."""
    n_req = cfg["n_req"]
    if cfg["scaling"] == "strong":
        from paper_2604_17353_b200.shard import local_trees

        n_req = len(local_trees(8, 0, world)) * (cfg["n_req"] // 8)
    esz = 2 if cfg["dtype"] == "bfloat16" else 4
    return {"workload": cfg["desc"], "config": args.config, "vocab": cfg["V"], "requests_per_gpu": n_req,
            "branches": cfg["nb"], "rows_per_entry": cfg["R"], "draws_per_row": cfg["nb"], "temperature": cfg["T"],
            "top_k": cfg["k"] or None, "top_p": cfg["p"], "slab_gb_per_gpu": n_req * cfg["R"] * cfg["V"] * esz / 1e9,
            "l2": "inputs larger than L2 (slab re-read every step)", "parallelism": f"tree-sharded x{world}",
            "replay_policy": args.policy,
            **({"hotspot_decay": 0.001, "hotspot_threshold": 0.6} if args.policy == "hotspot" else {})}


def traffic_per_launch(cfg, n_rows):
    """DRAM bytes (read + write) of one resample launch, from the committed ncu --set full captures
    of the bench launches (profiles/r2_traffic.json: bytes per row of the stage / row-warp / wide
    kernel), or None for a shape without a capture."""
    f = os.path.join(ROOT, "profiles", "r2_traffic.json")
    if not os.path.exists(f):
        return None
    with open(f) as fh:
        d = json.load(fh)
    key = ("c2" if cfg["dtype"] == "bfloat16" else "c1") if cfg["V"] <= 32000 else "c3"
    if key == "c3" and cfg["dtype"] != "bfloat16":
        return None
    return d[key]["dram_bytes_per_row"] * n_rows if key in d else None


def run_ours(args, cfg, rank, world, dev):
    import torch
    import torch.distributed as dist

    import paper_2604_17353_b200 as lcb

    sim = getattr(args, "one_rank_of", None)  # measure one rank's share of a G-GPU run on this GPU
    pw = sim or world
    if cfg["scaling"] == "strong":  # trees sharded across ranks: tree i -> rank i % world
        from paper_2604_17353_b200.shard import local_trees

        cfg = dict(cfg)
        n_trees = 8
        per_tree = cfg["n_req"] // n_trees
        cfg["n_req"] = len(local_trees(n_trees, rank if not sim else 0, pw)) * per_tree
    w = setup_workload(cfg, dev, rank, world)
    cache = w["cache"]
    V, n_req, nb, R = cfg["V"], cfg["n_req"], cfg["nb"], cfg["R"]
    esz = 2 if cfg["dtype"] == "bfloat16" else 4
    counters = torch.zeros(8, dtype=torch.int64, device=dev)
    n_rows = n_req * R
    n_draws = n_rows * nb

    # instrument the dominant kernel: CUDA events around the resample call, on its stream
    ev = []
    orig = lcb.sampling.resample

    def timed_resample(*a, **kw):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        r = orig(*a, **kw)
        e.record()
        ev.append((s, e))
        return r

    hot_rows = n_rows
    if args.policy == "hotspot":  # ReplayPolicy.HOTSPOT: hotspots per entry (memoised, untimed like the reference)
        # hotspot scores kept beside the rows + selection on the device (lc_cache_score_rows /
        # lc_cache_hotspots), no row or score leaves the GPU
        hp = lcb.HotspotParams(decay=0.001, threshold=0.6)
        slot0, gen0, _, _ = cache.lookup_batch(w["digests"])
        d_di, n_hot, hs_flags = cache.hotspot_draw_index_device(slot0, gen0, R, cfg["T"], hp)
        hot_l = cache.hotspot_list(d_di)
        hot_rows = int(n_hot.sum().item())
        hotspot_uncertain = int((hs_flags & 1).sum().item())

        def step():
            return cache.replay_hotspot(w["digests"], R, nb, w["seeds"], w["T"], w["K"], w["P"], counters=counters,
                                        bufs=w["bufs"], draw_index=d_di, hot_list=hot_l)
    else:
        def step():
            return cache.replay_stepwise(w["digests"], R, nb, w["seeds"], w["T"], w["K"], w["P"],
                                         counters=counters, bufs=w["bufs"])

    graph = None
    if args.graph:
        # capture one whole step (lookup -> tasks -> resample -> cached tokens -> acceptance, ~8
        # launches, no host sync) in a CUDA graph: small per-rank batches (C5 at G=8: 2048 rows per
        # GPU) are otherwise bound by launch latency and Python glue.  The dominant kernel's time
        # is still taken from eager launches (events cannot be read inside a graph).
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize(dev)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            g_out = step()
        eager_step = step

        def step():
            graph.replay()
            return g_out

    lcb.sampling.resample = timed_resample
    try:
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize(dev)
        if graph is not None:  # eager launches for the kernel-time share
            for _ in range(args.steps):
                eager_step()
            torch.cuda.synchronize(dev)
            k_ev = list(ev)
        ev.clear()
        counters.zero_()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        prof = os.environ.get("LCB_PROFILE_TIMED") == "1"  # ncu --profile-from-start off: timed steps only
        with ClockSampler(dev.index) as clk:
            if prof:
                torch.cuda.profiler.start()
            t0.record()
            for _ in range(args.steps):
                tok, rep, div, slot, ln = step()
            t1.record()
            torch.cuda.synchronize(dev)
            if prof:
                torch.cuda.profiler.stop()
        if world > 1:
            dist.barrier()
        ms = t0.elapsed_time(t1)
        k_ms = [s.elapsed_time(e) for s, e in (k_ev if graph is not None else ev)]
    finally:
        lcb.sampling.resample = orig
    accepted = int(rep.sum().item()) * args.steps
    cnt = counters.cpu().numpy()

    # ---- e2e through the public API with host buffers (hash from host prompts, tokens back to host)
    pin_tok = torch.empty(n_draws, dtype=torch.int32, pin_memory=True)
    pin_rep = torch.empty(n_req * nb, dtype=torch.int32, pin_memory=True)
    flat = np.concatenate([np.asarray(p, dtype=np.int32) for p in w["prompts"]])
    offs = np.zeros(n_req + 1, dtype=np.int64)
    np.cumsum([len(p) for p in w["prompts"]], out=offs[1:])
    h_tok = torch.from_numpy(flat).pin_memory()
    h_off = torch.from_numpy(offs).pin_memory()
    h_seed = w["seeds"].cpu().pin_memory()
    d_tok = torch.empty_like(h_tok, device=dev)
    d_off = torch.empty_like(h_off, device=dev)
    d_seed = torch.empty_like(h_seed, device=dev)
    d_dig = torch.empty(n_req, dtype=torch.int64, device=dev)
    from paper_2604_17353_b200 import _capi, _dev

    # two buffer sets: step i's tokens go back to the host on a copy stream while
    # step i+1 computes (double-buffered outputs, as a serving loop would run)
    pin_toks = [pin_tok, torch.empty(n_draws, dtype=torch.int32, pin_memory=True)]
    pin_reps = [pin_rep, torch.empty(n_req * nb, dtype=torch.int32, pin_memory=True)]
    bufsets = [w["bufs"], {}]
    copy_stream = torch.cuda.Stream(dev)
    ev_copy = [None, None]

    def e2e_step(i):
        k = i % 2
        main = torch.cuda.current_stream(dev)
        if ev_copy[k] is not None:
            main.wait_event(ev_copy[k])  # buffer set k's previous copy-out is done
        d_tok.copy_(h_tok, non_blocking=True)
        d_off.copy_(h_off, non_blocking=True)
        d_seed.copy_(h_seed, non_blocking=True)
        _capi.check(_capi.lib.lc_hash_prefix(d_tok.data_ptr(), d_off.data_ptr(), None, n_req, d_dig.data_ptr(),
                                             _dev.stream_ptr(dev)))
        if args.policy == "hotspot":
            tok, rep, div, slot, ln = cache.replay_hotspot(d_dig, R, nb, d_seed, w["T"], w["K"], w["P"],
                                                           bufs=bufsets[k], draw_index=d_di, hot_list=hot_l)
        else:
            tok, rep, div, slot, ln = cache.replay_stepwise(d_dig, R, nb, d_seed, w["T"], w["K"], w["P"],
                                                            bufs=bufsets[k])
        done = torch.cuda.Event()
        done.record(main)
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(done)
            pin_toks[k].copy_(tok, non_blocking=True)
            pin_reps[k].copy_(rep, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy_stream)
            ev_copy[k] = ev

    for i in range(2):
        e2e_step(i)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.steps):
        e2e_step(i)
    for ev in ev_copy:
        if ev is not None:
            torch.cuda.current_stream(dev).wait_event(ev)
    e1.record()
    torch.cuda.synchronize(dev)
    e2e_ms = e0.elapsed_time(e1)
    h2d = h_tok.numel() * 4 + h_off.numel() * 8 + h_seed.numel() * 8
    d2h = n_draws * 4 + n_req * nb * 4

    # ---- max over ranks, sums over ranks
    from paper_2604_17353_b200.shard import reduce_stats

    times = torch.tensor([ms, e2e_ms], dtype=torch.float64, device=dev)
    counts = torch.tensor([float(accepted), float(cnt[0]), float(cnt[1]), float(cnt[2]), float(cnt[3])],
                          dtype=torch.float64, device=dev)
    times, counts = reduce_stats(times, counts, world)  # NCCL: max of times, sum of counters
    ms, e2e_ms = float(times[0]), float(times[1])
    accepted, precise, unresolved, bad, exact = (int(x) for x in counts.tolist())
    if rank != 0:
        return None
    tokens_total = (n_draws * args.steps * world if cfg["scaling"] == "weak" or sim
                    else CONFIGS[args.config]["n_req"] * R * nb * args.steps)
    if args.policy == "hotspot":  # only hotspot positions draw
        tokens_total = hot_rows * nb * args.steps * world
    peak, peak_src = peaks()
    algo_bytes_launch = hot_rows * V * esz + hot_rows * nb * 20  # V*s per unique row + 20 B per draw
    k_avg = sum(k_ms) / max(len(k_ms), 1)
    achieved = algo_bytes_launch / (k_avg * 1e-3) / 1e9
    res = {
        "metric": "resampled_tokens_per_s",
        "value": tokens_total / (ms * 1e-3),
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms / args.steps,
        "higher_is_better": True,
        "scaling": cfg["scaling"],
        "vs_baseline": None,
        "dtype": "bf16" if esz == 2 else "f32",
        "data": "synthetic (reference producer fill_logits, seed 7, conc 2.5, range 5.0)",
        "config": {**workload_config(args, CONFIGS[args.config], world),
                   **({"hotspot_rows": hot_rows, "hotspot_uncertain_entries": hotspot_uncertain}
                      if args.policy == "hotspot" else {})},
        "accepted_tokens_per_s": accepted / (ms * 1e-3),
        "rows_per_s": (n_rows * world if cfg["scaling"] == "weak" or sim else CONFIGS[args.config]["n_req"] * R)
        * args.steps / (ms * 1e-3),
        "precise_tasks": precise,
        "exact_tasks": exact,
        "unresolved_draws": unresolved,
        "bad_rows": bad,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic_per_launch(cfg, hot_rows), "peak_source": peak_src,
                     "kernel": "lc_cache_resample (stage_kernel + resample_kernel requeue + exact_kernel)",
                     "kernel_ms_avg": k_avg, "algorithmic_bytes_per_launch": algo_bytes_launch},
        "e2e": {"value": tokens_total / (e2e_ms * 1e-3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                "d2h_overlap": "step i's tokens copied out on a second stream while step i+1 computes",
                "d2h_bytes_per_step": d2h},
        "gpu_launches": 8 * args.steps,
        "cuda_graph": graph is not None,
        **({"simulated_rank": {"of": sim, "rank": 0, "rows_per_step": n_rows,
                               "note": "one rank's share of a G-GPU run, measured alone on this GPU (ranks share "
                                       "nothing on the data path); value is that rank's throughput",
                               "aggregate_if_ranks_independent": tokens_total / (ms * 1e-3) * sim}}
           if sim else {}),
        "clocks": clk.summary(),
    }
    if not args.no_check and args.policy == "step_wise":
        res["check"] = run_check(args, cfg, w, rank, world, dev)
    if not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline(cfg, seconds=args.cpu_seconds)
    return res


def run_windowed(args, cfg, rank, world, dev):
    """C1/C2 step-wise replay in windows of ``--window`` positions (LogitsCache.replay_windowed):
    rows are resampled only while a branch of the request is still replaying, so the line's
    metric is ACCEPTED tokens/s (the replayed tokens the engine keeps, engine.py:296-331).  The
    full replay (resample every cached position, bench default) gives the same replayed_len /
    diverged_at; that equality is checked after the timed region."""
    import torch

    import paper_2604_17353_b200 as lcb

    w = setup_workload(cfg, dev, rank, world)
    cache = w["cache"]
    V, n_req, nb, R = cfg["V"], cfg["n_req"], cfg["nb"], cfg["R"]
    esz = 2 if cfg["dtype"] == "bfloat16" else 4
    counters = torch.zeros(8, dtype=torch.int64, device=dev)
    def step():
        slot, gen, ln, vv = cache.lookup_batch(w["digests"])
        tok, rep, div, nwin = cache.replay_windowed(slot, gen, ln, vv, R, nb, w["seeds"], w["T"], w["K"], w["P"],
                                                    window=args.window, counters=counters, bufs=w["bufs"])
        return tok, rep, div, nwin

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        t0.record()
        wins = 0
        for _ in range(args.steps):
            tok, rep, div, nwin = step()
            wins += nwin
        t1.record()
        torch.cuda.synchronize(dev)
    ms = t0.elapsed_time(t1)
    rep_w, div_w = rep.clone(), div.clone()
    accepted = int(rep_w.sum().item())
    rows_per_step = n_req * min(R, wins // args.steps * args.window)  # upper bound on rows resampled
    # equality with the full replay (untimed)
    _, rep_f, div_f, _, _ = cache.replay_stepwise(w["digests"], R, nb, w["seeds"], w["T"], w["K"], w["P"])
    same = bool(torch.equal(rep_f, rep_w) and torch.equal(div_f, div_w))
    if rank != 0:
        return None
    return {
        "metric": "accepted_tokens_per_s",
        "value": accepted * args.steps * world / (ms * 1e-3),
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms / args.steps,
        "higher_is_better": True,
        "scaling": cfg["scaling"],
        "vs_baseline": None,
        "dtype": "bf16" if esz == 2 else "f32",
        "data": "synthetic (reference producer fill_logits, seed 7, conc 2.5, range 5.0)",
        "config": {**workload_config(args, CONFIGS[args.config], world), "window": args.window},
        "accepted_tokens_per_step": accepted,
        "windows_per_step": wins / args.steps,
        "rows_resampled_per_step_max": rows_per_step,
        "equals_full_replay": same,
        "precise_tasks": int(counters[0].item()),
        "note": "windowed step-wise replay: same replayed_len/diverged_at as the full replay (checked); "
                "one host read of the live-branch count per window",
        "gpu_launches": None,
        "clocks": clk.summary(),
    }


# ------------------------------------------------------------------------ check leg (untimed)


def _pool_map(fn, jobs, cores):
    import multiprocessing as mp

    if cores <= 1 or len(jobs) <= 1:
        return [fn(j) for j in jobs]
    with mp.get_context("spawn").Pool(min(cores, len(jobs))) as pool:
        return pool.map(fn, jobs)


def run_check(args, cfg, w, rank, world, dev):
    """Validate whole steps against the oracle (oracle/bulk.py) on the host cores, after the
    timed region: S extra step-wise replay steps with fresh seed families, every token and every
    task's kept-set size recomputed by the oracle from the same rows and uniforms, the replay
    acceptance (replayed_len) recomputed from those tokens and the cached tokens, and (bf16
    slabs) one step cross-checked bit-for-bit against the non-staged kernels (LCB_NO_STAGE=1)."""
    import torch

    import paper_2604_17353_b200 as lcb
    from oracle import bulk
    from paper_2604_17353_b200.mixing import mix2

    t_start = time.perf_counter()
    cache = w["cache"]
    V, n_req, nb, R = cfg["V"], cfg["n_req"], cfg["nb"], cfg["R"]
    n_rows = n_req * R
    target = args.check_draws if args.check_draws is not None else (10_000_000 if V <= 32000 else 1_000_000)
    S = max(1, -(-target // (n_rows * nb)))
    toks, reps, seeds_all = [], [], []
    kept = torch.zeros(n_rows, dtype=torch.int32, device=dev)
    for s in range(S):
        seeds_h = [mix2(1 + s, (rank << 32) + b) for b in range(n_req * nb)]
        seeds = lcb._dev.u64_tensor(seeds_h, dev)
        tok, rep, div, slot, ln = cache.replay_stepwise(w["digests"], R, nb, seeds, w["T"], w["K"], w["P"],
                                                        bufs=w["bufs"], kept=kept if s == 0 else None)
        toks.append(tok.cpu().numpy().reshape(n_req, R, nb))
        reps.append(rep.cpu().numpy().reshape(n_req, nb))
        seeds_all.append(np.array(seeds_h, dtype=np.uint64).reshape(n_req, nb))
    kept_h = kept.cpu().numpy()
    cached = w["bufs"]["cached"].cpu().numpy()[: n_rows].reshape(n_req, R)
    # replay acceptance from the tokens (engine.py:301-310): first t with tok != cached, + 1
    acc_bad = 0
    for s in range(S):
        diff = toks[s] != cached[:, :, None]
        first = np.where(diff.any(1), diff.argmax(1) + 1, R)
        acc_bad += int((first != reps[s]).sum())
    # cross-check one step against the non-staged kernels, bit for bit
    cross = None
    if cfg["dtype"] == "bfloat16":
        os.environ["LCB_NO_STAGE"] = "1"
        try:
            seeds = lcb._dev.u64_tensor([mix2(1, (rank << 32) + b) for b in range(n_req * nb)], dev)
            k2 = torch.zeros(n_rows, dtype=torch.int32, device=dev)
            tok2 = cache.replay_stepwise(w["digests"], R, nb, seeds, w["T"], w["K"], w["P"], kept=k2)[0]
            t2 = tok2.cpu().numpy().reshape(n_req, R, nb)
            cross = {"path": "LCB_NO_STAGE=1 (row-warp / CTA kernels)", "draws": int(t2.size),
                     "token_mismatches": int((t2 != toks[0]).sum()),
                     "kept_mismatches": int((k2.cpu().numpy() != kept_h).sum())}
        finally:
            del os.environ["LCB_NO_STAGE"]
    cores = max(1, (os.cpu_count() or 1) // max(world, 1))
    states = np.array([mix2(7, (rank << 40) + i) for i in range(n_rows)], dtype=np.uint64)  # row r*R+t
    tok_rows = np.stack(toks, 2).reshape(n_rows, S * nb)  # [r, t] x [s, b]
    seed_rows = np.repeat(np.stack(seeds_all, 1).reshape(n_req, S * nb), R, axis=0)
    index = np.tile(np.arange(R), n_req)
    n_jobs = max(cores * 4, 1)
    bounds = np.linspace(0, n_rows, n_jobs + 1).astype(int)
    jobs = [dict(V=V, T=cfg["T"], k=cfg["k"] or None, p=cfg["p"], bf16=cfg["dtype"] == "bfloat16", conc=2.5,
                 states=states[a:b], seeds=seed_rows[a:b], index=index[a:b], tokens=tok_rows[a:b],
                 kept=kept_h[a:b], row_ids=np.arange(a, b))
            for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
    res = bulk.merge(_pool_map(bulk.check_rows, jobs, cores))
    res.update({"steps": S, "seed_families": S, "acceptance_mismatches": acc_bad, "cores": cores,
                "seconds": round(time.perf_counter() - t_start, 1), "cross_check": cross,
                "oracle": "oracle/bulk.py: sample(truncate(softmax(z,T),k,p)) per row (sampling.py:57-109), "
                          "rows from the reference producer, u = RngStream(seed) at draw number = position"})
    return res


# ------------------------------------------------------------------------ CPU (reference) arm


def _cpu_worker(a):
    """Reference per-draw path: sample(truncate(softmax(z, T), k, p), u) on rows of the workload,
    in steps: ``warmup`` calibration steps, then ``steps`` timed steps of a fixed draw count sized
    so one step takes about ``step_s`` seconds."""
    V, T, k, p, bf16, warmup, steps, step_s, wid = a
    sys.path.insert(0, ROOT)
    from oracle import mixing_ref, sampling_ref

    rng = np.random.default_rng(wid)
    rows = mixing_ref.fill_rows_np([mixing_ref.mix2(7, wid * 1000 + i) for i in range(16)], V, 2.5)
    if bf16:
        rows = mixing_ref.bf16_round(rows)
    n = [0]

    def run(count):
        for _ in range(count):
            z = rows[n[0] % len(rows)]
            q = sampling_ref.truncate(sampling_ref.softmax(z, T), k or None, p)
            sampling_ref.draw(q, float(rng.random()))
            n[0] += 1

    t0 = time.perf_counter()
    for _ in range(max(warmup, 1)):
        run(4)
    per_draw = (time.perf_counter() - t0) / (4 * max(warmup, 1))
    per_step = max(1, int(step_s / max(per_draw, 1e-9)))
    times = []
    for _ in range(steps):
        t = time.perf_counter()
        run(per_step)
        times.append(time.perf_counter() - t)
    return per_step, times


def _cpu_model():
    try:
        return [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    except Exception:
        return "unknown"


def cpu_baseline(cfg, seconds=12.0, cores=None, steps=1, warmup=1):
    """The oracle port on every host core: ``steps`` steps, each a bounded sample of the
    workload's draws (about seconds/steps of CPU time per worker).  Step time = max over
    workers; value = all workers' draws / the summed step times."""
    import multiprocessing as mp

    cores = cores or os.cpu_count() or 1
    args = [(cfg["V"], cfg["T"], cfg["k"], cfg["p"], cfg["dtype"] == "bfloat16", warmup, steps, seconds / steps, i)
            for i in range(cores)]
    with mp.get_context("spawn").Pool(cores) as pool:
        out = pool.map(_cpu_worker, args)
    step_times = [max(o[1][s] for o in out) for s in range(steps)]
    n = sum(o[0] * steps for o in out)
    t = sum(step_times)
    return {"value": n / t, "unit": "tokens/s", "cores": cores, "kind": "port",
            "ms_per_step": 1e3 * t / steps, "draws_per_step": n // steps,
            "sample": f"{steps} step(s) x {n // steps} draws of the workload's rows (V={cfg['V']}, T={cfg['T']}, "
                      f"top_k={cfg['k'] or None}, top_p={cfg['p']}; {cores} workers x {n // steps // cores} draws "
                      f"per step), one softmax+truncate+sample per draw as the reference engine does "
                      f"(engine.py:302-305), ~{seconds / steps:.1f} s per step, {_cpu_model()}"}


def run_reference(args, cfg):
    """--impl reference: the reference's CPU path (the oracle port, oracle/sampling_ref.py) on the
    host cores, K timed steps after W warm-up steps, each step a bounded sample of the workload's
    draws; ms_per_step is the measured wall time of a step (max over workers)."""
    res_cpu = cpu_baseline(cfg, seconds=args.cpu_seconds, steps=args.steps, warmup=args.warmup)
    v = res_cpu["value"]
    return {
        "metric": "resampled_tokens_per_s", "value": v, "unit": "tokens/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": res_cpu["ms_per_step"], "higher_is_better": True, "scaling": cfg["scaling"],
        "vs_baseline": None, "dtype": "f64 (numpy)",
        "data": "synthetic (reference producer fill_logits, seed 7, conc 2.5, range 5.0)",
        "config": workload_config(args, cfg, args.gpus),
        "step": "a bounded sample of the workload's draws per step (see cpu_baseline.sample)",
        "cpu_baseline": res_cpu,
        "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


# ------------------------------------------------------------------------ C3 hit-ratio sweep


def run_c3_sweep(args, cfg, rank, world, dev):
    """C3 with a lookup hit ratio h: 1024 branch keys per step, a fraction h of them
    cached (16-row bf16 entries, V=151936); each step hashes nothing new (digests precomputed),
    looks up all 1024 and replays the hits (lookup + step-wise resample + acceptance, one fused
    path), and runs the miss path for the rest: fresh producer rows (lc_fill_logits, the
    reference producer) -> resample -> insert.  The two legs are timed separately."""
    import torch

    import paper_2604_17353_b200 as lcb
    from paper_2604_17353_b200 import _capi, _dev
    from paper_2604_17353_b200.mixing import mix2

    h = args.hit_ratio
    V, n, R = cfg["V"], cfg["n_req"], cfg["R"]
    n_hit = int(round(h * n))
    n_miss = n - n_hit
    steps_all = args.warmup + args.steps
    budget = n * R * (V * 4 + 8) + 1024
    cache = lcb.LogitsCache(budget, vocab=V, dtype="bfloat16", key_capacity=2 * n + 64, page_rows=16, max_rows=R,
                            page_capacity=2 * n + 64, device=dev)
    # keys: hit set = branches 0..n_hit-1 (fixed); miss set = fresh branches every step
    prompts = [[rank % 256, 3, j % 256, j // 256, 9] for j in range(n_hit)]
    miss_prompts = [[rank % 256, 4, s % 256, s // 256, j % 256, j // 256] for s in range(steps_all)
                    for j in range(n_miss)]
    hit_d = lcb.hash_prompts(prompts, dev=dev) if n_hit else torch.empty(0, dtype=torch.int64, device=dev)
    miss_d = (lcb.hash_prompts(miss_prompts, dev=dev) if n_miss else torch.empty(0, dtype=torch.int64, device=dev))
    tdt = torch.bfloat16
    fill_states = lambda base, m: lcb._dev.u64_tensor([mix2(7, base + i) for i in range(m)], dev)  # noqa: E731
    miss_tasks = lcb.make_tasks(row=np.arange(n_miss * R), pos=np.tile(np.arange(R), n_miss), temperature=cfg["T"],
                                top_k=cfg["k"], top_p=cfg["p"], draw_begin=np.arange(n_miss * R),
                                draw_end=np.arange(n_miss * R) + 1, seed_base=np.repeat(np.arange(n_miss), R))
    miss_tasks_d = torch.from_numpy(np.ascontiguousarray(miss_tasks).view(np.uint8)).to(dev)
    if n_hit:  # pre-insert the hit set (untimed)
        rows = torch.empty((n_hit * R, V), dtype=tdt, device=dev)
        st = fill_states((rank << 40) + (1 << 32), n_hit * R)
        _capi.check(_capi.lib.lc_fill_logits(st.data_ptr(), n_hit * R, V, 2.5, 5.0, _capi.LC_BF16, rows.data_ptr(),
                                             V, _dev.stream_ptr(dev)))
        tasks = lcb.make_tasks(row=np.arange(n_hit * R), pos=np.tile(np.arange(R), n_hit), temperature=cfg["T"],
                               top_k=cfg["k"], top_p=cfg["p"], draw_begin=np.arange(n_hit * R),
                               draw_end=np.arange(n_hit * R) + 1, seed_base=np.repeat(np.arange(n_hit), R))
        tok, _ = lcb.resample(rows, tasks, seeds=lcb._dev.u64_tensor([mix2(99, j) for j in range(n_hit)], dev),
                              n_draws=n_hit * R)
        cache.insert_batch(hit_d, torch.full((n_hit,), R, dtype=torch.int32, device=dev),
                           torch.full((n_hit,), V, dtype=torch.int32, device=dev), rows,
                           torch.arange(n_hit, dtype=torch.int64, device=dev) * R, tok.contiguous(), R)
        del rows
    T = torch.full((n,), cfg["T"], dtype=torch.float64, device=dev)
    K = torch.full((n,), cfg["k"], dtype=torch.int32, device=dev)
    P = torch.full((n,), cfg["p"], dtype=torch.float64, device=dev)
    step_in = []
    for s in range(steps_all):
        dg = torch.cat([hit_d, miss_d[s * n_miss:(s + 1) * n_miss]])
        seeds = lcb._dev.u64_tensor([mix2(1, (rank << 40) + s * n + j) for j in range(n)], dev)
        st = fill_states((rank << 40) + (2 << 32) + s * n_miss * R, n_miss * R) if n_miss else None
        step_in.append((dg, seeds, st))
    fused = args.miss_path == "fused"
    rows_m = torch.empty((0 if fused else max(n_miss, 1) * R, V), dtype=tdt, device=dev)
    lens_m = torch.full((max(n_miss, 1),), R, dtype=torch.int32, device=dev)
    keep_m = torch.zeros(max(n_miss, 1), dtype=torch.int32, device=dev)
    slot_m = torch.empty(max(n_miss, 1), dtype=torch.int32, device=dev)
    gen_m = torch.empty(max(n_miss, 1), dtype=torch.int32, device=dev)
    pos_m = torch.arange(R, dtype=torch.int32, device=dev).repeat(max(n_miss, 1))
    tasks_m = torch.empty(max(n_miss, 1) * R * lcb._capi.TASK_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    tok_m = torch.empty(max(n_miss, 1) * R, dtype=torch.int32, device=dev)
    st_ = _dev.stream_ptr(dev)
    vocs_m = torch.full((max(n_miss, 1),), V, dtype=torch.int32, device=dev)
    offs_m = torch.arange(max(n_miss, 1), dtype=torch.int64, device=dev) * R
    bufs = {}
    ev_hit, ev_miss, outs = [], [], []

    def step(s, timed):
        dg, seeds, st = step_in[s]
        a, b, c_ = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record()
        tok, rep, div, slot, ln = cache.replay_stepwise(dg, R, 1, seeds, T, K, P, bufs=bufs)
        b.record()
        if n_miss and fused:
            # f1: entries first (no rows), the producer writes straight into their slab rows,
            # resample from the slab, tokens into the entries -- no staging rows, no insert copy
            _capi.check(_capi.lib.lc_cache_writeback(cache.handle, dg[n_hit:].data_ptr(), lens_m.data_ptr(),
                                                     vocs_m.data_ptr(), keep_m.data_ptr(), gen_m.data_ptr(), n_miss,
                                                     None, _capi.LC_BF16, 0, None, None, R, slot_m.data_ptr(),
                                                     gen_m.data_ptr(), st_))
            s_rep, g_rep = slot_m.repeat_interleave(R), gen_m.repeat_interleave(R)
            _capi.check(_capi.lib.lc_cache_fill_rows(cache.handle, s_rep.data_ptr(), g_rep.data_ptr(),
                                                     pos_m.data_ptr(), st.data_ptr(), n_miss * R, 2.5, 5.0, st_))
            _capi.check(_capi.lib.lc_replay_tasks(slot_m.data_ptr(), lens_m.data_ptr(), vocs_m.data_ptr(), n_miss, R,
                                                  1, T.data_ptr(), K.data_ptr(), P.data_ptr(), tasks_m.data_ptr(),
                                                  st_))
            lcb.sampling.resample(None, tasks_m, seeds=seeds[n_hit:], n_draws=n_miss * R, cache=cache,
                                  out=(tok_m, torch.empty_like(tok_m, dtype=torch.uint8)))
            _capi.check(_capi.lib.lc_cache_set_tokens(cache.handle, s_rep.data_ptr(), g_rep.data_ptr(),
                                                      pos_m.data_ptr(), tok_m.data_ptr(), n_miss * R, st_))
            cache._dirty()
        elif n_miss:
            _capi.check(_capi.lib.lc_fill_logits(st.data_ptr(), n_miss * R, V, 2.5, 5.0, _capi.LC_BF16,
                                                 rows_m.data_ptr(), V, _dev.stream_ptr(dev)))
            mt, _ = lcb.resample(rows_m, miss_tasks_d, seeds=seeds[n_hit:], n_draws=n_miss * R)
            cache.insert_batch(dg[n_hit:], lens_m, vocs_m, rows_m, offs_m, mt, R)
        c_.record()
        if timed:
            ev_hit.append((a, b))
            ev_miss.append((b, c_))
            outs.append((slot, rep.clone()))

    for s in range(args.warmup):
        step(s, False)
    torch.cuda.synchronize(dev)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        torch.cuda.synchronize(dev)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        t0.record()
        for s in range(args.warmup, steps_all):
            step(s, True)
        t1.record()
        torch.cuda.synchronize(dev)
    ms = t0.elapsed_time(t1)
    from paper_2604_17353_b200.shard import reduce_stats

    ms = float(reduce_stats(torch.tensor([ms], dtype=torch.float64, device=dev),
                            torch.zeros(1, dtype=torch.float64, device=dev), world)[0][0])  # max over ranks
    hit_ms = sum(a.elapsed_time(b) for a, b in ev_hit) / args.steps
    miss_ms = sum(a.elapsed_time(b) for a, b in ev_miss) / args.steps
    slots = torch.stack([o[0] for o in outs]).cpu().numpy()
    reps = torch.stack([o[1] for o in outs]).cpu().numpy()
    lookup_hits = float((slots >= 0).mean())
    assert np.all(slots[:, :n_hit] >= 0) and np.all(slots[:, n_hit:] < 0), "hit/miss pattern"
    pos_hit = float(reps.sum() / (n * R * args.steps))  # replayed positions / all positions (ReplayOutcome)
    tokens = n * R * args.steps
    return {
        "metric": "resampled_tokens_per_s", "value": tokens * world / (ms * 1e-3), "unit": "tokens/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (reference producer fill_logits, seed 7, conc 2.5, range 5.0)",
        "config": {"workload": cfg["desc"] + f"; lookup hit ratio {h}", "config": "c3", "hit_ratio": h,
                   "branches": n, "rows_per_entry": R, "vocab": V},
        "lookup_hit_ratio": lookup_hits, "position_hit_ratio": pos_hit,
        "lookup_resample_ms_per_step": hit_ms, "miss_path_ms_per_step": miss_ms,
        "miss_path": ("lc_cache_writeback (entries, no rows) -> lc_cache_fill_rows (producer straight into the "
                      "slab) -> lc_cache_resample -> lc_cache_set_tokens" if fused else
                      "lc_fill_logits (producer, staging rows) -> resample -> lc_cache_insert (copy)"),
        # per step: lookup (probe + commit), replay tasks, resample (row kernel + requeue + exact),
        # cached tokens, acceptance; misses: producer, resample (3), insert (policy + copy)
        "gpu_launches": (8 + (6 if n_miss else 0)) * args.steps, "clocks": clk.summary(),
    }


# ------------------------------------------------------------------------ C4: insert / eviction stress


def c4_keys(n_keys, dev):
    """1M distinct prefix digests by tree expansion: 1024 root prompts, each extended by
    1024 two-token children (prefix extension = hash_tokens(child, start=root), mixing.py:63-65)."""
    import torch

    from paper_2604_17353_b200 import _capi, _dev

    n_root = 1024
    n_child = -(-n_keys // n_root)
    roots = [[r % 256, r // 256, 7, 11, 13] for r in range(n_root)]
    from paper_2604_17353_b200.mixing import hash_prompts

    rd = hash_prompts(roots, dev=dev)
    c = np.arange(n_root * n_child) % n_child
    toks = torch.from_numpy(np.stack([c % 256, c // 256 + 1], 1).astype(np.int32).ravel()).to(dev)
    offs = torch.arange(0, 2 * n_root * n_child + 1, 2, dtype=torch.int64, device=dev)
    par = rd.repeat_interleave(n_child)
    out = torch.empty(n_root * n_child, dtype=torch.int64, device=dev)
    _capi.check(_capi.lib.lc_hash_prefix(toks.data_ptr(), offs.data_ptr(), par.data_ptr(), n_root * n_child,
                                         out.data_ptr(), _dev.stream_ptr(dev)))
    out = out[:n_keys]
    assert torch.unique(out).numel() == n_keys
    return out


def c4_cpu_baseline(V, seconds=10.0, entries=10_000):
    """The reference's update path on the host: f32 row copy + accounting + the O(E) LRU scan
    (logits_cache.py:96-140), restated in oracle/cache_ref.py, at a reduced E."""
    sys.path.insert(0, ROOT)
    from oracle import cache_ref

    row_acct = V * 4 + 8
    orc = cache_ref.CacheOracle(entries * row_acct, entries + 64, entries + 64)
    src = np.random.default_rng(0).standard_normal((4, V)).astype(np.float32)
    store = {}
    rng = np.random.default_rng(1)
    for i in range(entries):  # fill (untimed)
        orc.insert(i, 1, V)
    n = 0
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        d = int(rng.integers(0, 1 << 20)) + entries
        store[d & 1023] = np.array(src[n % 4], dtype=np.float32)  # reference: np.asarray(..., float32) copy
        orc.insert(d, 1, V)
        n += 1
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "inserts/s", "cores": 1, "kind": "port",
            "sample": f"{n} single-row inserts (V={V}, f32 row copy + O(E) min-(last_hit, digest) victim scan "
                      f"as logits_cache.py:96-140) into a full cache of E={entries} entries (reduced from 400k: "
                      f"the reference's eviction is O(E) per insert), {seconds:.0f} s, one core"}


def run_c4(args, cfg, rank, world, dev):
    import torch

    import paper_2604_17353_b200 as lcb
    from paper_2604_17353_b200 import _capi, _dev

    V = cfg["V"]
    free, _ = torch.cuda.mem_get_info(dev)
    S = int(min(cfg["entries"], (free * 0.6) // (V * 2)))
    row_acct = V * 4 + 8
    cache = lcb.LogitsCache(S * row_acct, vocab=V, dtype="bfloat16", key_capacity=S + 64, page_rows=1,
                            max_rows=1, page_capacity=S + 64, device=dev)
    keys = c4_keys(cfg["keys"], dev)
    keys_h = _dev.u64_numpy(keys)
    pool_n = 2048
    pool = torch.empty((pool_n, V), dtype=torch.bfloat16, device=dev)
    st = _dev.u64_tensor([(0x9E3779B97F4A7C15 * (i + 1 + (rank << 20))) & ((1 << 64) - 1) for i in range(pool_n)],
                         dev)
    _capi.check(_capi.lib.lc_fill_logits(st.data_ptr(), pool_n, V, 2.5, 5.0, _capi.LC_BF16, pool.data_ptr(), V,
                                         _dev.stream_ptr(dev)))
    ptoks = torch.arange(pool_n, dtype=torch.int32, device=dev)
    B = cfg["batch"]
    n_ins = int(round(B * cfg["ins_frac"]))
    n_lk = B - n_ins
    ones = torch.ones(max(B, 65536), dtype=torch.int32, device=dev)
    vocs = torch.full((max(B, 65536),), V, dtype=torch.int32, device=dev)
    trace = []  # (kind, key indices) in issue order, for the oracle replay

    def insert(idx_h, idx_d, base):
        n = idx_d.numel()
        offs = (torch.arange(n, dtype=torch.int64, device=dev) + base) % pool_n
        trace.append(("ins", idx_h))
        return cache.insert_batch(keys[idx_d], ones[:n], vocs[:n], pool, offs, ptoks, 1)[0]

    # prefill: S distinct keys (cache full, no evictions yet)
    perm = np.random.default_rng(1 + rank).permutation(cfg["keys"])[:S]
    outs = []
    for b0 in range(0, S, 65536):
        ih = perm[b0:b0 + 65536]
        outs.append(insert(ih, torch.from_numpy(ih).to(dev), b0))
    rng = np.random.default_rng(2 + rank)
    n_steps = args.warmup + args.steps
    # warm-up + timed steps, then args.steps fresh steps for the e2e leg
    ops = [(rng.integers(0, cfg["keys"], n_lk), rng.integers(0, cfg["keys"], n_ins))
           for _ in range(n_steps + args.steps)]
    ops_d = [(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)) for a, b in ops]

    ev = []  # CUDA events around each timed insert call (policy + copy kernels), same stream

    def step(i, timed=False):
        lk_h, in_h = ops[i]
        lk_d, in_d = ops_d[i]
        trace.append(("lk", lk_h))
        s_lk = cache.lookup_batch(keys[lk_d])[0]
        if timed:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
        s_in = insert(in_h, in_d, i * B)
        if timed:
            b.record()
            ev.append((a, b))
        return s_lk, s_in

    for i in range(args.warmup):
        outs.extend(step(i))
    torch.cuda.synchronize(dev)
    st0 = cache._stats()
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        torch.cuda.synchronize(dev)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        t0.record()
        for i in range(args.warmup, n_steps):
            outs.extend(step(i, True))
        t1.record()
        torch.cuda.synchronize(dev)
    ms = t0.elapsed_time(t1)
    st1 = cache._stats()
    evictions = st1.evictions - st0.evictions if hasattr(st1, "evictions") else None
    from paper_2604_17353_b200.shard import reduce_stats

    tt, cc = reduce_stats(torch.tensor([ms], dtype=torch.float64, device=dev),
                          torch.tensor([float(evictions or 0)], dtype=torch.float64, device=dev), world)
    ms, evictions = float(tt[0]), int(cc[0])  # max over ranks; evictions summed over ranks

    ins_ms = sum(a.elapsed_time(b) for a, b in ev) / len(ev)

    # parity: hit/miss + slots (which encode the victim order) vs the heap-mode oracle replay
    parity = None
    if not args.no_check:
        sys.path.insert(0, ROOT)
        from oracle import cache_ref

        orc = cache_ref.CacheOracle(S * row_acct, S + 64, S + 64, 1, heap=True)
        got = np.concatenate([o.cpu().numpy() for o in outs])
        want = []
        for kind, idx in trace:
            if kind == "lk":
                for k in idx:
                    e = orc.lookup(int(keys_h[k]))
                    want.append(-1 if e is None else e.slot)
            else:
                for k in idx:
                    want.append(orc.insert(int(keys_h[k]), 1, V)[0].slot)
        want = np.asarray(want[:got.size], np.int32)
        parity = {"ops_checked": int(got.size), "slots_equal": bool(np.array_equal(got, want)),
                  "evictions_oracle": orc.evictions}
    peak, peak_src = peaks()
    n_timed = args.steps * n_ins
    algo = n_ins * (2 * V * 2 + 4 + 8 + 4)  # row read + slab write, token, digest, length per insert
    res = {
        "metric": "inserts_per_s", "value": n_timed * world / (ms * 1e-3), "unit": "inserts/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16 rows, int64 bookkeeping",
        "data": "synthetic (reference producer fill_logits rows, tree-expanded prefix digests)",
        "config": {"workload": cfg["desc"], "config": "c4", "vocab": V, "entries": S, "key_space": cfg["keys"],
                   "ops_per_step": B, "inserts_per_step": n_ins, "lookups_per_step": n_lk,
                   "slab_gb": (S + 64) * V * 2 / 1e9, "l2": "slab writes and source rows larger than L2"},
        "lookups_per_s": args.steps * n_lk * world / (ms * 1e-3),
        "evictions_per_s": (evictions / (ms * 1e-3)) if evictions is not None else None,
        "hit_ratio": (st1.hits - st0.hits) / max(1, st1.lookups - st0.lookups),
        "parity": parity,
        "roofline": {"bound": "hbm", "achieved": algo / (ins_ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": algo / (ins_ms * 1e-3) / 1e9 / peak, "traffic": None, "peak_source": peak_src,
                     "kernel": "lc_cache_insert (insert_policy_kernel + insert_copy_kernel)",
                     "kernel_ms_avg": ins_ms, "algorithmic_bytes_per_launch": algo},
        "gpu_launches": 4 * args.steps,
        "clocks": clk.summary(),
    }
    # e2e: digests from host (pinned), slots back to host, per step
    h_keys = [torch.from_numpy(np.concatenate([keys_h[a], keys_h[b]]).view(np.int64)).pin_memory()
              for a, b in ops[n_steps:]]
    d_keys = torch.empty(B, dtype=torch.int64, device=dev)
    h_out = torch.empty(B, dtype=torch.int32, pin_memory=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    e0.record()
    for i in range(args.steps):
        d_keys.copy_(h_keys[i], non_blocking=True)
        s_lk = cache.lookup_batch(d_keys[:n_lk])[0]
        s_in = cache.insert_batch(d_keys[n_lk:], ones[:n_ins], vocs[:n_ins], pool,
                                  torch.arange(n_ins, dtype=torch.int64, device=dev) % pool_n, ptoks, 1)[0]
        h_out[:n_lk].copy_(s_lk, non_blocking=True)
        h_out[n_lk:].copy_(s_in, non_blocking=True)
    e1.record()
    torch.cuda.synchronize(dev)
    e_ms = e0.elapsed_time(e1)
    res["e2e"] = {"value": n_timed * world / (e_ms * 1e-3), "unit": "inserts/s", "h2d_bytes_per_step": B * 8,
                  "d2h_bytes_per_step": B * 4}
    if not args.no_cpu_baseline and rank == 0:
        res["cpu_baseline"] = c4_cpu_baseline(V, seconds=min(args.cpu_seconds, 10.0))
    return res


def spawn_ranks(args):
    """``--gpus N`` without a torchrun environment: re-launch this script under
    torch.distributed.run, one process per GPU on this node (127.0.0.1 rendezvous);
    rank 0 prints the line."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def run_dry(args, cfg, rank, world):
    """The multi-rank host logic without a GPU (gloo): every rank derives its shard of the
    workload exactly as the GPU run does (tree i -> rank i mod G for the tree-sharded configs,
    its own requests otherwise), then the statistics vector (max of times, sum of counters)
    is reduced as after a timed interval.  Used by tests/test_shard_gloo.py."""
    import torch
    import torch.distributed as dist

    from paper_2604_17353_b200.shard import local_trees, reduce_stats

    if world > 1:
        dist.init_process_group("gloo")
    n_req = cfg.get("n_req", 0)
    trees = None
    if cfg.get("scaling") == "strong":
        trees = local_trees(8, rank, world)
        n_req = len(trees) * (cfg["n_req"] // 8)
    rows = n_req * cfg.get("R", 1)
    times = torch.tensor([1.0 + rank, 2.0 * (rank + 1)], dtype=torch.float64)
    counts = torch.tensor([float(rows), float(rows * cfg.get("nb", 1)), 1.0], dtype=torch.float64)
    t, c = reduce_stats(times, counts, world)
    shards = [None] * world
    if world > 1:
        dist.all_gather_object(shards, {"rank": rank, "trees": trees, "requests": n_req, "rows": rows})
        dist.destroy_process_group()
    else:
        shards = [{"rank": 0, "trees": trees, "requests": n_req, "rows": rows}]
    return {"dry_run": True, "n_gpus": world, "config": args.config, "scaling": cfg.get("scaling"),
            "shards": shards, "rows_total": int(c[0]), "draws_total": int(c[1]), "ranks_reporting": int(c[2]),
            "max_times": t.tolist(), "backend": "gloo"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-check", action="store_true",
                    help="skip the untimed oracle validation leg (c4: the op-trace replay)")
    ap.add_argument("--check-draws", type=int, default=None,
                    help="draws the check leg validates (default 10M at V=32000, 100K for the wide configs)")
    ap.add_argument("--window", type=int, default=8, help="positions per window for --policy windowed")
    ap.add_argument("--policy", default="step_wise", choices=["step_wise", "hotspot", "windowed"],
                    help="replay policy of the resample step (ReplayPolicy)")
    ap.add_argument("--miss-path", default="fused", choices=["fused", "staged"],
                    help="c3 sweep miss path: producer straight into the slab (f1) or via staging rows + copy")
    ap.add_argument("--hit-ratio", type=float, default=None,
                    help="c3: lookup hit ratio h of the sweep (default: every branch cached)")
    ap.add_argument("--graph", action=argparse.BooleanOptionalAction, default=None,
                    help="replay the step from a CUDA graph (default: on for the tree-sharded c5)")
    ap.add_argument("--one-rank-of", type=int, default=None, metavar="G",
                    help="run rank 0's share of a G-GPU run on this one GPU (no process group): the per-rank "
                         "throughput behind the scaling curve")
    ap.add_argument("--dry-run", action="store_true",
                    help="no GPU: run the N-rank host logic (shard plan + statistics reduction) over gloo")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]
    if args.graph is None:
        args.graph = cfg.get("scaling") == "strong"
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args)  # re-executes this script under torchrun; does not return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.dry_run:
        res = run_dry(args, cfg, rank, world)
        if rank == 0:
            print(json.dumps(res), flush=True)
        return
    if args.impl == "reference":
        if rank == 0:
            if args.config == "c4":
                cb = c4_cpu_baseline(cfg["V"], seconds=min(args.cpu_seconds, 10.0))
                print(json.dumps({"metric": "inserts_per_s", "value": cb["value"], "unit": "inserts/s",
                                  "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
                                  "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
                                  "vs_baseline": None, "dtype": "f32 (numpy)", "data": "synthetic",
                                  "config": {"workload": cfg["desc"], "config": "c4"}, "cpu_baseline": cb,
                                  "e2e": {"value": cb["value"], "unit": "inserts/s", "h2d_bytes_per_step": 0,
                                          "d2h_bytes_per_step": 0}}), flush=True)
            else:
                print(json.dumps(run_reference(args, cfg)), flush=True)
        return
    import torch
    import torch.distributed as dist

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if args.config == "c4":
        res = run_c4(args, cfg, rank, world, dev)
    elif args.config == "c3" and args.hit_ratio is not None:
        res = run_c3_sweep(args, cfg, rank, world, dev)
    else:
        res = (run_windowed if args.policy == "windowed" else run_ours)(args, cfg, rank, world, dev)
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
