#!/usr/bin/env python
"""Benchmark of the Pair-HMM forward hot path (BASELINE.json metric: GCUPS).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c5] [--cpu-seconds 10] [--no-secondary]

Workload (default c5 = BASELINE.json configs[4], the config the 1/2/4/8-GPU metric is
quoted on; it fits one B200): ONE batch list of 10,000,384 GATK-shaped pairs (reads
50-250 x haplotypes 100-600, derived, seed 20240811+4), scored with the GATK FP64 retry
(FP32 fast path + guard band + bit-exact FP32 reruns + FP64 retry of FP32-underflowed
pairs).  One step = one pass of the engine over the whole batch list.

Under torchrun the batch list is SHARDED: every rank draws the same list, takes its
cost-balanced, bin-stratified share of the reads (shards.plan_shards: one read with all
of its batch's haplotypes is the planning unit) and scores it on its GPU; results are
gathered on the host into global-id order through shared memory (shards.HostGather).
No collective on the data path — NCCL only carries the max-over-ranks timing.

  value     GCUPS with inputs resident in HBM: true cells (all ranks) / max over ranks of
            the engine device time per step (CUDA events on the engine stream, phmm_execute).
  e2e       GCUPS through the C-ABI call phmm_score from pinned HOST buffers (H2D of the
            inputs, planning, kernels, D2H of scores + status, finishing) plus the host
            gather into the global result arrays, wall clock, max over ranks.
  roofline  the dominant kernel (k_stream FP32 streaming wavefront, all tiling bins of the
            FP32 phase) against the FP32-FMA roofline of SURVEY.md §8(d): 148 SMs x 128
            lanes x f_SM / 8 ops per cell; plus the whole step and a per-phase breakdown.
  cpu_baseline  the reference's own CPU path (the unmodified pairhmm package installed in
            baseline/_ref, numba, pairhmm.run on all host cores; kind "reference") on a
            bounded sample of the same workload, rank 0 only, with the C port of its
            recursion (oracle/, kind "port") beside it.
--impl reference times the reference package alone (the C port when baseline/_ref is absent).
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

WORKLOAD_TEXT = {
    "c5": "c5: 10,000,384-pair GATK-shaped batch list (19,532 batches x 64 reads x 8 haps; reads 50-250 x "
          "haps 100-600, derived, seed 20240811+4), FP64 retry of FP32-underflowed pairs",
    "c2": "c2: 65,536 uniform pairs 250x250 FP32 on 1xB200 (peak-kernel microbench), derived, seed 20240811+1",
    "c3": "c3: GATK-shaped 65,536 pairs, reads 50-250 x haps 100-600, derived, seed 20240811+2",
    "c1": "c1: 1,000 pairs 100x150, fixed qualities",
    "c4": "c4: 2,048 long pairs, reads 512-1024 x haps 1024-2048",
}
# headline flags per workload: c5/c3/c4 GATK FP64 retry; c1/c2 the reference's FP32 semantics
RETRY_WORKLOADS = ("c5", "c3", "c4")
FP32_LANES_PER_SM = 128          # tools/microbench/pipes.cu: FFMA 128 lanes/clk/SM
FP64_LANES_PER_SM = 64           # tools/microbench/pipes.cu: DFMA 64 lanes/clk/SM
OPS_PER_CELL = 8                 # 1 FADD + 4 FMUL + 3 FFMA per cell
PHASES = ("precompute", "fp32_stream", "post_a_exact32_and_fp64_units", "post_bc_fp64_per_pair")


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.Q,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 5 + i and r[5 + i].lower().startswith("active")})
        loaded = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def pinned_copy(flat):
    """FlatBatches whose arrays live in pinned host memory (torch pin_memory)."""
    import torch
    from paper_2411_11547_b200.model import FlatBatches
    arrays = {}
    for name in FlatBatches.FIELDS:
        a = getattr(flat, name)
        t = torch.empty(a.shape[0], dtype=getattr(torch, {"int8": "int8", "uint8": "uint8",
                                                          "int64": "int64"}[a.dtype.name]),
                        pin_memory=True)
        t.numpy()[:] = a
        arrays[name] = t.numpy()
    out = FlatBatches.__new__(FlatBatches)
    for name in FlatBatches.FIELDS:
        setattr(out, name, arrays[name])
    return out


def pair_cells(flat):
    pr, ph = flat.pair_index()
    return flat.read_len[pr] * flat.hap_len[ph]


def cpu_baseline(flat, seconds, flags_retry=False):
    """Time the C oracle (reference recursion port) on a bounded prefix of the workload:
    FP32 on every pair of the prefix, plus (GATK semantics) FP64 on its FP32-flagged pairs."""
    from oracle import oracle
    oracle.build()
    ofl = oracle.Flat(**flat.as_dict())
    pr, ph = flat.pair_index()
    cores = os.cpu_count() or 1
    done = cells = retried = 0
    t0 = time.perf_counter()
    chunk = 256
    while done < pr.shape[0] and time.perf_counter() - t0 < seconds:
        sl = slice(done, min(done + chunk, pr.shape[0]))
        acc, st = oracle.score_raw(ofl, "f32", 120, threads=cores, pairs=(pr[sl], ph[sl]))
        if flags_retry:
            bad = np.flatnonzero(st == oracle.OVERFLOW)
            if bad.size:
                oracle.score_raw(ofl, "f64", 0, threads=cores, pairs=(pr[sl][bad], ph[sl][bad]))
                retried += int(bad.size)
        cells += int((flat.read_len[pr[sl]] * flat.hap_len[ph[sl]]).sum())
        done = sl.stop
        chunk = min(chunk * 2, 65536)
    dt = time.perf_counter() - t0
    return {"value": cells / dt / 1e9, "unit": "GCUPS", "cores": cores, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": "first %d of %d pairs (%.3g cells) of the same workload, FP32%s, oracle/phmm_oracle.c "
                      "with %d threads, %.1f s" % (done, pr.shape[0], cells,
                                                    " + FP64 on its %d FP32-flagged pairs" % retried
                                                    if flags_retry else "", cores, dt)}


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_package():
    """The unmodified reference package (pairhmm 0.1.0, numpy + numba) installed by
    `pip install --no-index --no-deps --target baseline/_ref`, or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "pairhmm")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import pairhmm
        import numba  # noqa: F401
    except ImportError:
        return None
    return pairhmm


def _ref_batches(pairhmm, flat, b0, b1):
    """Reference Batch objects (the reference's own types) for batches [b0, b1) of flat."""
    out = []
    for b in range(b0, b1):
        reads = []
        for r in range(int(flat.batch_read_off[b]), int(flat.batch_read_off[b + 1])):
            s = slice(int(flat.read_off[r]), int(flat.read_off[r + 1]))
            reads.append(pairhmm.ReadRecord(flat.read_bases[s], flat.bq[s], flat.iq[s], flat.dq[s], flat.gq[s]))
        haps = [pairhmm.Haplotype(flat.hap_bases[int(flat.hap_off[h]):int(flat.hap_off[h + 1])])
                for h in range(int(flat.batch_hap_off[b]), int(flat.batch_hap_off[b + 1]))]
        out.append(pairhmm.Batch(reads, haps))
    return out


def reference_cpu(flat, seconds, flags_retry=False, warm=True):
    """The reference's own CPU path, pairhmm.run(batches, default_configs('f32'),
    workers=all cores) (pipeline.py:77-142), on the first batches of the workload, grown
    until about `seconds` of work; GATK semantics re-score the pairs it flags
    (NumericOverflowError, NaN) with pairhmm.run(..., default_configs('f64')) — the
    reference has no automatic retry, so a caller does exactly this.  Cells = every pair's
    m*n once (the GPU arm's accounting)."""
    pairhmm = reference_package()
    if pairhmm is None:
        return None
    cores = os.cpu_count() or 1
    cf32, cf64 = pairhmm.default_configs("f32"), pairhmm.default_configs("f64")
    nb = flat.batch_read_off.shape[0] - 1
    if warm:                                   # numba JIT (cache=True) outside the timed region
        w = _ref_batches(pairhmm, flat, 0, 1)
        pairhmm.run(w, cf32, workers=1)
        pairhmm.run(w, cf64, workers=1)
    done = cells = retried = 0
    step = 1
    t_all = 0.0
    while done < nb and t_all < seconds:
        b1 = min(nb, done + step)
        batches = _ref_batches(pairhmm, flat, done, b1)
        t0 = time.perf_counter()
        scores, rep = pairhmm.run(batches, cf32, workers=cores)
        if flags_retry:
            bad = np.flatnonzero(np.isnan(scores))
            if bad.size:
                items = pairhmm.enumerate_work_items(batches)
                pairs = [pairhmm.Batch([batches[items[g].batch_index].reads[items[g].read_index]],
                                       [batches[items[g].batch_index].haps[items[g].hap_index]]) for g in bad]
                pairhmm.run(pairs, cf64, workers=cores)
                retried += int(bad.size)
        t_all += time.perf_counter() - t0
        cells += int(rep.total_cells)
        done = b1
        step = min(step * 2, 64)
    pr0 = int(flat.batch_read_off[done])
    return {"value": cells / t_all / 1e9, "unit": "GCUPS", "cores": cores, "kind": "reference",
            "cpu_model": cpu_model(),
            "sample": "first %d of %d batches (%d reads, %.3g cells) of the same workload through the unmodified "
                      "reference pairhmm.run(batches, default_configs('f32'), workers=%d)%s (numba %s), %.1f s"
                      % (done, nb, pr0, cells, cores,
                         " + pairhmm.run(..., default_configs('f64')) on its %d flagged pairs" % retried
                         if flags_retry else "", _numba_version(), t_all)}


def _numba_version():
    try:
        import numba
        return numba.__version__
    except ImportError:
        return None


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args, ws, rank):
    """--impl reference: the reference's own CPU path (pairhmm.run from baseline/_ref, numba,
    all host cores) on bounded samples of the workload; the C port of its recursion
    (oracle/) when the package is not installed.  Rank 0 only."""
    if rank != 0:
        return 0
    from paper_2411_11547_b200 import datagen
    flat = datagen.workload(args.workload)
    retry = args.workload in RETRY_WORKLOADS
    use_pkg = reference_package() is not None
    per = max(2.0, args.cpu_seconds / max(1, args.steps))

    def sample(seconds, warm):
        if use_pkg:
            return reference_cpu(flat, seconds, retry, warm=warm)
        return cpu_baseline(flat, seconds, retry)

    per_step = []
    base = None
    for i in range(args.warmup + args.steps):
        b = sample(per if i >= args.warmup else 1.0, warm=(i == 0))
        if i >= args.warmup:
            per_step.append(b["value"])
            base = b
    v = statistics.mean(per_step)
    base = dict(base, value=v)
    line = {"impl": "reference", "metric": "GCUPS (cell updates/s)", "value": v, "unit": "GCUPS",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak" if args.workload != "c5" else "strong",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": {"workload": WORKLOAD_TEXT.get(args.workload, args.workload)},
            "cpu_baseline": base,
            "e2e": {"value": v, "unit": "GCUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def reduce_time_cells(seconds, cells, ws, device):
    """(max over ranks of seconds, sum over ranks of cells) — the only cross-rank traffic:
    pairs are independent, so the data path has no collective."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(seconds)], dtype=torch.float64, device=device)
    c = torch.tensor([float(cells)], dtype=torch.float64, device=device)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
    return float(t.item()), float(c.item())


def shard_for_rank(flat, ws, rank):
    """This rank's share of the ONE batch list (shards.plan_shards); ws == 1: all of it."""
    from paper_2411_11547_b200.shards import Shard, make_shard, plan_shards, read_costs
    if ws == 1:
        return Shard(flat, np.arange(flat.num_pairs, dtype=np.int64), 0.0)
    owner = plan_shards(flat, ws)
    return make_shard(flat, owner, rank, read_costs(flat)[0])


def gather_name():
    return "phmm_bench_%s_%s" % (os.environ.get("MASTER_PORT", "0"), os.environ.get("TORCHELASTIC_RUN_ID", "x"))


def secondary(ctx, name, flags, steps=3):
    """Device GCUPS of another BASELINE config on the same engine (reported, not headline)."""
    from paper_2411_11547_b200 import datagen, default_configs
    from paper_2411_11547_b200.pipeline import config_tuples
    flat = datagen.workload(name)
    cfg = config_tuples(default_configs("f32"))
    ctx.prepare(flat, cfg, flags)
    ctx.execute()
    ms, fast, ph = [], [], []
    for _ in range(steps):
        ctx.execute()
        d, f, _n = ctx.last_timing()
        ms.append(d)
        fast.append(f)
        ph.append(ctx.last_phases())
    _, _, st = ctx.fetch()
    cells = st.total_cells
    return {"workload": WORKLOAD_TEXT.get(name, name), "gcups": cells / (np.mean(ms) * 1e-3) / 1e9,
            "pairs": st.num_pairs, "cells": cells, "fast_pairs": st.fast_pairs,
            "exact_pairs": st.exact_pairs, "f64_retry_pairs": st.f64_pairs,
            "device_ms": float(np.mean(ms)), "fast_ms": float(np.mean(fast)),
            "fp32_phase_gcups": cells / (np.mean(fast) * 1e-3) / 1e9,
            "phases_ms": dict(zip(PHASES, np.mean(ph, axis=0).tolist())),
            "flags": "retry_f64" if flags & 1 else "reference-f32"}


def e2e_run(name, steps=3):
    """Wall GCUPS of the drop-in API pipeline.run(batches) from reference-style Batch
    objects (flatten + budget check + engine call + report), c2/c3-sized."""
    from paper_2411_11547_b200 import datagen, default_configs, run
    kw = dict(datagen.WORKLOADS[name])
    batches = datagen.generate_synthetic(**kw)
    cfg = default_configs("f32")
    run(batches, cfg)
    vals = []
    for _ in range(steps):
        t0 = time.perf_counter()
        _, rep = run(batches, cfg)
        vals.append(rep.total_cells / (time.perf_counter() - t0) / 1e9)
    return {"workload": WORKLOAD_TEXT.get(name, name), "api": "pipeline.run(list[Batch])",
            "gcups": float(np.median(vals))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c5")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    ws, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, ws, rank)

    import torch
    import torch.distributed as dist
    from paper_2411_11547_b200 import _native, datagen, default_configs
    from paper_2411_11547_b200.build import build_native
    from paper_2411_11547_b200.pipeline import config_tuples
    from paper_2411_11547_b200.shards import HostGather

    build_native()
    # PHMM_BENCH_SHARE_DEVICE=1 (testing the N>1 path on a 1-GPU box): every rank on cuda:0,
    # timing reductions over gloo
    share = os.environ.get("PHMM_BENCH_SHARE_DEVICE") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    red_dev = "cpu" if share else "cuda"
    if ws > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    full = datagen.workload(args.workload)
    t_plan = time.perf_counter()
    shard = shard_for_rank(full, ws, rank)
    t_plan = time.perf_counter() - t_plan
    flat = shard.flat
    n_total = full.num_pairs
    cfg = config_tuples(default_configs("f32"))
    flags = _native.FLAG_RETRY_F64 if args.workload in RETRY_WORKLOADS else 0
    ctx = _native.Context(local)
    n_pairs = ctx.prepare(flat, cfg, flags)
    l2_flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    for _ in range(args.warmup):
        ctx.execute()
    barrier()
    dev_ms, fast_ms, phases = [], [], []
    launches = 0
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            l2_flush.zero_()
            torch.cuda.synchronize()
            ctx.execute()
            d, f, n = ctx.last_timing()          # CUDA events on the engine stream
            dev_ms.append(d)
            fast_ms.append(f)
            phases.append(ctx.last_phases())
            launches += n
        barrier()
    scores, status, st = ctx.fetch()
    cells = st.total_cells
    t_max, total_cells = reduce_time_cells(float(np.sum(dev_ms)) * 1e-3, cells, ws, red_dev)
    value = total_cells * args.steps / t_max / 1e9
    fast_max, _ = reduce_time_cells(float(np.sum(fast_ms)) * 1e-3, 0, ws, red_dev)
    retried = (status & _native.ST_RETRIED_F64) != 0
    retry_cells = int(pair_cells(flat)[retried].sum()) if retried.any() else 0

    # ---- e2e through the C-ABI from pinned host buffers (phmm_score) + host gather
    # (caller-owned result buffers, reused across calls like any C-ABI caller's)
    pflat = pinned_copy(flat)
    res = np.empty(pflat.num_pairs, np.float64)
    res_st = np.empty(pflat.num_pairs, np.uint8)
    gather = None
    if ws > 1:
        if rank == 0:
            gather = HostGather(gather_name(), n_total, create=True)
        dist.barrier()
        if rank != 0:
            gather = HostGather(gather_name(), n_total, create=False)
    for _ in range(2):                      # warm-up (also first-touches the gather pages)
        out, ost, _ = ctx.score(pflat, cfg, flags, out=res, status=res_st)
        if gather is not None:
            gather.put(shard.gids, out, ost)
    barrier()
    t0 = time.perf_counter()
    call_ms = []
    for _ in range(args.steps):
        tc = time.perf_counter()
        out, ost, est = ctx.score(pflat, cfg, flags, out=res, status=res_st)
        if gather is not None:
            gather.put(shard.gids, out, ost)
        call_ms.append((time.perf_counter() - tc) * 1e3)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e2e_max, _ = reduce_time_cells(time.perf_counter() - t0, 0, ws, red_dev)
    e2e_value = total_cells * args.steps / e2e_max / 1e9
    gathered_ok = None
    if gather is not None:
        dist.barrier()
        if rank == 0:   # every global id was written by exactly one rank, statuses consistent
            gathered_ok = bool(np.array_equal(np.isnan(gather.scores), (gather.status & 0x0F) != 0))
        dist.barrier()
        gather.close()

    if rank != 0:
        dist.destroy_process_group() if ws > 1 else None
        return 0

    peaks = measured_peaks()
    clk = clocks.summary()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    props = torch.cuda.get_device_properties(local)
    nsm = props.multi_processor_count
    peak = nsm * FP32_LANES_PER_SM * sm_max * 1e6 / OPS_PER_CELL / 1e9
    peak64 = nsm * FP64_LANES_PER_SM * sm_max * 1e6 / OPS_PER_CELL / 1e9
    fast_gcups = cells / (float(np.mean(fast_ms)) * 1e-3) / 1e9
    ph_mean = np.mean(phases, axis=0)
    traffic = profile_traffic(args.workload)
    line = {
        "metric": "GCUPS (cell updates/s)", "value": value, "unit": "GCUPS", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong" if args.workload == "c5" else "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": WORKLOAD_TEXT.get(args.workload, args.workload), "pairs_total": n_total,
                   "pairs_rank0": n_pairs, "cells_per_step_total": int(total_cells),
                   "l2": "inputs (%.2f GB) larger than L2, and L2 flushed between timed steps (256 MiB write)"
                         % (flat.nbytes() / 1e9),
                   "parallelism": ("dp%d: one batch list sharded by cost-balanced length bins "
                                   "(shards.plan_shards), host gather, no collective" % ws) if ws > 1 else "1 GPU",
                   "mode": ("fast FP32 + guard band (bit-exact FP32 reruns) + FP64 retry of FP32-underflowed pairs"
                            if flags & _native.FLAG_RETRY_F64 else "fast FP32 + guard band (reference f32 semantics)")},
        "roofline": {"bound": "fp32", "achieved": fast_gcups, "peak": peak, "unit": "GCUPS",
                     "frac": fast_gcups / peak, "traffic": traffic,
                     "traffic_source": "ncu --set full dram__bytes_read.sum + dram__bytes_write.sum of the workload's "
                                       "largest FP32 tiling bin, per launch (profiles/k_stream_traffic.json)",
                     "kernel": "k_stream<kFast32,P,K> FP32 streaming wavefront (all tiling bins of the FP32 phase)",
                     "algorithmic_units": "every pair's true m*n cells once (SURVEY §8(d): 8 FP32-pipe ops/cell)",
                     "peak_source": "SURVEY.md §8(d): %d SMs x %d FP32 lanes x sm_max_mhz %.0f (MEASURED_PEAKS.json) / %d ops per cell"
                                    % (nsm, FP32_LANES_PER_SM, sm_max, OPS_PER_CELL),
                     "frac_at_sampled_clock": (fast_gcups / (nsm * FP32_LANES_PER_SM * clk["sm_mhz"] * 1e6 / OPS_PER_CELL / 1e9)
                                               if clk.get("sm_mhz") else None),
                     "whole_step_frac": value / ws / peak,
                     # transparency only: the flop form, 11 flops per cell
                     # against 2 x 128 lanes x f_SM (not the denominator: 5 of the 8 ops
                     # are not FMAs); microbench FFMA2 peaks at 106 lanes/clk/SM, so 128
                     # stays the lane peak (profiles/r02_microbench_pipes.txt)
                     "flop_form": {"peak_gcups": nsm * 2 * FP32_LANES_PER_SM * sm_max * 1e6 / 11 / 1e9,
                                   "frac": fast_gcups / (nsm * 2 * FP32_LANES_PER_SM * sm_max * 1e6 / 11 / 1e9)},
                     "fast_share_of_step": float(np.mean(fast_ms) / np.mean(dev_ms)),
                     "phases_ms": dict(zip(PHASES, ph_mean.tolist())),
                     "fp64_retry": {"pairs": int(retried.sum()), "cells": retry_cells,
                                    "gcups_in_post_pass_a": (retry_cells / (ph_mean[2] * 1e-3) / 1e9) if ph_mean[2] > 0 else None,
                                    "peak_fp64_gcups": peak64}},
        "e2e": {"value": e2e_value, "unit": "GCUPS", "h2d_bytes_per_step": int(est.h2d_bytes) * ws,
                "d2h_bytes_per_step": int(est.d2h_bytes) * ws,
                "api": "phmm_score (C-ABI) from pinned host buffers" + (" + shared-memory host gather" if ws > 1 else ""),
                "call_ms_rank0": [round(x, 1) for x in call_ms]},
        "clocks": clk,
        "gpu_launches": int(launches),
        "engine": {"device_ms_mean": float(np.mean(dev_ms)), "fast_ms_mean": float(np.mean(fast_ms)),
                   "fast_ms_max_over_ranks": fast_max / args.steps * 1e3,
                   "fast_pairs": int(st.fast_pairs), "exact_pairs": int(st.exact_pairs),
                   "f64_pairs": int(st.f64_pairs), "plan_ms": float(est.plan_ms),
                   "h2d_ms": float(est.h2d_ms), "d2h_ms": float(est.d2h_ms), "shard_plan_s": t_plan,
                   "gather_complete": gathered_ok},
    }
    if not args.no_secondary and ws == 1:
        sec = []
        for name, fl in (("c2", 0), ("c3", _native.FLAG_RETRY_F64), ("c3", 0), ("c4", _native.FLAG_RETRY_F64)):
            try:
                sec.append(secondary(ctx, name, fl))
            except Exception as exc:    # reported, never fatal for the headline
                sec.append({"workload": name, "error": repr(exc)})
        line["secondary"] = sec
        try:
            line["e2e_run"] = [e2e_run("c2"), e2e_run("c3")]
        except Exception as exc:
            line["e2e_run"] = [{"error": repr(exc)}]
    if not args.no_cpu_baseline and ws == 1:          # contract: rank 0 at N = 1 only
        retry = bool(flags & _native.FLAG_RETRY_F64)
        port = cpu_baseline(full, args.cpu_seconds, retry)
        ref = reference_cpu(full, args.cpu_seconds, retry)
        line["cpu_baseline"] = dict(ref, port=port) if ref is not None else port
    print(json.dumps(line))
    if ws > 1:
        dist.destroy_process_group()
    return 0


def profile_traffic(workload):
    """dram bytes per launch of the workload's dominant k_stream launch from the committed
    ncu --set full capture (profiles/k_stream_traffic.json; c5: the largest FP32 bin)."""
    path = os.path.join(ROOT, "profiles", "k_stream_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
    except OSError:
        return None
    d = d.get(workload) if isinstance(d, dict) else None
    return d.get("dram_bytes_per_launch") if isinstance(d, dict) else None


if __name__ == "__main__":
    sys.exit(main())
