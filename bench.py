#!/usr/bin/env python
"""Benchmark of the Pair-HMM forward hot path (BASELINE.json metric: GCUPS).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2] [--cpu-seconds 10] [--no-secondary]

One step = one pass of the engine over the whole workload (default c2 =
BASELINE.json configs[1]: 65,536 pairs 250x250, FP32, 1 B200).  Under torchrun
each rank scores its own seeded copy of the workload on its GPU (weak scaling;
pairs are independent, no data-path collective); the timed region is bracketed
by a barrier + device sync and the time is the MAX over ranks.

  value     GCUPS with inputs resident in HBM: true cells / engine device time
            (CUDA events on the engine stream, phmm_execute), L2 flushed between steps.
  e2e       GCUPS through the C-ABI call phmm_score from pinned HOST buffers (H2D of the
            inputs, planning, kernels, D2H of scores + status, finishing), wall clock.
  roofline  the dominant kernel (k_stream, FP32 streaming wavefront) against the FP32-FMA
            roofline of SURVEY.md §8(d): 148 SMs x 128 lanes x f_SM / 8 ops per cell.
  cpu_baseline  the C oracle (a port of the reference recursion, oracle/) on the host
            cores, bounded sample of the same workload, rank 0 only.
--impl reference times that CPU port alone (the reference package itself is not
installable on the GPU box: it is numba-based and absent there).
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
    "c2": "c2: 65,536 uniform pairs 250x250 FP32 on 1xB200 (peak-kernel microbench), derived, seed 20240811+1",
    "c3": "c3: GATK-shaped 65,536 pairs, reads 50-250 x haps 100-600, derived, seed 20240811+2",
    "c1": "c1: 1,000 pairs 100x150, fixed qualities",
    "c4": "c4: 2,048 long pairs, reads 512-1024 x haps 1024-2048",
    "c5": "c5: 10M-pair mixed-length batch (reads 50-250, haps 100-600)",
}
FP32_LANES_PER_SM = 128          # tools/microbench/pipes.cu: FFMA 113/clk/SM of 128 nominal
OPS_PER_CELL = 8                 # 1 FADD + 4 FMUL + 3 FFMA per cell


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


def cpu_baseline(flat, seconds):
    """Time the C oracle (reference recursion port) on a bounded prefix of the workload."""
    from oracle import oracle
    oracle.build()
    ofl = oracle.Flat(**flat.as_dict())
    pr, ph = flat.pair_index()
    cores = os.cpu_count() or 1
    done = cells = 0
    t0 = time.perf_counter()
    chunk = 256
    while done < pr.shape[0] and time.perf_counter() - t0 < seconds:
        sl = slice(done, min(done + chunk, pr.shape[0]))
        oracle.score_raw(ofl, "f32", 120, threads=cores, pairs=(pr[sl], ph[sl]))
        cells += int((flat.read_len[pr[sl]] * flat.hap_len[ph[sl]]).sum())
        done = sl.stop
        chunk = min(chunk * 2, 8192)
    dt = time.perf_counter() - t0
    return {"value": cells / dt / 1e9, "unit": "GCUPS", "cores": cores, "kind": "port",
            "sample": "first %d of %d pairs (%.3g cells) of the same workload, FP32, oracle/phmm_oracle.c "
                      "with %d threads, %.1f s" % (done, pr.shape[0], cells, cores, dt)}


def run_reference(args, ws, rank):
    """--impl reference: the CPU port of the reference recursion on all host cores."""
    if rank != 0:
        return 0
    from paper_2411_11547_b200 import datagen
    flat = datagen.workload(args.workload)
    per_step = []
    base = None
    for i in range(args.warmup + args.steps):
        b = cpu_baseline(flat, args.cpu_seconds / max(1, args.steps))
        if i >= args.warmup:
            per_step.append(b["value"])
            base = b
    v = statistics.mean(per_step)
    base = dict(base, value=v)
    line = {"impl": "reference", "metric": "GCUPS (cell updates/s)", "value": v, "unit": "GCUPS",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
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


def shard_seed_offset(rank):
    """Weak scaling: rank r scores its own copy of the workload drawn with seed + r."""
    return int(rank)


def secondary(ctx, name, flags, steps=3):
    """Device GCUPS of another BASELINE config on the same engine (reported, not headline)."""
    from paper_2411_11547_b200 import datagen, default_configs
    from paper_2411_11547_b200.pipeline import config_tuples
    flat = datagen.workload(name)
    cfg = config_tuples(default_configs("f32"))
    ctx.prepare(flat, cfg, flags)
    ctx.execute()
    ms, fast = [], []
    for _ in range(steps):
        ctx.execute()
        d, f, _n = ctx.last_timing()
        ms.append(d)
        fast.append(f)
    _, _, st = ctx.fetch()
    cells = st.total_cells
    return {"workload": WORKLOAD_TEXT.get(name, name), "gcups": cells / (np.mean(ms) * 1e-3) / 1e9,
            "pairs": st.num_pairs, "cells": cells, "fast_pairs": st.fast_pairs,
            "exact_pairs": st.exact_pairs, "f64_retry_pairs": st.f64_pairs,
            "device_ms": float(np.mean(ms)), "fast_ms": float(np.mean(fast)),
            "flags": "retry_f64" if flags & 1 else "reference-f32"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2")
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

    build_native()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    flat = datagen.workload(args.workload, seed_offset=shard_seed_offset(rank))
    cfg = config_tuples(default_configs("f32"))
    flags = 0                                        # reference f32 semantics (c2 has no underflow)
    ctx = _native.Context(local)
    n_pairs = ctx.prepare(flat, cfg, flags)
    l2_flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        ctx.execute()
    barrier()
    dev_ms, fast_ms = [], []
    launches = 0
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            l2_flush.zero_()
            torch.cuda.synchronize()
            ctx.execute()
            d, f, n = ctx.last_timing()          # CUDA events on the engine stream
            dev_ms.append(d)
            fast_ms.append(f)
            launches += n
        barrier()
    scores, status, st = ctx.fetch()
    cells = st.total_cells
    t_max, total_cells = reduce_time_cells(float(np.sum(dev_ms)) * 1e-3, cells, ws, "cuda")
    value = total_cells * args.steps / t_max / 1e9

    # ---- e2e through the C-ABI from pinned host buffers (phmm_score)
    # (caller-owned result buffers, reused across calls like any C-ABI caller's)
    pflat = pinned_copy(flat)
    res = np.empty(pflat.num_pairs, np.float64)
    res_st = np.empty(pflat.num_pairs, np.uint8)
    for _ in range(2):
        ctx.score(pflat, cfg, flags, out=res, status=res_st)
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        out, ost, est = ctx.score(pflat, cfg, flags, out=res, status=res_st)
    torch.cuda.synchronize()
    e2e_max, _ = reduce_time_cells(time.perf_counter() - t0, 0, ws, "cuda")
    e2e_value = total_cells * args.steps / e2e_max / 1e9

    if rank != 0:
        dist.destroy_process_group() if ws > 1 else None
        return 0

    peaks = measured_peaks()
    clk = clocks.summary()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    props = torch.cuda.get_device_properties(local)
    nsm = props.multi_processor_count
    peak = nsm * FP32_LANES_PER_SM * sm_max * 1e6 / OPS_PER_CELL / 1e9
    fast_gcups = cells / (float(np.mean(fast_ms)) * 1e-3) / 1e9
    traffic = profile_traffic()
    line = {
        "metric": "GCUPS (cell updates/s)", "value": value, "unit": "GCUPS", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": WORKLOAD_TEXT.get(args.workload, args.workload), "pairs_per_gpu": n_pairs,
                   "cells_per_step_per_gpu": cells, "l2": "flushed between timed steps (256 MiB write)",
                   "parallelism": "dp%d: independent per-GPU shards, no collective" % ws,
                   "mode": "fast FP32 + guard band + exact FP32 (reference f32 semantics)"},
        "roofline": {"bound": "fp32", "achieved": fast_gcups, "peak": peak, "unit": "GCUPS",
                     "frac": fast_gcups / peak, "traffic": traffic,
                     "kernel": "k_stream<FP32,16,16> (FP32 streaming wavefront)",
                     "peak_source": "SURVEY.md §8(d): %d SMs x %d FP32 lanes x sm_max_mhz %.0f (MEASURED_PEAKS.json) / %d ops per cell"
                                    % (nsm, FP32_LANES_PER_SM, sm_max, OPS_PER_CELL),
                     "frac_at_sampled_clock": (fast_gcups / (nsm * FP32_LANES_PER_SM * clk["sm_mhz"] * 1e6 / OPS_PER_CELL / 1e9)
                                               if clk.get("sm_mhz") else None),
                     "fast_share_of_step": float(np.mean(fast_ms) / np.mean(dev_ms))},
        "e2e": {"value": e2e_value, "unit": "GCUPS", "h2d_bytes_per_step": int(est.h2d_bytes),
                "d2h_bytes_per_step": int(est.d2h_bytes)},
        "clocks": clk,
        "gpu_launches": int(launches),
        "engine": {"device_ms_mean": float(np.mean(dev_ms)), "fast_ms_mean": float(np.mean(fast_ms)),
                   "fast_pairs": int(st.fast_pairs), "exact_pairs": int(st.exact_pairs),
                   "f64_pairs": int(st.f64_pairs), "plan_ms": float(est.plan_ms),
                   "h2d_ms": float(est.h2d_ms), "d2h_ms": float(est.d2h_ms)},
    }
    if not args.no_secondary and ws == 1:
        try:
            # c3 with the GATK FP64 retry and with the reference's own FP32 semantics
            # (flagged pairs NaN, pipeline.py has no automatic retry); c4 long pairs
            line["secondary"] = [secondary(ctx, "c3", _native.FLAG_RETRY_F64), secondary(ctx, "c3", 0),
                                 secondary(ctx, "c4", _native.FLAG_RETRY_F64)]
        except Exception as exc:    # reported, never fatal for the headline
            line["secondary"] = [{"error": repr(exc)}]
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(flat, args.cpu_seconds)
    print(json.dumps(line))
    if ws > 1:
        dist.destroy_process_group()
    return 0


def profile_traffic():
    """dram bytes per k_stream launch (c2) from the committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", "k_stream_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except OSError:
        return None


if __name__ == "__main__":
    sys.exit(main())
