"""Multi-GPU sharding of one batch list (north_star: "cost-balanced length bins with one
process or stream per GPU and a host-side gather"; no collective — pairs are independent).

    scores, status, stats = score_sharded(flat, configs, flags, devices=[0, 1, 2, 3])

The batches are cut into ``len(devices)`` contiguous ranges of ~equal estimated cost
(sum over the range of pairs x m x n, the wavefront's cell count), so every shard owns a
contiguous range of global ids and the gather is a concatenation.  Each shard is scored
by its own libphmm context on its device from one host thread per device (ctypes
releases the GIL, so the shards run concurrently); the contexts are cached per
(device, shard slot), so ``devices=[0, 0]`` exercises the same path on a single GPU.
"""
from __future__ import annotations

import threading

import numpy as np

from . import _native
from .model import FlatBatches

_shard_contexts = {}
_lock = threading.Lock()


def shard_context(device: int, slot: int) -> "_native.Context":
    with _lock:
        ctx = _shard_contexts.get((device, slot))
        if ctx is None:
            ctx = _native.Context(device)
            _shard_contexts[(device, slot)] = ctx
        return ctx


def batch_costs(flat: FlatBatches) -> np.ndarray:
    """Cells per batch: sum over its reads and haplotypes of m x n."""
    rl, hl = flat.read_len, flat.hap_len
    rsum = np.add.reduceat(rl, flat.batch_read_off[:-1]) if flat.num_reads else np.zeros(0)
    hsum = np.add.reduceat(hl, flat.batch_hap_off[:-1]) if flat.num_haps else np.zeros(0)
    return rsum.astype(np.float64) * hsum.astype(np.float64)


def cut_points(costs: np.ndarray, parts: int) -> np.ndarray:
    """Batch boundaries of ``parts`` contiguous ranges with ~equal total cost."""
    B = costs.shape[0]
    cum = np.concatenate([[0.0], np.cumsum(costs)])
    goals = cum[-1] * np.arange(1, parts) / parts
    inner = np.searchsorted(cum, goals, side="left")
    cuts = np.concatenate([[0], np.clip(inner, 0, B), [B]]).astype(np.int64)
    return np.maximum.accumulate(cuts)


def sub_flat(flat: FlatBatches, b0: int, b1: int) -> FlatBatches:
    """The batches [b0, b1) as a FlatBatches with rebased offsets (array views)."""
    r0, r1 = int(flat.batch_read_off[b0]), int(flat.batch_read_off[b1])
    h0, h1 = int(flat.batch_hap_off[b0]), int(flat.batch_hap_off[b1])
    ro0, ro1 = int(flat.read_off[r0]), int(flat.read_off[r1])
    ho0, ho1 = int(flat.hap_off[h0]), int(flat.hap_off[h1])
    return FlatBatches(read_bases=flat.read_bases[ro0:ro1], bq=flat.bq[ro0:ro1], iq=flat.iq[ro0:ro1],
                       dq=flat.dq[ro0:ro1], gq=flat.gq[ro0:ro1],
                       read_off=flat.read_off[r0:r1 + 1] - ro0,
                       hap_bases=flat.hap_bases[ho0:ho1], hap_off=flat.hap_off[h0:h1 + 1] - ho0,
                       batch_read_off=flat.batch_read_off[b0:b1 + 1] - r0,
                       batch_hap_off=flat.batch_hap_off[b0:b1 + 1] - h0)


def score_sharded(flat: FlatBatches, config_rows, flags: int, devices):
    """(scores, status, stats dict) of ``flat`` scored across ``devices``."""
    devices = list(devices)
    n = flat.num_pairs
    cuts = cut_points(batch_costs(flat), len(devices))
    pairs = np.concatenate([[0], np.cumsum(np.diff(flat.batch_read_off) * np.diff(flat.batch_hap_off))])
    scores = np.empty(n, np.float64)
    status = np.empty(n, np.uint8)
    results, errors = [None] * len(devices), [None] * len(devices)

    def work(i):
        b0, b1 = int(cuts[i]), int(cuts[i + 1])
        if b1 <= b0:
            return
        try:
            s, st, stats = shard_context(devices[i], i).score(sub_flat(flat, b0, b1), config_rows, flags)
            g0, g1 = int(pairs[b0]), int(pairs[b1])
            scores[g0:g1] = s
            status[g0:g1] = st
            results[i] = stats.as_dict()
        except Exception as exc:          # re-raised in the caller's thread
            errors[i] = exc

    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(devices))]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    for exc in errors:
        if exc is not None:
            raise exc
    total = {}
    for r in results:
        if r is None:
            continue
        for k, v in r.items():
            if k in ("device_ms", "fast_ms", "h2d_ms", "d2h_ms", "plan_ms"):
                total[k] = max(total.get(k, 0.0), v)          # shards run concurrently
            else:
                total[k] = total.get(k, 0) + v
    total["devices"] = devices
    total["shard_batches"] = np.diff(cuts).tolist()
    return scores, status, total
