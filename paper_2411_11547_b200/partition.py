"""Read-length binning and memory-bounded chunking (mirror of reference partition.py).

select_config / build_plan / estimate_item_bytes keep the reference semantics
(partition.py:20-139): each read binds to the registered configuration with the
smallest p*k >= m, ties to fewer lanes; the haplotype never matters; chunks are
contiguous global-id ranges whose estimated footprint fits the budget, and one
item over budget is a BudgetError.

The CUDA engine does its own, finer binning (csrc/phmm_engine.cu: per-unit
(P, K, stripes) chosen by a cost model over read AND haplotype length, LPT order);
this module is the reference-visible planning API and the source of the
RunReport.per_config keys.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import BudgetError, ConfigTooSmallError
from .model import FlatBatches, WorkItem, enumerate_work_items

DEFAULT_BUDGET_BYTES = 512 * 1024 * 1024


def select_config(m: int, configs):
    """Smallest configuration with p*k >= m; ties broken by fewer lanes."""
    fitting = [c for c in configs if c.m_max >= m]
    if not fitting:
        raise ConfigTooSmallError("no registered configuration holds a read of length %d" % m)
    return min(fitting, key=lambda c: (c.m_max, c.p))


def estimate_item_bytes(read_len: int, hap_len: int, cfg) -> int:
    """Live bytes of one item: padded read, 4 quality tracks, haplotype, staged
    emission + transition tables (5 + 5 rows of m_max reals), score slot."""
    real = np.dtype(cfg.dtype).itemsize
    return cfg.m_max + 4 * read_len + hap_len + 10 * cfg.m_max * real + 8


def config_index(read_len: np.ndarray, configs) -> np.ndarray:
    """Vectorised select_config: index into ``configs`` per read, -1 when none fits."""
    if not configs:
        return np.full(read_len.shape[0], -1, np.int64)
    order = sorted(range(len(configs)), key=lambda i: (configs[i].m_max, configs[i].p))
    caps = np.array([configs[i].m_max for i in order], np.int64)
    pos = np.searchsorted(caps, read_len, side="left")
    out = np.full(read_len.shape[0], -1, np.int64)
    ok = pos < caps.shape[0]
    out[ok] = np.array(order, np.int64)[pos[ok]]
    return out


@dataclass(frozen=True)
class Chunk:
    start: int
    stop: int
    bytes_estimate: int


@dataclass(frozen=True)
class PartitionPlan:
    items: tuple
    by_config: dict
    chunks: tuple


def item_bytes(flat: FlatBatches, configs):
    """Per-pair footprint estimate (int64, -1 for unassignable) in global_id order."""
    cfg_idx = config_index(flat.read_len, configs)
    pr, ph = flat.pair_index()
    cidx = cfg_idx[pr]
    est = np.full(pr.shape[0], -1, np.int64)
    ok = cidx >= 0
    if ok.any():
        mmax = np.array([c.m_max for c in configs], np.int64)
        real = np.array([np.dtype(c.dtype).itemsize for c in configs], np.int64)
        ci = cidx[ok]
        est[ok] = (mmax[ci] + 4 * flat.read_len[pr[ok]] + flat.hap_len[ph[ok]]
                   + 10 * mmax[ci] * real[ci] + 8)
    return est, cidx


def check_budget(flat: FlatBatches, configs, budget_bytes: int):
    """Raise BudgetError for the first item (global_id order) over the budget.

    O(reads + haplotypes): an item's estimate grows with its haplotype length, so a read
    has an item over budget iff its batch's longest haplotype exceeds the read's slack
    (budget - the read's part of the estimate); only that read's items are expanded."""
    R = flat.num_reads
    if R == 0:
        return
    cidx = config_index(flat.read_len, configs)
    ok = cidx >= 0
    if not ok.any():
        return
    mmax = np.array([c.m_max for c in configs], np.int64)
    real = np.array([np.dtype(c.dtype).itemsize for c in configs], np.int64)
    ci = np.where(ok, cidx, 0)
    base = mmax[ci] + 4 * flat.read_len + 10 * mmax[ci] * real[ci] + 8
    rb = np.repeat(np.arange(flat.num_batches), np.diff(flat.batch_read_off))
    hmax = np.maximum.reduceat(flat.hap_len, flat.batch_hap_off[:-1]) if flat.num_haps else np.zeros(0, np.int64)
    over = np.flatnonzero(ok & (base + hmax[rb] > budget_bytes))
    if over.size:
        r = int(over[0])
        b = int(rb[r])
        h0, h1 = int(flat.batch_hap_off[b]), int(flat.batch_hap_off[b + 1])
        est = base[r] + flat.hap_len[h0:h1]
        k = int(np.flatnonzero(est > budget_bytes)[0])
        H = h1 - h0
        gid = int((np.diff(flat.batch_read_off) * np.diff(flat.batch_hap_off))[:b].sum()
                  + (r - int(flat.batch_read_off[b])) * H + k)
        raise BudgetError("work item %d alone needs ~%d bytes, over the %d-byte budget"
                          % (gid, int(est[k]), budget_bytes))


def cut_chunks(est: np.ndarray, budget_bytes: int) -> tuple:
    """Greedy contiguous chunks over assignable items (partition.py:88-119)."""
    chunks = []
    start = last = None
    acc = 0
    for gid in np.flatnonzero(est >= 0).tolist():
        e = int(est[gid])
        if start is None:
            start, acc = gid, e
        elif acc + e > budget_bytes:
            chunks.append(Chunk(start, last + 1, acc))
            start, acc = gid, e
        else:
            acc += e
        last = gid
    if start is not None:
        chunks.append(Chunk(start, last + 1, acc))
    return tuple(chunks)


def build_plan(batches, configs, budget_bytes: int = DEFAULT_BUDGET_BYTES) -> PartitionPlan:
    """Bind every item to a configuration and cut chunk boundaries; the first read
    no configuration holds raises ConfigTooSmallError."""
    if not configs:
        raise ConfigTooSmallError("no configurations registered")
    flat = FlatBatches.from_batches(batches)
    items = enumerate_work_items(batches)
    cfg_idx = config_index(flat.read_len, configs)
    pr, _ = flat.pair_index()
    cidx = cfg_idx[pr] if pr.shape[0] else np.zeros(0, np.int64)
    bad = np.flatnonzero(cidx < 0)
    if bad.size:
        item: WorkItem = items[int(bad[0])]
        m = batches[item.batch_index].reads[item.read_index].length
        raise ConfigTooSmallError("read %d of batch %d (length %d) exceeds every registered "
                                  "configuration" % (item.read_index, item.batch_index, m))
    by_config = {}
    for i, cfg in enumerate(configs):
        by_config.setdefault(cfg, []).extend(np.flatnonzero(cidx == i).tolist())
    check_budget(flat, configs, budget_bytes)
    est, _ = item_bytes(flat, configs)
    return PartitionPlan(tuple(items), by_config, cut_chunks(est, budget_bytes))
