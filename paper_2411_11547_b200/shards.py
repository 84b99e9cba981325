"""Multi-GPU sharding of ONE batch list (north_star: "cost-balanced length bins with one
process or stream per GPU and a host-side gather").  Pairs are
independent, so the data path has no collective: every GPU scores its own shard and
the results are scattered back into global-id order on the host.

Plan (``plan_shards``), per READ — a read with all the haplotypes of its batch is the
engine's planning unit (phmm_engine.cu units = one read x two lanes of the batch's
haplotypes), so moving whole reads between GPUs changes neither a pair's kernel path
nor its value:

* cost of a read = the cells its FP32 stream units evaluate, padding included:
  ``W(m) * (sum of the batch's haplotype lengths + units * (P - 1))`` where ``W(m)`` is
  the engine tiling width the read pads to (the narrowest of ``TILING_WIDTHS`` >= m + 1,
  Q stripes of 512 beyond) and ``P - 1`` the wavefront fill/drain per unit;
* bins = (tiling width class, longest-haplotype bucket of 64 rows): reads of one bin run
  the same kernel instantiation with similar lane lengths, and their FP64-retry and
  guard-band rerun rates are a property of the bin (read length, haplotype length, the
  batch's qualities), not of the GPU — so dealing every bin evenly gives every GPU the
  same expected rerun cost as well as the same FP32 work;
* inside a bin reads are dealt in descending cost order, snake order over the GPUs
  (0..G-1, G-1..0, ...), the starting GPU rotated per bin: per-GPU totals differ by at
  most about one read's cost per bin.

``make_shard`` cuts a GPU's reads out as a FlatBatches (every batch with at least one of
its reads, carrying all of that batch's haplotypes) plus the global id of each of its
pairs, so the gather is ``scores[shard.gids] = shard_scores``.

Two drivers:
* ``score_sharded`` — one host process, one thread + one libphmm context per device
  (``run(devices=[...])``);
* ``HostGather`` — one process per GPU (bench.py under torchrun): the ranks scatter into a
  shared-memory result array on the host, no collective on the data path.
"""
from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np

from . import _native
from .model import FlatBatches

# FP32 stream tiling widths W = P*K of the engine (k_stream_fast32.cu: P in {4,8,16,32},
# K in {4,8,12,16}); reads with m + 1 > 512 stripe in Q = ceil((m+1)/512) stripes of 512
TILING_WIDTHS = np.array([16, 32, 48, 64, 96, 128, 192, 256, 384, 512], np.int64)
STRIPE_W = 512
ROW_BUCKET = 64

_shard_contexts = {}
_lock = threading.Lock()


def shard_context(device: int, slot: int) -> "_native.Context":
    with _lock:
        ctx = _shard_contexts.get((device, slot))
        if ctx is None:
            ctx = _native.Context(device)
            _shard_contexts[(device, slot)] = ctx
        return ctx


def _read_batch(flat: FlatBatches) -> np.ndarray:
    return np.repeat(np.arange(flat.num_batches, dtype=np.int64), np.diff(flat.batch_read_off))


def read_costs(flat: FlatBatches):
    """(cost, bin key) per read: padded cells of its FP32 stream units, (width class,
    longest-haplotype bucket)."""
    m = flat.read_len
    hl = flat.hap_len
    rb = _read_batch(flat)
    if flat.num_haps:
        hsum = np.add.reduceat(hl, flat.batch_hap_off[:-1])
        hmax = np.maximum.reduceat(hl, flat.batch_hap_off[:-1])
    else:
        hsum = hmax = np.zeros(flat.num_batches, np.int64)
    cls = np.searchsorted(TILING_WIDTHS, m + 1, side="left")
    striped = cls >= TILING_WIDTHS.shape[0]
    W = np.where(striped, -(-(m + 1) // STRIPE_W) * STRIPE_W, TILING_WIDTHS[np.minimum(cls, TILING_WIDTHS.shape[0] - 1)])
    cls = np.where(striped, TILING_WIDTHS.shape[0] + (m + 1) // STRIPE_W, cls)
    P = np.minimum(32, np.maximum(4, W // 16))
    rows = hsum[rb]
    units = np.maximum(1, -(-rows // (2 * 4096)))
    cost = W.astype(np.float64) * (rows + units * (P - 1))
    key = cls * (1 << 20) + hmax[rb] // ROW_BUCKET
    return cost, key


def plan_shards(flat: FlatBatches, parts: int) -> np.ndarray:
    """Owner GPU index (0..parts-1) of every read: bin-stratified, cost-balanced deal."""
    R = flat.num_reads
    if parts < 1:
        raise ValueError("parts must be >= 1")
    if parts == 1 or R == 0:
        return np.zeros(R, np.int64)
    cost, key = read_costs(flat)
    order = np.lexsort((-cost, key))               # by bin, then descending cost
    k_sorted = key[order]
    starts = np.flatnonzero(np.concatenate([[True], k_sorted[1:] != k_sorted[:-1]]))
    bin_id = np.cumsum(np.concatenate([[True], k_sorted[1:] != k_sorted[:-1]])) - 1
    pos = np.arange(R, dtype=np.int64) - starts[bin_id]          # rank within the bin
    rnd, lane = pos // parts, pos % parts
    snake = np.where(rnd % 2 == 0, lane, parts - 1 - lane)
    owner = np.empty(R, np.int64)
    owner[order] = (snake + bin_id) % parts
    return owner


def _ranges(starts: np.ndarray, lengths: np.ndarray) -> np.ndarray:
    """Concatenation of arange(s, s + l) for every (s, l)."""
    lengths = lengths.astype(np.int64)
    total = int(lengths.sum())
    if total == 0:
        return np.zeros(0, np.int64)
    offs = np.cumsum(lengths) - lengths
    return np.repeat(starts.astype(np.int64) - offs, lengths) + np.arange(total, dtype=np.int64)


@dataclass
class Shard:
    flat: FlatBatches          # this GPU's reads, grouped in their batches (global order kept)
    gids: np.ndarray           # int64[flat.num_pairs]: global id of each local pair
    cost: float                # planned cost (read_costs units)


def make_shard(flat: FlatBatches, owner: np.ndarray, rank: int, cost=None) -> Shard:
    """The reads ``owner == rank`` as a FlatBatches plus the global id of each pair."""
    sel = np.flatnonzero(owner == rank)
    rb = _read_batch(flat)[sel]
    H = np.diff(flat.batch_hap_off)
    ub, rcount = np.unique(rb, return_counts=True)
    rl = flat.read_len[sel]
    ridx = _ranges(flat.read_off[sel], rl)
    hsel = _ranges(flat.batch_hap_off[ub], H[ub])
    hl = flat.hap_len[hsel]
    hidx = _ranges(flat.hap_off[hsel], hl)

    def offs(lengths):
        o = np.zeros(lengths.shape[0] + 1, np.int64)
        np.cumsum(lengths, out=o[1:])
        return o

    sub = FlatBatches(read_bases=flat.read_bases[ridx], bq=flat.bq[ridx], iq=flat.iq[ridx],
                      dq=flat.dq[ridx], gq=flat.gq[ridx], read_off=offs(rl),
                      hap_bases=flat.hap_bases[hidx], hap_off=offs(hl),
                      batch_read_off=offs(rcount), batch_hap_off=offs(H[ub]))
    pair_base = np.concatenate([[0], np.cumsum(np.diff(flat.batch_read_off) * H)])
    b_all = _read_batch(flat)
    gbase = pair_base[b_all[sel]] + (sel - flat.batch_read_off[b_all[sel]]) * H[b_all[sel]]
    gids = _ranges(gbase, H[rb])
    c = float(cost[sel].sum()) if cost is not None else float(read_costs(flat)[0][sel].sum())
    return Shard(sub, gids, c)


def shards(flat: FlatBatches, parts: int):
    """All ``parts`` shards of ``flat`` (see plan_shards)."""
    owner = plan_shards(flat, parts)
    cost = read_costs(flat)[0] if flat.num_reads else np.zeros(0)
    return [make_shard(flat, owner, g, cost) for g in range(parts)]


def score_sharded(flat: FlatBatches, config_rows, flags: int, devices):
    """(scores, status, stats dict) of ``flat`` scored across ``devices`` (one host thread
    and one libphmm context per device; ctypes releases the GIL)."""
    devices = list(devices)
    n = flat.num_pairs
    parts = shards(flat, len(devices))
    scores = np.empty(n, np.float64)
    status = np.empty(n, np.uint8)
    results, errors = [None] * len(devices), [None] * len(devices)

    def work(i):
        sh = parts[i]
        if sh.flat.num_pairs == 0:
            return
        try:
            s, st, stats = shard_context(devices[i], i).score(sh.flat, config_rows, flags)
            scores[sh.gids] = s
            status[sh.gids] = st
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
    total["shard_pairs"] = [int(p.flat.num_pairs) for p in parts]
    total["shard_cost"] = [p.cost for p in parts]
    return scores, status, total


_scatter = []


def _scatter_fn():
    """phmm_scatter_results from libphmm_host.so (host-only library), or None."""
    if not _scatter:
        import ctypes
        import os
        fn = None
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libphmm_host.so")
        try:
            fn = ctypes.CDLL(path).phmm_scatter_results
            fn.restype = None
            fn.argtypes = [ctypes.c_void_p] * 5 + [ctypes.c_int64]
        except (OSError, AttributeError):
            fn = None
        _scatter.append(fn)
    return _scatter[0]


class HostGather:
    """Host-side gather for one process per GPU: a shared-memory (float64 scores, uint8
    status) array of the whole batch list; each rank scatters its shard's results at
    their global ids (``put``); after a barrier every rank — rank 0 for the report — reads
    the complete arrays.  ``name`` must be identical on all ranks; rank 0 creates the
    segment before the others attach (call ``attach`` after a barrier)."""

    def __init__(self, name: str, num_pairs: int, create: bool):
        from multiprocessing import shared_memory
        size = max(1, num_pairs * 9)
        if create:
            try:
                old = shared_memory.SharedMemory(name=name)
                old.close()
                old.unlink()
            except FileNotFoundError:
                pass
            self.shm = shared_memory.SharedMemory(name=name, create=True, size=size)
        else:
            self.shm = shared_memory.SharedMemory(name=name)
            # the creating rank owns the segment (it unlinks it); attaching ranks must not
            # have Python's resource tracker unlink it, or warn about a "leak", at exit
            try:
                from multiprocessing import resource_tracker
                resource_tracker.unregister(self.shm._name, "shared_memory")
            except (ImportError, AttributeError, KeyError):
                pass
        self.owner = create
        self.scores = np.ndarray((num_pairs,), np.float64, buffer=self.shm.buf, offset=0)
        self.status = np.ndarray((num_pairs,), np.uint8, buffer=self.shm.buf, offset=num_pairs * 8)

    def put(self, gids: np.ndarray, scores: np.ndarray, status: np.ndarray):
        """scores/status of a shard at their global ids (ascending runs: a streaming copy in
        libphmm_host.so's phmm_scatter_results; numpy fancy assignment without it)."""
        fn = _scatter_fn()
        n = int(gids.shape[0])
        if fn is None or n == 0:
            self.scores[gids] = scores
            self.status[gids] = status
            return
        g = np.ascontiguousarray(gids, dtype=np.int64)
        sc = np.ascontiguousarray(scores, dtype=np.float64)
        st = np.ascontiguousarray(status, dtype=np.uint8)
        if g.min() < 0 or g.max() >= self.scores.shape[0]:
            raise IndexError("global id out of range")
        fn(self.scores.ctypes.data, self.status.ctypes.data, g.ctypes.data, sc.ctypes.data, st.ctypes.data, n)

    def close(self):
        self.scores = self.status = None
        self.shm.close()
        if self.owner:
            try:
                self.shm.unlink()
            except FileNotFoundError:
                pass
