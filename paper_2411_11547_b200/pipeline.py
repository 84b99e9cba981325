"""run(): the drop-in batch-likelihood API (mirror of reference pipeline.py:77-142).

    scores, report = run(batches, configs=None, budget_bytes=512 MiB, workers=1)

Same inputs, outputs and error semantics as the reference: float64 log10 scores
in global_id order (NaN where an item failed), a RunReport whose errors are
(global_id, kind) pairs sorted by id, total_cells counting true m*n of every
executed item (numeric-overflow items included; config-too-small /
degenerate-transition / data excluded, pipeline.py:27,103-111), and GCUPS =
total_cells / wall.  BudgetError (one item over the chunk budget) and
ValueError (workers < 1) are raised like the reference.

Underneath, the whole batch list is flattened once (FlatBatches) and scored by
ONE call into libphmm.so on the GPU (GIL released).  ``workers`` is accepted
for compatibility; GPU concurrency replaces the reference thread pool.
Extra keyword-only options:
  retry_f64  rerun FP32-underflowing pairs in FP64 (GATK behaviour); such items
             get finite scores and are listed in report.retried instead of errors.
  exact      run every FP32 pair on the bit-exact kernel (no fast path).
  device     CUDA device ordinal.
  devices    list of CUDA devices: the batches are sharded across them by cost with one
             host thread (and one context) per device and gathered in global-id order
             (shards.py; north_star multi-GPU path, no collective).
  device_budget_bytes  bound on the engine's device working set: a larger batch list
             streams through three chunk contexts in budget-sized chunks (the reference's
             chunk budget, partition.py:88-119, for inputs larger than HBM); without it the
             engine streams automatically only when a call would not fit free memory.
``budget_bytes`` keeps the reference's meaning: one item estimated over it raises
BudgetError (partition.py:104-112).
"""
from __future__ import annotations

import threading
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import InvalidMeasurementError
from .model import FlatArena, FlatBatches, default_configs
from .partition import DEFAULT_BUDGET_BYTES, check_budget, config_index

_NOT_EXECUTED = ("config-too-small", "degenerate-transition", "data")


def throughput(total_cells: int, wall_seconds: float) -> float:
    """Giga cell updates per second."""
    if wall_seconds <= 0.0:
        raise InvalidMeasurementError("non-positive runtime %r" % wall_seconds)
    return total_cells / (wall_seconds * 1.0e9)


@dataclass(frozen=True)
class ConfigStats:
    cells: int
    seconds: float


@dataclass(frozen=True)
class RunReport:
    total_cells: int
    wall_seconds: float
    gcups: float
    per_config: dict = field(default_factory=dict)
    errors: list = field(default_factory=list)
    retried: list = field(default_factory=list)     # global ids rescued by the FP64 retry
    engine: dict = field(default_factory=dict)      # libphmm phmm_stats of the call


_ARENAS = threading.local()


class _PinnedArena(FlatArena):
    """The flattening arena of run(), page-locked (phmm_pin_host) so the engine's uploads
    from it are DMA transfers overlapping the host planning; re-pinned when it grows."""

    def __init__(self):
        super().__init__()
        self._pinned = []

    def alloc(self, read_bytes: int, hap_bytes: int):
        old = (self._tracks, self._haps)
        bufs = super().alloc(read_bytes, hap_bytes)
        if self._tracks is not old[0] or self._haps is not old[1] or not self._pinned:
            for a in self._pinned:
                _native.unpin_host(a)
            self._pinned = [a for a in (self._tracks, self._haps) if a.nbytes and _native.pin_host(a)]
        return bufs

    def __del__(self):
        try:
            for a in getattr(self, "_pinned", []):
                _native.unpin_host(a)
        except Exception:             # interpreter shutdown: the process releases the pages
            pass


def _arena() -> FlatArena:
    """This thread's flattening scratch (run() holds its flat arrays only for the call)."""
    a = getattr(_ARENAS, "arena", None)
    if a is None:
        a = _ARENAS.arena = _PinnedArena()
    return a


def config_tuples(configs):
    return [(c.p, c.k, 0 if c.precision == "f32" else 1, c.scale_log2) for c in configs]


def engine_flags(retry_f64: bool = False, exact: bool = False) -> int:
    return (_native.FLAG_RETRY_F64 if retry_f64 else 0) | (_native.FLAG_EXACT if exact else 0)


def score_flat(flat: FlatBatches, configs, retry_f64=False, exact=False, device=0, device_budget_bytes=None):
    """Engine call on flat arrays -> (scores, status, stats)."""
    ctx = _native.context(device)
    if device_budget_bytes is None:
        return ctx.score(flat, config_tuples(configs), engine_flags(retry_f64, exact))
    with ctx._lock:
        ctx.set_device_budget(device_budget_bytes)
        try:
            return ctx.score(flat, config_tuples(configs), engine_flags(retry_f64, exact))
        finally:
            ctx.set_device_budget(0)


# status kind -> error kind name, as an object array (one vectorised gather per call)
_KIND_NAME_ARR = np.array([_native.KIND_NAMES.get(k) for k in range(256)], dtype=object)


def errors_from_status(status: np.ndarray) -> list:
    """[(global pair id, kind name)] of the failed pairs, in pair order."""
    kinds = status & _native.ST_KIND_MASK
    bad = np.flatnonzero(kinds != _native.ST_OK)
    return list(zip(bad.tolist(), _KIND_NAME_ARR[kinds[bad]].tolist()))


def _config_cells(flat: FlatBatches, configs, status: np.ndarray, device_s: float):
    """({geometry: ConfigStats}, total executed cells) in O(reads)."""
    H = np.diff(flat.batch_hap_off)
    rb = np.repeat(np.arange(flat.num_batches), np.diff(flat.batch_read_off))
    pair_base = np.concatenate([[0], np.cumsum(np.diff(flat.batch_read_off) * H)])
    first = pair_base[rb] + (np.arange(flat.num_reads) - flat.batch_read_off[rb]) * H[rb]
    kinds = status[first] & _native.ST_KIND_MASK
    executed = (kinds == _native.ST_OK) | (kinds == _native.ST_OVERFLOW)
    hsum = np.add.reduceat(flat.hap_len, flat.batch_hap_off[:-1])
    cells = flat.read_len * hsum[rb]
    cidx = config_index(flat.read_len, configs)
    sel = executed & (cidx >= 0)
    per = np.bincount(cidx[sel], weights=cells[sel].astype(np.float64), minlength=len(configs))
    exact = np.zeros(len(configs), np.int64)
    np.add.at(exact, cidx[sel], cells[sel])
    total = int(exact.sum())
    per_config = {}
    for i in np.flatnonzero(per > 0).tolist():
        geo = configs[i].geometry
        c = int(exact[i])
        sec = device_s * c / total if total else 0.0
        prev = per_config.get(geo)
        per_config[geo] = ConfigStats(c + (prev.cells if prev else 0), sec + (prev.seconds if prev else 0.0))
    return per_config, total


def run(batches, configs=None, budget_bytes: int = DEFAULT_BUDGET_BYTES, workers: int = 1, *,
        retry_f64: bool = False, exact: bool = False, device: int = 0, devices=None,
        device_budget_bytes=None):
    """Score every work item of ``batches`` on the GPU; see the module docstring."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    if configs is None:
        configs = default_configs()
    flat = batches if isinstance(batches, FlatBatches) else FlatBatches.from_batches(batches, _arena())
    check_budget(flat, configs, budget_bytes)
    n = flat.num_pairs
    if n and not (devices is not None and len(devices) > 1):
        _native.context(devices[0] if devices else device)   # engine setup (CUDA context) is not scoring time
    t0 = time.perf_counter()
    if n and devices is not None and len(devices) > 1:
        from .shards import score_sharded
        scores, status, engine = score_sharded(flat, config_tuples(configs), engine_flags(retry_f64, exact),
                                               devices)
    elif n:
        dev = devices[0] if devices else device
        scores, status, stats = score_flat(flat, configs, retry_f64, exact, dev, device_budget_bytes)
        engine = stats.as_dict()
    else:
        scores, status, engine = np.zeros(0), np.zeros(0, np.uint8), {}
    wall = time.perf_counter() - t0
    errors = errors_from_status(status)
    retried = np.flatnonzero((status & _native.ST_RETRIED_F64) != 0).tolist()

    # per-config accounting keyed like the reference (geometry of the bound config), per
    # READ: a read's items are all executed or none (config-too-small and
    # degenerate-transition are properties of the read; numeric-overflow items count)
    per_config = {}
    total_cells = 0
    if n:
        per_config, total_cells = _config_cells(flat, configs, status, engine.get("device_ms", 0.0) * 1e-3)
    report = RunReport(total_cells, wall, throughput(total_cells, wall), per_config, errors,
                       retried, engine)
    return scores, report
