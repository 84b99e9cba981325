"""CPU oracle for the Pair-HMM forward hot path — TEST INFRASTRUCTURE ONLY.

Wraps oracle/liboracle.so (phmm_oracle.c, a plain-C restatement of the
reference recursion) with numpy helpers.  Only tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline legs import this module; the product package
(paper_2411_11547_b200) never does.

Reference anchors (/root/reference/pkg/src/pairhmm):
  PHRED_TO_PROB          prob.py:34-36   (scalar CPython pow per entry)
  enumeration order      model.py:123-136 (batch-major, read-major, hap-minor)
  config selection       partition.py:20-37 (smallest p*k >= m, ties -> fewer lanes)
  finishing              wavefront.py:428-434 (flag acc<=0 / non-finite, log10 - s*log10 2)
  run() error kinds      pipeline.py:94-96, wavefront.py:474-493

Parity of this restatement is pinned by tests/test_oracle_golden.py against
tests/golden/*.npz, which tests/golden/make_golden.py produced by importing
and running the reference package itself.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

# Phred -> probability, scalar CPython evaluation exactly like prob.py:36.
PHRED_TO_PROB = np.array([10.0 ** (-q / 10.0) for q in range(94)])
LOG10_2 = np.log10(2.0)          # prob.py:41

OK, OVERFLOW, TOO_SMALL, DEGENERATE = 0, 1, 2, 3
KIND = {OVERFLOW: "numeric-overflow", TOO_SMALL: "config-too-small",
        DEGENERATE: "degenerate-transition"}

_lib = None


def build():
    """Compile liboracle.so with the committed Makefile (gcc only)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        p = ctypes.c_void_p
        L.oracle_score_pairs.argtypes = [p, p, p, p, p, p, p, p, p, p, ctypes.c_int64,
                                         ctypes.c_int, ctypes.c_int, ctypes.c_int, p,
                                         ctypes.c_int, p, p]
        L.oracle_score_pairs.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class Flat:
    """Flat arrays of a batch list (same layout as the engine C-ABI)."""

    FIELDS = ("read_bases", "bq", "iq", "dq", "gq", "read_off", "hap_bases", "hap_off",
              "batch_read_off", "batch_hap_off")

    def __init__(self, **kw):
        for name in self.FIELDS:
            setattr(self, name, np.ascontiguousarray(kw[name]))

    @classmethod
    def from_batches(cls, batches):
        """Flatten reference-style Batch objects (duck-typed)."""
        reads = [r for b in batches for r in b.reads]
        haps = [h for b in batches for h in b.haps]

        def cat(arrs, dtype):
            return (np.concatenate(arrs).astype(dtype) if arrs
                    else np.zeros(0, dtype))

        def offs(arrs):
            o = np.zeros(len(arrs) + 1, np.int64)
            np.cumsum([a.shape[0] for a in arrs], out=o[1:])
            return o

        rb = [r.bases for r in reads]
        return cls(read_bases=cat(rb, np.int8),
                   bq=cat([r.base_qual for r in reads], np.uint8),
                   iq=cat([r.ins_qual for r in reads], np.uint8),
                   dq=cat([r.del_qual for r in reads], np.uint8),
                   gq=cat([r.gcp_qual for r in reads], np.uint8),
                   read_off=offs(rb),
                   hap_bases=cat([h.bases for h in haps], np.int8),
                   hap_off=offs([h.bases for h in haps]),
                   batch_read_off=np.concatenate([[0], np.cumsum([len(b.reads) for b in batches])]).astype(np.int64),
                   batch_hap_off=np.concatenate([[0], np.cumsum([len(b.haps) for b in batches])]).astype(np.int64))

    @classmethod
    def from_npz(cls, z):
        return cls(**{name: z[name] for name in cls.FIELDS})

    def as_dict(self):
        return {name: getattr(self, name) for name in self.FIELDS}


def enumerate_pairs(batch_read_off, batch_hap_off):
    """(pair_read, pair_hap) global indices in global_id order (model.py:123-136)."""
    R = np.diff(batch_read_off)
    H = np.diff(batch_hap_off)
    N = R * H
    total = int(N.sum())
    if total == 0:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    b = np.repeat(np.arange(len(N)), N)
    start = np.concatenate([[0], np.cumsum(N)[:-1]])
    k = np.arange(total, dtype=np.int64) - start[b]
    pair_read = batch_read_off[b] + k // H[b]
    pair_hap = batch_hap_off[b] + k % H[b]
    return pair_read.astype(np.int64), pair_hap.astype(np.int64)


def score_raw(flat, precision="f32", scale_log2=None, max_m=1024, threads=None,
              pairs=None):
    """Raw accumulators + OR_* status per pair (global_id order unless ``pairs``)."""
    if scale_log2 is None:
        scale_log2 = 120 if precision == "f32" else 0
    if pairs is None:
        pairs = enumerate_pairs(flat.batch_read_off, flat.batch_hap_off)
    pr, ph = (np.ascontiguousarray(a, dtype=np.int64) for a in pairs)
    n = pr.shape[0]
    acc = np.empty(n, np.float64)
    st = np.empty(n, np.uint8)
    if n:
        lut = np.ascontiguousarray(PHRED_TO_PROB)
        lib().oracle_score_pairs(
            _ptr(flat.read_bases), _ptr(flat.bq), _ptr(flat.iq), _ptr(flat.dq), _ptr(flat.gq),
            _ptr(flat.read_off), _ptr(flat.hap_bases), _ptr(flat.hap_off), _ptr(pr), _ptr(ph),
            n, 0 if precision == "f32" else 1, int(scale_log2), int(max_m), _ptr(lut),
            int(threads or os.cpu_count() or 1), _ptr(acc), _ptr(st))
    return acc, st


def finish(acc, status, scale_log2):
    """log10 scores exactly as wavefront._finish_value (math.log10 per item)."""
    out = np.full(acc.shape[0], np.nan)
    off = scale_log2 * LOG10_2
    for i in np.flatnonzero(status == OK):
        out[i] = math.log10(float(acc[i])) - off
    return out


def score(flat, precision="f32", scale_log2=None, max_m=1024, threads=None):
    """(scores float64[N], status uint8[N]) with the reference run() semantics."""
    if scale_log2 is None:
        scale_log2 = 120 if precision == "f32" else 0
    acc, st = score_raw(flat, precision, scale_log2, max_m, threads)
    return finish(acc, st, scale_log2), st
