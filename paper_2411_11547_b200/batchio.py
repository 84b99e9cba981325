"""Batch text format and score output (drop-in for the reference's batchio.py:1-159).

Format (UTF-8, '#' starts a comment, blank lines ignored):

    BATCH <num_reads> <num_haps>
    READ <bases> <baseQ> <insQ> <delQ> <gcpQ>     x num_reads
    HAP <bases>                                    x num_haps

Quality strings are Phred+33; the five READ fields have equal length.  Scores are
written one line per work item, ``<batch> <read> <hap> <value>`` (``%.6f``) in
enumeration order, or ``<batch> <read> <hap> ERROR:<kind>``, followed by a
``# cells=... seconds=... gcups=...`` comment when a run report is attached.

The engine path reads and writes through libphmm_host.so (csrc/batchio.cpp): the file
goes straight into the flat C-ABI arrays (``parse_batch_file_flat``) and scores come out
of one native writer, so a c5-sized file (10M items) needs no per-read Python objects.
Input the native reader does not take verbatim (any syntax or content error, non-ASCII
text, a lone carriage return) is re-read by ``_parse_lines`` below, which follows the
reference parser line for line (batchio.py:50-108) and raises its ParseError messages.
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

from .errors import DataError, ParseError
from .model import Batch, FlatBatches, Haplotype, ReadRecord, decode_bases, encode_bases

_PHRED_OFFSET = 33
_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libphmm_host.so")
_lib = None


def _host():
    """libphmm_host.so (built by build.build_host; g++ only, no CUDA)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            from .build import build_host
            build_host()
        L = ctypes.CDLL(_LIB)
        vp, i64 = ctypes.c_void_p, ctypes.c_int64
        L.phmm_io_parse.restype = vp
        L.phmm_io_parse.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int)]
        L.phmm_io_sizes.argtypes = [vp] + [ctypes.POINTER(i64)] * 5
        L.phmm_io_copy.argtypes = [vp] * 11
        L.phmm_io_free.argtypes = [vp]
        L.phmm_io_write_batches.restype = ctypes.c_int
        L.phmm_io_write_batches.argtypes = [ctypes.c_char_p] + [vp] * 10 + [i64]
        L.phmm_io_write_scores.restype = ctypes.c_int
        L.phmm_io_write_scores.argtypes = [ctypes.c_char_p, vp, vp, i64, vp, vp, vp, ctypes.c_char_p]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


# ---- Phred strings (batchio.py:24-40)

def decode_phred_string(text: str) -> np.ndarray:
    """Phred+33 string -> uint8 array; DataError names the first illegal position."""
    raw = np.frombuffer(text.encode("utf-32-le"), dtype=np.uint32).astype(np.int64) - _PHRED_OFFSET
    bad = np.flatnonzero((raw < 0) | (raw > 93))
    if bad.size:
        pos = int(bad[0])
        raise DataError("illegal quality character %r at position %d" % (text[pos], pos + 1))
    return raw.astype(np.uint8)


def encode_phred_string(qual) -> str:
    return (np.asarray(qual, dtype=np.uint8) + _PHRED_OFFSET).tobytes().decode("ascii")


# ---- reading

def _parse_lines(path) -> list:
    """The reference parser's semantics, line for line (batchio.py:50-108): every error
    names the offending (1-based) line."""
    with open(path, "r", encoding="utf-8") as handle:
        lines = [(no, raw.strip()) for no, raw in enumerate(handle, start=1)]
    lines = [(no, text) for no, text in lines if text and not text.startswith("#")]
    pos = 0

    def take(expected):
        nonlocal pos
        if pos >= len(lines):
            raise ParseError("unexpected end of file, expected %s" % expected,
                             lines[-1][0] if lines else 0)
        pos += 1
        return lines[pos - 1]

    batches = []
    while pos < len(lines):
        no, text = take("BATCH header")
        f = text.split()
        if f[0] != "BATCH":
            raise ParseError("expected BATCH header, got %r" % f[0], no)
        if len(f) != 3:
            raise ParseError("BATCH header needs <num_reads> <num_haps>", no)
        try:
            nr, nh = int(f[1]), int(f[2])
        except ValueError:
            raise ParseError("BATCH counts must be integers", no) from None
        if nr < 1 or nh < 1:
            raise ParseError("BATCH counts must be >= 1", no)
        reads = []
        for _ in range(nr):
            no, text = take("READ record")
            f = text.split()
            if f[0] != "READ":
                raise ParseError("expected READ record, got %r" % f[0], no)
            if len(f) != 6:
                raise ParseError("READ needs <bases> <baseQ> <insQ> <delQ> <gcpQ>", no)
            for name, track in zip(("baseQ", "insQ", "delQ", "gcpQ"), f[2:]):
                if len(track) != len(f[1]):
                    raise ParseError("%s length %d does not match %d bases"
                                     % (name, len(track), len(f[1])), no)
            try:
                reads.append(ReadRecord(encode_bases(f[1]), *(decode_phred_string(t) for t in f[2:])))
            except DataError as exc:
                raise ParseError(str(exc), no) from None
        haps = []
        for _ in range(nh):
            no, text = take("HAP record")
            f = text.split()
            if f[0] != "HAP":
                raise ParseError("expected HAP record, got %r" % f[0], no)
            if len(f) != 2:
                raise ParseError("HAP needs exactly one base string", no)
            try:
                haps.append(Haplotype(encode_bases(f[1])))
            except DataError as exc:
                raise ParseError(str(exc), no) from None
        batches.append(Batch(tuple(reads), tuple(haps)))
    return batches


def parse_batch_file_flat(path) -> FlatBatches:
    """Parse a batch file straight into the flat C-ABI arrays (native reader)."""
    L = _host()
    rc = ctypes.c_int(0)
    h = L.phmm_io_parse(os.fsencode(path), ctypes.byref(rc))
    if not h:
        if rc.value == 1:                    # not canonical: the reference's reading / error
            return FlatBatches.from_batches(_parse_lines(path))
        raise OSError("cannot read batch file %r" % (path,))
    try:
        n = [ctypes.c_int64() for _ in range(5)]
        L.phmm_io_sizes(h, *[ctypes.byref(x) for x in n])
        RL, HL, R, H, B = (x.value for x in n)
        arr = dict(read_bases=np.empty(RL, np.int8), bq=np.empty(RL, np.uint8), iq=np.empty(RL, np.uint8),
                   dq=np.empty(RL, np.uint8), gq=np.empty(RL, np.uint8), read_off=np.empty(R + 1, np.int64),
                   hap_bases=np.empty(HL, np.int8), hap_off=np.empty(H + 1, np.int64),
                   batch_read_off=np.empty(B + 1, np.int64), batch_hap_off=np.empty(B + 1, np.int64))
        L.phmm_io_copy(h, *[_p(arr[k]) for k in FlatBatches.FIELDS])
    finally:
        L.phmm_io_free(h)
    return FlatBatches(**arr)


def parse_batch_file(path) -> list:
    """Parse a batch file into Batch objects (the reference's return type)."""
    return parse_batch_file_flat(path).to_batches()


# ---- writing

def _flat(batches) -> FlatBatches:
    return batches if isinstance(batches, FlatBatches) else FlatBatches.from_batches(batches)


def write_batch_file(path, batches):
    """Write a batch list (Batch objects or FlatBatches) in the batch text format."""
    f = _flat(batches)
    rc = _host().phmm_io_write_batches(os.fsencode(path), *[_p(getattr(f, k)) for k in FlatBatches.FIELDS],
                                       f.num_batches)
    if rc != 0:
        raise OSError("cannot write batch file %r" % (path,))


def format_score_lines(batches, scores, errors) -> list:
    """Score lines in (batch, read, hap) enumeration order; failed items carry their error
    kind instead of a value (batchio.py:126-145)."""
    f = _flat(batches)
    kind_of = dict(errors)
    R = np.diff(f.batch_read_off)
    H = np.diff(f.batch_hap_off)
    lines = []
    gid = 0
    for b in range(f.num_batches):
        for r in range(int(R[b])):
            for h in range(int(H[b])):
                value = float(scores[gid])
                if gid in kind_of or math.isnan(value):
                    lines.append("%d %d %d ERROR:%s" % (b, r, h, kind_of.get(gid, "unscored")))
                else:
                    lines.append("%d %d %d %.6f" % (b, r, h, value))
                gid += 1
    return lines


def write_scores(path, batches, scores, errors, report=None):
    """format_score_lines to a file (+ the report comment), native writer."""
    f = _flat(batches)
    n = f.num_pairs
    scores = np.ascontiguousarray(scores, dtype=np.float64)
    if scores.shape[0] != n:
        raise DataError("%d scores for %d work items" % (scores.shape[0], n))
    kinds = np.full(n, -1, np.int8)
    names = []
    index = {}
    for gid, kind in errors:
        if kind not in index:
            index[kind] = len(names)
            names.append(kind.encode())
        kinds[int(gid)] = index[kind]
    name_arr = (ctypes.c_char_p * max(1, len(names)))(*names) if names else (ctypes.c_char_p * 1)()
    footer = None
    if report is not None:
        footer = ("# cells=%d seconds=%.6f gcups=%.6f\n"
                  % (report.total_cells, report.wall_seconds, report.gcups)).encode()
    rc = _host().phmm_io_write_scores(os.fsencode(path), _p(f.batch_read_off), _p(f.batch_hap_off),
                                      f.num_batches, _p(scores), _p(kinds),
                                      ctypes.cast(name_arr, ctypes.c_void_p), footer)
    if rc != 0:
        raise OSError("cannot write scores to %r" % (path,))


__all__ = ["decode_phred_string", "encode_phred_string", "parse_batch_file", "parse_batch_file_flat",
           "write_batch_file", "format_score_lines", "write_scores", "decode_bases"]
