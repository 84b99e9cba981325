"""Seeded synthetic inputs (restatement of reference datagen.py:78-158).

The benchmark and the GPU parity tests must run where /root/reference does not
exist, so the reference generator is restated here with the IDENTICAL sequence
of numpy Generator calls (same methods, bounds, sizes and dtypes, same order):
for a given seed the batches are element-for-element those of
pairhmm.datagen.generate_synthetic / generate_verification_pairs
(tests/test_datagen.py checks this against the reference-generated fixtures).

``generate_synthetic_flat`` draws the same stream but writes straight into the
flat C-ABI arrays (FlatBatches) without building per-read objects.
Modes: "independent" (uniform random bases) and "derived" (per batch one locus:
haplotypes are mutated prefixes of a shared sequence, reads mutated substrings).
"""
from __future__ import annotations

import numpy as np

from .errors import DataError
from .model import Batch, FlatBatches, Haplotype, ReadRecord

DEFAULT_BASE_QUAL = (10, 40)
DEFAULT_INDEL_QUAL = (30, 45)
DEFAULT_GCP_QUAL = 10
DEFAULT_MUTATION_RATE = 0.01


def _lengths(spec, what):
    if isinstance(spec, (int, np.integer)):
        if spec < 1:
            raise DataError("%s length must be >= 1, got %d" % (what, spec))
        fixed = int(spec)
        return lambda rng: fixed
    try:
        lo, hi = int(spec[0]), int(spec[1])
    except (TypeError, ValueError, IndexError):
        raise DataError("%s length spec %r is neither an int nor (min, max)" % (what, spec)) from None
    if not 1 <= lo <= hi:
        raise DataError("%s length range (%d, %d) is invalid" % (what, lo, hi))
    return lambda rng: int(rng.integers(lo, hi + 1))


def _quals(spec):
    if isinstance(spec, (int, np.integer)):
        fixed = int(spec)
        return lambda rng, size: np.full(size, fixed, dtype=np.uint8)
    lo, hi = spec
    return lambda rng, size: rng.integers(lo, hi + 1, size=size).astype(np.uint8)


def _bases(rng, length):
    return rng.integers(0, 4, size=length, dtype=np.int8)


def _mutate(rng, bases, rate):
    out = bases.copy()
    hits = rng.random(out.shape[0]) < rate
    count = int(hits.sum())
    if count:
        out[hits] = (out[hits] + rng.integers(1, 4, size=count)) % 4
    return out


def _read_from(rng, source, m, rate):
    n = source.shape[0]
    if m <= n:
        start = int(rng.integers(0, n - m + 1))
        core = source[start:start + m]
    else:
        core = np.concatenate([source, _bases(rng, m - n)])
    return _mutate(rng, core, rate)


def _stream(num_batches, reads_per_batch, haps_per_batch, read_len_spec, hap_len_spec, seed,
            mode, mutation_rate, base_qual, indel_qual, gcp_qual):
    """Yields (haps, reads) per batch; reads are (bases, bq, iq, dq, gq) tuples."""
    if mode not in ("independent", "derived"):
        raise DataError("unknown generation mode %r" % mode)
    read_len = _lengths(read_len_spec, "read")
    hap_len = _lengths(hap_len_spec, "haplotype")
    bq, iq, dq, gq = _quals(base_qual), _quals(indel_qual), _quals(indel_qual), _quals(gcp_qual)
    rng = np.random.default_rng(seed)
    for _ in range(num_batches):
        lengths = [hap_len(rng) for _ in range(haps_per_batch)]
        if mode == "independent":
            haps = [_bases(rng, n) for n in lengths]
        else:
            locus = _bases(rng, max(lengths))
            haps = [_mutate(rng, locus[:n], mutation_rate) for n in lengths]
            common = locus[:min(lengths)]
        reads = []
        for _ in range(reads_per_batch):
            m = read_len(rng)
            if mode == "independent":
                b = _bases(rng, m)
            else:
                b = _read_from(rng, common, m, mutation_rate)
            q1 = bq(rng, m)
            q2 = iq(rng, m)
            q3 = dq(rng, m)
            q4 = gq(rng, m)
            reads.append((b, q1, q2, q3, q4))
        yield haps, reads


def generate_synthetic(num_batches, reads_per_batch, haps_per_batch, read_len_spec, hap_len_spec,
                       seed, mode="independent", mutation_rate=DEFAULT_MUTATION_RATE,
                       base_qual=DEFAULT_BASE_QUAL, indel_qual=DEFAULT_INDEL_QUAL,
                       gcp_qual=DEFAULT_GCP_QUAL):
    """list[Batch], element-identical to the reference generator for the same arguments."""
    out = []
    for haps, reads in _stream(num_batches, reads_per_batch, haps_per_batch, read_len_spec,
                               hap_len_spec, seed, mode, mutation_rate, base_qual, indel_qual,
                               gcp_qual):
        out.append(Batch(tuple(ReadRecord(*r) for r in reads), tuple(Haplotype(h) for h in haps)))
    return out


def _spec3(spec, what, is_len):
    """(lo, hi, fixed) of a length / quality spec, validated like _lengths / _quals."""
    if isinstance(spec, (int, np.integer)):
        if is_len:
            _lengths(spec, what)                 # raises DataError like the reference
        return (int(spec), int(spec), 1)
    if is_len:
        _lengths(spec, what)
    lo, hi = int(spec[0]), int(spec[1])
    return (lo, hi, 0)


def _native_flat(num_batches, reads_per_batch, haps_per_batch, read_len_spec, hap_len_spec, seed,
                 mode, mutation_rate, base_qual, indel_qual, gcp_qual):
    """The same stream drawn by csrc/datagen.cpp (libphmm_host.so), or None when the
    library is not built.  Ranges must fit the 32-bit bounded draw (always true here)."""
    import ctypes
    import os
    lib_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libphmm_host.so")
    if not os.path.exists(lib_path) or num_batches < 1:
        return None
    if mode not in ("independent", "derived"):
        raise DataError("unknown generation mode %r" % mode)
    specs = [_spec3(read_len_spec, "read", True), _spec3(hap_len_spec, "haplotype", True),
             _spec3(base_qual, "base_qual", False), _spec3(indel_qual, "indel_qual", False),
             _spec3(gcp_qual, "gcp_qual", False)]
    if any(s[1] - s[0] >= (1 << 32) - 1 or s[1] < s[0] for s in specs[2:]):
        return None
    L = ctypes.CDLL(lib_path)
    vp, i64 = ctypes.c_void_p, ctypes.c_int64
    L.phmm_gen_run.restype = vp
    L.phmm_gen_run.argtypes = [ctypes.c_uint64] * 4 + [ctypes.c_int, ctypes.c_uint32, i64, i64, i64, vp, vp,
                                                       ctypes.c_int, ctypes.c_double, vp, vp, vp]
    L.phmm_gen_sizes.argtypes = [vp] + [ctypes.POINTER(i64)] * 4
    L.phmm_gen_copy.argtypes = [vp] * 9
    L.phmm_gen_free.argtypes = [vp]
    st = np.random.default_rng(seed).bit_generator.state
    s, inc = st["state"]["state"], st["state"]["inc"]
    m64 = (1 << 64) - 1
    arrs = [np.ascontiguousarray(x, np.int64) for x in specs]
    h = L.phmm_gen_run(s >> 64, s & m64, inc >> 64, inc & m64, int(st["has_uint32"]), int(st["uinteger"]),
                       num_batches, reads_per_batch, haps_per_batch,
                       *[a.ctypes.data_as(vp) for a in arrs[:2]], 1 if mode == "derived" else 0,
                       float(mutation_rate), *[a.ctypes.data_as(vp) for a in arrs[2:]])
    if not h:
        return None
    try:
        RL, HL, R, H = i64(), i64(), i64(), i64()
        L.phmm_gen_sizes(h, ctypes.byref(RL), ctypes.byref(HL), ctypes.byref(R), ctypes.byref(H))
        rb = np.empty(RL.value, np.int8)
        q = [np.empty(RL.value, np.uint8) for _ in range(4)]
        rlen = np.empty(R.value, np.int64)
        hb = np.empty(HL.value, np.int8)
        hlen = np.empty(H.value, np.int64)
        L.phmm_gen_copy(h, *[a.ctypes.data_as(vp) for a in [rb] + q + [rlen, hb, hlen]])
    finally:
        L.phmm_gen_free(h)
    ro = np.zeros(R.value + 1, np.int64)
    np.cumsum(rlen, out=ro[1:])
    ho = np.zeros(H.value + 1, np.int64)
    np.cumsum(hlen, out=ho[1:])
    return FlatBatches(read_bases=rb, bq=q[0], iq=q[1], dq=q[2], gq=q[3], read_off=ro, hap_bases=hb,
                       hap_off=ho,
                       batch_read_off=np.arange(num_batches + 1, dtype=np.int64) * reads_per_batch,
                       batch_hap_off=np.arange(num_batches + 1, dtype=np.int64) * haps_per_batch)


def generate_synthetic_flat(num_batches, reads_per_batch, haps_per_batch, read_len_spec,
                            hap_len_spec, seed, mode="independent",
                            mutation_rate=DEFAULT_MUTATION_RATE, base_qual=DEFAULT_BASE_QUAL,
                            indel_qual=DEFAULT_INDEL_QUAL, gcp_qual=DEFAULT_GCP_QUAL,
                            native=True) -> FlatBatches:
    """Same stream as generate_synthetic, returned as FlatBatches (no per-read objects).
    ``native``: draw it with libphmm_host.so (csrc/datagen.cpp, identical arrays, ~100x
    faster) when that library is built; otherwise the numpy restatement below."""
    if native:
        out = _native_flat(num_batches, reads_per_batch, haps_per_batch, read_len_spec, hap_len_spec,
                           seed, mode, mutation_rate, base_qual, indel_qual, gcp_qual)
        if out is not None:
            return out
    rb, q1, q2, q3, q4, rl, hb, hl = [], [], [], [], [], [], [], []
    for haps, reads in _stream(num_batches, reads_per_batch, haps_per_batch, read_len_spec,
                               hap_len_spec, seed, mode, mutation_rate, base_qual, indel_qual,
                               gcp_qual):
        for b, a, c, d, e in reads:
            rb.append(b); q1.append(a); q2.append(c); q3.append(d); q4.append(e); rl.append(b.shape[0])
        for h in haps:
            hb.append(h); hl.append(h.shape[0])

    def cat(arrs, dt):
        return np.concatenate(arrs).astype(dt, copy=False) if arrs else np.zeros(0, dt)

    def offs(lengths):
        o = np.zeros(len(lengths) + 1, np.int64)
        np.cumsum(lengths, out=o[1:])
        return o

    return FlatBatches(read_bases=cat(rb, np.int8), bq=cat(q1, np.uint8), iq=cat(q2, np.uint8),
                       dq=cat(q3, np.uint8), gq=cat(q4, np.uint8), read_off=offs(rl),
                       hap_bases=cat(hb, np.int8), hap_off=offs(hl),
                       batch_read_off=np.arange(num_batches + 1, dtype=np.int64) * reads_per_batch,
                       batch_hap_off=np.arange(num_batches + 1, dtype=np.int64) * haps_per_batch)


def generate_verification_pairs(num_pairs, seed, max_read_len=1024, max_hap_len=1024,
                                mutation_rate=0.005):
    """Single-pair batches spanning lengths [1, max] jointly (reference datagen.py:124-158)."""
    rng = np.random.default_rng(seed)
    bq, iq, gq = _quals((15, 40)), _quals(DEFAULT_INDEL_QUAL), _quals(DEFAULT_GCP_QUAL)
    out = []
    for _ in range(num_pairs):
        u = rng.random()
        if u < 0.10:
            m = int(rng.integers(max(1, max_read_len * 3 // 4), max_read_len + 1))
            n = int(rng.integers(min(m, max_hap_len), max_hap_len + 1))
        elif u < 0.25:
            m = n = int(rng.integers(1, min(max_read_len, max_hap_len) + 1))
        elif u < 0.30:
            n = int(rng.integers(1, max_hap_len + 1))
            m = min(n + int(rng.integers(1, 17)), max_read_len)
        else:
            n = int(rng.integers(1, max_hap_len + 1))
            m = int(rng.integers(1, min(n, max_read_len) + 1))
        hap = _bases(rng, n)
        read = _read_from(rng, hap, m, mutation_rate)
        a = bq(rng, m)
        b = iq(rng, m)
        c = iq(rng, m)
        d = gq(rng, m)
        out.append(Batch((ReadRecord(read, a, b, c, d),), (Haplotype(hap),)))
    return out


# Benchmark / parity workloads of BASELINE.json "configs", SEED as
# test_acceptance.py:28.  Each entry: generate_synthetic arguments.
SEED = 20240811
WORKLOADS = {
    "c1": dict(num_batches=10, reads_per_batch=25, haps_per_batch=4, read_len_spec=100,
               hap_len_spec=150, seed=SEED, mode="derived", base_qual=30, indel_qual=45,
               gcp_qual=10),
    "c1_independent": dict(num_batches=10, reads_per_batch=25, haps_per_batch=4, read_len_spec=100,
                           hap_len_spec=150, seed=SEED, mode="independent", base_qual=30,
                           indel_qual=45, gcp_qual=10),
    "c2": dict(num_batches=1024, reads_per_batch=16, haps_per_batch=4, read_len_spec=250,
               hap_len_spec=250, seed=SEED + 1, mode="derived"),
    "c3": dict(num_batches=128, reads_per_batch=64, haps_per_batch=8, read_len_spec=(50, 250),
               hap_len_spec=(100, 600), seed=SEED + 2, mode="derived"),
    "c4": dict(num_batches=64, reads_per_batch=8, haps_per_batch=4, read_len_spec=(512, 1024),
               hap_len_spec=(1024, 2048), seed=SEED + 3, mode="derived"),
    "c4_underflow": dict(num_batches=64, reads_per_batch=8, haps_per_batch=4,
                         read_len_spec=(512, 1024), hap_len_spec=(1024, 2048), seed=SEED + 3,
                         mode="derived", mutation_rate=0.10, base_qual=(10, 11)),
    "c5": dict(num_batches=19532, reads_per_batch=64, haps_per_batch=8, read_len_spec=(50, 250),
               hap_len_spec=(100, 600), seed=SEED + 4, mode="derived"),
}


def workload(name: str, num_batches=None, seed_offset: int = 0) -> FlatBatches:
    """FlatBatches of a named workload; ``num_batches`` takes a prefix (same stream)."""
    kw = dict(WORKLOADS[name])
    if num_batches is not None:
        kw["num_batches"] = num_batches
    kw["seed"] = kw["seed"] + seed_offset
    return generate_synthetic_flat(**kw)
