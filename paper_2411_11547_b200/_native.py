"""ctypes binding of libphmm.so (the C-ABI declared in include/phmm.h).

The library is built in-tree by __graft_entry__.build() / build.py into
paper_2411_11547_b200/_lib/libphmm.so.  There is no fallback: if the library
or a CUDA device is missing, every engine call raises EngineUnavailableError.
ctypes releases the GIL for the duration of each foreign call, like the
reference's nogil numba kernels (wavefront.py:61).
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import EngineError, EngineUnavailableError

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib")
LIB_PATH = os.path.join(LIB_DIR, "libphmm.so")

SUCCESS = 0
ST_OK, ST_OVERFLOW, ST_TOO_SMALL, ST_DEGENERATE = 0, 1, 2, 3
ST_KIND_MASK = 0x0F
ST_EXACT_F32 = 0x20
ST_RETRIED_F64 = 0x40
FLAG_RETRY_F64 = 0x1
FLAG_EXACT = 0x2

KIND_NAMES = {ST_OVERFLOW: "numeric-overflow", ST_TOO_SMALL: "config-too-small",
              ST_DEGENERATE: "degenerate-transition"}

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32


class PhmmInput(ctypes.Structure):
    _fields_ = [("read_bases", _vp), ("base_qual", _vp), ("ins_qual", _vp), ("del_qual", _vp),
                ("gcp_qual", _vp), ("read_off", _vp), ("num_reads", _i64),
                ("hap_bases", _vp), ("hap_off", _vp), ("num_haps", _i64),
                ("batch_read_off", _vp), ("batch_hap_off", _vp), ("num_batches", _i64)]


class PhmmOptions(ctypes.Structure):
    _fields_ = [("num_configs", _i32), ("p", _vp), ("k", _vp), ("precision", _vp),
                ("scale_log2", _vp), ("flags", _i32)]


class PhmmStats(ctypes.Structure):
    _fields_ = [("num_pairs", _i64), ("total_cells", _i64), ("computed_cells", _i64),
                ("fast_pairs", _i64), ("exact_pairs", _i64), ("f64_pairs", _i64),
                ("flagged_pairs", _i64), ("h2d_bytes", _i64), ("d2h_bytes", _i64),
                ("kernel_launches", _i32), ("reserved", _i32), ("device_ms", ctypes.c_double),
                ("fast_ms", ctypes.c_double), ("h2d_ms", ctypes.c_double),
                ("d2h_ms", ctypes.c_double), ("plan_ms", ctypes.c_double)]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_ if name != "reserved"}


# every symbol include/phmm.h declares (tests/test_abi.py checks the .so exports them)
EXPORTS = ("phmm_abi_version", "phmm_create", "phmm_destroy", "phmm_last_error", "phmm_score",
           "phmm_prepare", "phmm_execute", "phmm_fetch", "phmm_fast_geometry", "phmm_last_timing",
           "phmm_last_phases", "phmm_forward_matrices", "phmm_set_device_budget", "phmm_device_bytes",
           "phmm_set_pipeline", "phmm_pin_host", "phmm_unpin_host")

_lib = None


def load():
    """Load libphmm.so (raises EngineUnavailableError when it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise EngineUnavailableError(
            "libphmm.so not built at %s — run `python -c 'import __graft_entry__ as g; g.build()'`"
            % LIB_PATH)
    L = ctypes.CDLL(LIB_PATH)
    L.phmm_abi_version.restype = ctypes.c_int
    L.phmm_create.argtypes = [ctypes.POINTER(_vp), ctypes.c_int, _vp]
    L.phmm_create.restype = ctypes.c_int
    L.phmm_destroy.argtypes = [_vp]
    L.phmm_destroy.restype = ctypes.c_int
    L.phmm_last_error.argtypes = [_vp]
    L.phmm_last_error.restype = ctypes.c_char_p
    L.phmm_score.argtypes = [_vp, ctypes.POINTER(PhmmInput), ctypes.POINTER(PhmmOptions), _vp, _vp,
                             ctypes.POINTER(PhmmStats)]
    L.phmm_score.restype = ctypes.c_int
    L.phmm_prepare.argtypes = [_vp, ctypes.POINTER(PhmmInput), ctypes.POINTER(PhmmOptions),
                               ctypes.POINTER(_i64)]
    L.phmm_prepare.restype = ctypes.c_int
    L.phmm_execute.argtypes = [_vp]
    L.phmm_execute.restype = ctypes.c_int
    L.phmm_fetch.argtypes = [_vp, _vp, _vp, ctypes.POINTER(PhmmStats)]
    L.phmm_fetch.restype = ctypes.c_int
    L.phmm_fast_geometry.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                     ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
    L.phmm_fast_geometry.restype = ctypes.c_int
    L.phmm_last_timing.argtypes = [_vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                   ctypes.POINTER(ctypes.c_int)]
    L.phmm_last_timing.restype = ctypes.c_int
    L.phmm_last_phases.argtypes = [_vp, _vp]
    L.phmm_last_phases.restype = ctypes.c_int
    L.phmm_forward_matrices.argtypes = [_vp] * 6 + [_i32, _vp, _i32, _i32, _vp, _vp, _vp]
    L.phmm_forward_matrices.restype = ctypes.c_int
    L.phmm_set_device_budget.argtypes = [_vp, _i64]
    L.phmm_set_device_budget.restype = ctypes.c_int
    L.phmm_pin_host.argtypes = [_vp, _i64]
    L.phmm_pin_host.restype = ctypes.c_int
    L.phmm_unpin_host.argtypes = [_vp]
    L.phmm_unpin_host.restype = ctypes.c_int
    L.phmm_set_pipeline.argtypes = [_vp, _i32]
    L.phmm_set_pipeline.restype = ctypes.c_int
    L.phmm_device_bytes.argtypes = [_vp, ctypes.POINTER(_i64)]
    L.phmm_device_bytes.restype = ctypes.c_int
    if L.phmm_abi_version() != 1:
        raise EngineUnavailableError("libphmm ABI version mismatch")
    _lib = L
    return L


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_vp) if a is not None else None


def make_input(flat) -> tuple:
    """PhmmInput over a FlatBatches (the arrays must stay alive while it is used)."""
    s = PhmmInput(_ptr(flat.read_bases), _ptr(flat.bq), _ptr(flat.iq), _ptr(flat.dq), _ptr(flat.gq),
                  _ptr(flat.read_off), flat.num_reads, _ptr(flat.hap_bases), _ptr(flat.hap_off),
                  flat.num_haps, _ptr(flat.batch_read_off), _ptr(flat.batch_hap_off),
                  flat.num_batches)
    return s, flat


def make_options(configs, flags: int) -> tuple:
    p = np.array([c[0] for c in configs], np.int32)
    k = np.array([c[1] for c in configs], np.int32)
    prec = np.array([c[2] for c in configs], np.int32)
    scale = np.array([c[3] for c in configs], np.int32)
    s = PhmmOptions(len(configs), _ptr(p), _ptr(k), _ptr(prec), _ptr(scale), flags)
    return s, (p, k, prec, scale)


def fast_geometry(m: int, n: int):
    P, K, Q = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    load().phmm_fast_geometry(m, n, ctypes.byref(P), ctypes.byref(K), ctypes.byref(Q))
    return P.value, K.value, Q.value


class Context:
    """One libphmm context bound to one CUDA device.

    The C context is single-caller (include/phmm.h); ctypes releases the GIL, so every
    entry point here takes the context's lock: concurrent callers of one Context (e.g.
    two threads calling run()) are serialized instead of racing on device buffers."""

    def __init__(self, device: int = 0, lut=None):
        from .prob import PHRED_TO_PROB
        self._lock = threading.RLock()
        L = load()
        self._lut = np.ascontiguousarray(PHRED_TO_PROB if lut is None else lut, dtype=np.float64)
        h = _vp()
        rc = L.phmm_create(ctypes.byref(h), int(device), _ptr(self._lut))
        self._h = h
        self._L = L
        if rc != SUCCESS:
            msg = L.phmm_last_error(h).decode() if h.value else "phmm_create failed"
            L.phmm_destroy(h)
            self._h = None
            raise EngineUnavailableError("CUDA engine unavailable on device %d: %s" % (device, msg))
        self.device = device

    def _check(self, rc):
        if rc != SUCCESS:
            msg = self._L.phmm_last_error(self._h).decode()
            if rc == -1:
                from .errors import DataError
                raise DataError(msg)
            raise EngineError("libphmm error %d: %s" % (rc, msg))

    def score(self, flat, configs, flags=0, out=None, status=None):
        """phmm_score; ``out`` (float64[N]) / ``status`` (uint8[N]) are caller-owned result
        buffers (reused across calls by a C-ABI caller), allocated when omitted."""
        cin, keep1 = make_input(flat)
        copt, keep2 = make_options(configs, flags)
        n = flat.num_pairs
        out = np.empty(n, np.float64) if out is None else out
        st = np.empty(n, np.uint8) if status is None else status
        if out.shape != (n,) or out.dtype != np.float64 or not out.flags.c_contiguous:
            raise ValueError("out must be a contiguous float64 array of %d pairs" % n)
        if st.shape != (n,) or st.dtype != np.uint8 or not st.flags.c_contiguous:
            raise ValueError("status must be a contiguous uint8 array of %d pairs" % n)
        stats = PhmmStats()
        with self._lock:
            self._check(self._L.phmm_score(self._h, ctypes.byref(cin), ctypes.byref(copt), _ptr(out),
                                           _ptr(st), ctypes.byref(stats)))
        return out, st, stats

    def prepare(self, flat, configs, flags=0) -> int:
        cin, keep1 = make_input(flat)
        copt, keep2 = make_options(configs, flags)
        n = _i64()
        with self._lock:
            self._check(self._L.phmm_prepare(self._h, ctypes.byref(cin), ctypes.byref(copt), ctypes.byref(n)))
            self._n = n.value
        return n.value

    def execute(self):
        with self._lock:
            self._check(self._L.phmm_execute(self._h))

    def last_timing(self):
        """(device_ms, fast_ms, launches) of the last execute (CUDA events, engine stream)."""
        d, f, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
        with self._lock:
            self._L.phmm_last_timing(self._h, ctypes.byref(d), ctypes.byref(f), ctypes.byref(n))
        return d.value, f.value, n.value

    def last_phases(self):
        """[precompute, FP32 stream, post-pass (a), post-pass (b)+(c)] ms of the last execute."""
        out = np.zeros(4, np.float64)
        with self._lock:
            self._L.phmm_last_phases(self._h, _ptr(out))
        return out.tolist()

    def fetch(self):
        with self._lock:
            out = np.empty(self._n, np.float64)
            st = np.empty(self._n, np.uint8)
            stats = PhmmStats()
            self._check(self._L.phmm_fetch(self._h, _ptr(out), _ptr(st), ctypes.byref(stats)))
        return out, st, stats

    def set_device_budget(self, nbytes: int):
        """Bound the device working set of score() (0: none; see phmm_set_device_budget)."""
        with self._lock:
            self._check(self._L.phmm_set_device_budget(self._h, int(nbytes)))

    def set_pipeline(self, n: int):
        """phmm_score pipelining depth (0 automatic, 1 never, 2..8 equal chunks)."""
        with self._lock:
            self._check(self._L.phmm_set_pipeline(self._h, int(n)))

    def device_bytes(self) -> int:
        v = _i64()
        with self._lock:
            self._check(self._L.phmm_device_bytes(self._h, ctypes.byref(v)))
        return v.value

    def forward_matrices(self, read, hap, scale_log2: int = 0):
        """(M, I, D) float64 (m+1, n+1) of one ReadRecord / Haplotype pair (k_matrices)."""
        m, n = int(read.length), int(hap.length)
        arrs = [np.ascontiguousarray(a) for a in (read.bases, read.base_qual, read.ins_qual, read.del_qual,
                                                   read.gcp_qual, hap.bases)]
        out = [np.empty((m + 1, n + 1), np.float64) for _ in range(3)]
        with self._lock:
            self._check(self._L.phmm_forward_matrices(self._h, *[_ptr(a) for a in arrs[:5]], m, _ptr(arrs[5]), n,
                                                      int(scale_log2), *[_ptr(o) for o in out]))
        return out

    def close(self):
        lock = getattr(self, "_lock", None)
        if lock is None:
            return
        with lock:
            if self._h is not None:
                self._L.phmm_destroy(self._h)
                self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_contexts = {}
_contexts_lock = threading.Lock()


def context(device: int = 0) -> Context:
    """Process-wide cached context per device (created once under a module lock; its calls
    are serialized by the context's own lock)."""
    with _contexts_lock:
        ctx = _contexts.get(device)
        if ctx is None:
            ctx = Context(device)
            _contexts[device] = ctx
        return ctx


def pin_host(arr: np.ndarray) -> bool:
    """Page-lock a host array for DMA uploads (phmm_pin_host); False when unavailable."""
    try:
        return load().phmm_pin_host(arr.ctypes.data, arr.nbytes) == SUCCESS
    except (OSError, EngineUnavailableError):
        return False


def unpin_host(arr: np.ndarray) -> None:
    try:
        load().phmm_unpin_host(arr.ctypes.data)
    except (OSError, EngineUnavailableError):
        pass
