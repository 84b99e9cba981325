// flatten.cpp — CPython extension _phmm_flatten: Batch objects -> flat C-ABI arrays.
//
// The drop-in API takes the reference's list[Batch] (model.py:55-136: ReadRecord with
// int8 bases + four uint8 Phred tracks, Haplotype bases).  FlatBatches.from_batches must
// copy every read's five arrays and every haplotype into contiguous buffers; done per
// read in Python (attribute lookups + np.concatenate of 16k-1M small arrays) that cost
// ~100 ms per 65k pairs, on the run() path.  This walks the list once in C through the
// buffer protocol and memcpy's each array into its slot (two passes: sizes, then copy).
//
//   flatten(batches) -> (read_bases, base_qual, ins_qual, del_qual, gcp_qual, read_len,
//                        hap_bases, hap_len, batch_reads, batch_haps)
// as bytearrays (int8/uint8 data, int64 lengths/counts) that numpy wraps without a copy.
// The arrays are located with the numpy C API (PyArray_DATA), other buffers through the
// buffer protocol.
// Tracks must be C-contiguous 1-byte arrays of the read's length (ReadRecord guarantees
// it; anything else raises ValueError and the caller falls back to numpy).
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#define NPY_NO_DEPRECATED_API NPY_2_0_API_VERSION
#include <numpy/arrayobject.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <chrono>
#include <deque>
#include <thread>
#include <vector>

namespace {

// Source spans of the arrays to copy.  numpy arrays are read through the numpy C API
// (data pointer + size: no buffer export, which costs ~0.7 us per array); other objects
// through the buffer protocol, whose views are held until the copy is done.
struct Spans {
  std::vector<const char*> p;
  std::vector<Py_ssize_t> n;
  std::deque<Py_buffer> views;        // buffer-protocol exports only (stable addresses)
  explicit Spans(size_t cap) {
    p.reserve(cap);
    n.reserve(cap);
  }
  ~Spans() {
    for (Py_buffer& v : views) PyBuffer_Release(&v);
  }
  bool get(PyObject* obj, PyObject* name, const char* attr) {
    PyObject* a = PyObject_GetAttr(obj, name);
    if (!a) return false;
    const bool ok = take(a, attr);
    Py_DECREF(a);          // the owning record keeps the array alive
    return ok;
  }
  // a: borrowed reference to the attribute value
  bool take(PyObject* a, const char* attr) {
    if (PyArray_Check(a)) {
      PyArrayObject* arr = reinterpret_cast<PyArrayObject*>(a);
      const bool ok = PyArray_NDIM(arr) == 1 && PyArray_ITEMSIZE(arr) == 1 && PyArray_IS_C_CONTIGUOUS(arr);
      if (ok) {
        p.push_back(static_cast<const char*>(PyArray_DATA(arr)));
        n.push_back(PyArray_DIM(arr, 0));
      }
      if (!ok) PyErr_Format(PyExc_ValueError, "%s must be a contiguous 1-D array of 1-byte elements", attr);
      return ok;
    }
    views.emplace_back();
    Py_buffer& b = views.back();
    if (PyObject_GetBuffer(a, &b, PyBUF_C_CONTIGUOUS | PyBUF_FORMAT) != 0) {
      views.pop_back();
      return false;
    }
    if (b.itemsize != 1 || b.ndim != 1) {
      PyErr_Format(PyExc_ValueError, "%s must be a 1-D array of 1-byte elements", attr);
      return false;
    }
    p.push_back(static_cast<const char*>(b.buf));
    n.push_back(b.len);
    return true;
  }
};

// Instances of a class with __slots__ (the package's frozen slotted dataclasses) keep each
// field at a fixed offset: resolve the member descriptors once per type and read the
// fields directly (no dict, no attribute-lookup machinery).  ok = false: not slotted.
struct SlotOffsets {
  PyTypeObject* tp = nullptr;
  bool ok = false;
  Py_ssize_t off[5] = {0, 0, 0, 0, 0};
  void resolve(PyTypeObject* t, PyObject* const* names, int n) {
    tp = t;
    ok = true;
    for (int x = 0; x < n && ok; ++x) {
      PyObject* d = _PyType_Lookup(t, names[x]);          // borrowed
      ok = d && Py_IS_TYPE(d, &PyMemberDescr_Type) &&
           reinterpret_cast<PyMemberDescrObject*>(d)->d_member->type == Py_T_OBJECT_EX;
      if (ok) off[x] = reinterpret_cast<PyMemberDescrObject*>(d)->d_member->offset;
    }
  }
  // borrowed field x of obj (nullptr: unset)
  PyObject* get(PyObject* obj, int x) const { return *reinterpret_cast<PyObject**>(reinterpret_cast<char*>(obj) + off[x]); }
};

PyObject* new_bytes(const void* src, Py_ssize_t n) {
  return PyByteArray_FromStringAndSize(static_cast<const char*>(src), n);
}

PyObject* flatten(PyObject*, PyObject* args) {
  PyObject* arg = nullptr;
  PyObject* alloc_fn = Py_None;   // optional alloc(RL, HL) -> 6 writable buffers (reused arena)
  if (!PyArg_ParseTuple(args, "O|O", &arg, &alloc_fn)) return nullptr;
  PyObject* seq = PySequence_Fast(arg, "batches must be a sequence");
  if (!seq) return nullptr;
  const Py_ssize_t B = PySequence_Fast_GET_SIZE(seq);
  static const char* kTracks[5] = {"bases", "base_qual", "ins_qual", "del_qual", "gcp_qual"};
  static PyObject* kNames[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  static PyObject *kReads = nullptr, *kHaps = nullptr;
  if (!kReads) {                      // interned attribute names (GetAttrString builds a str per call)
    for (int x = 0; x < 5; ++x) kNames[x] = PyUnicode_InternFromString(kTracks[x]);
    kReads = PyUnicode_InternFromString("reads");
    kHaps = PyUnicode_InternFromString("haps");
  }
  // PHMM_TRACE=1: stage times on stderr
  static const bool trace = getenv("PHMM_TRACE") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  auto ms = [&]() { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); };
  double t_pass1 = 0, t_pass2 = 0, t_alloc = 0;
  std::vector<int64_t> bre(B), bha(B), rlen, hlen;
  int64_t RL = 0, HL = 0;
  bool ok = true;
  std::vector<PyObject*> keep;   // the reads / haps sequences of each batch
  // pass 1: the batches' read / haplotype sequences and counts
  size_t nreads = 0, nhaps = 0;
  for (Py_ssize_t b = 0; ok && b < B; ++b) {
    PyObject* batch = PySequence_Fast_GET_ITEM(seq, b);
    PyObject* reads = PyObject_GetAttr(batch, kReads);
    PyObject* haps = reads ? PyObject_GetAttr(batch, kHaps) : nullptr;
    PyObject* rs = reads ? PySequence_Fast(reads, "reads must be a sequence") : nullptr;
    PyObject* hs = haps ? PySequence_Fast(haps, "haps must be a sequence") : nullptr;
    Py_XDECREF(reads);
    Py_XDECREF(haps);
    if (!rs || !hs) { Py_XDECREF(rs); Py_XDECREF(hs); ok = false; break; }
    keep.push_back(rs);
    keep.push_back(hs);
    bre[b] = PySequence_Fast_GET_SIZE(rs);
    bha[b] = PySequence_Fast_GET_SIZE(hs);
    nreads += (size_t)bre[b];
    nhaps += (size_t)bha[b];
  }
  // every read record in order: pass 2 prefetches the records and their track arrays a few
  // reads ahead (the objects are scattered over the heap; the walk is latency bound)
  std::vector<PyObject*> recs;
  recs.reserve(nreads);
  for (Py_ssize_t b = 0; ok && b < B; ++b) {
    PyObject** it = PySequence_Fast_ITEMS(keep[2 * b]);
    recs.insert(recs.end(), it, it + bre[b]);
  }
  t_pass1 = ms();
  // pass 2: buffer views and lengths
  Spans rv(ok ? 5 * nreads : 0), hv(ok ? nhaps : 0);
  SlotOffsets rslots, hslots;
  rlen.reserve(nreads);
  hlen.reserve(nhaps);
  // Fast path: every read a record of one slotted type whose five tracks are 1-D contiguous
  // 1-byte numpy arrays of equal length (the package's ReadRecord).  The views are plain
  // field reads, taken on several threads while this thread keeps the GIL (no Python code
  // runs meanwhile, so the objects cannot change); anything else -> the serial walk below,
  // which also produces the error messages.
  bool fast = false;
  if (ok && nreads >= 4096) {
    PyTypeObject* tp = Py_TYPE(recs[0]);
    rslots.resolve(tp, kNames, 5);
    if (rslots.ok) {
      rv.p.resize(5 * nreads);
      rv.n.resize(5 * nreads);
      rlen.resize(nreads);
      const int nt = (int)std::min<size_t>(8, nreads / 2048);
      std::atomic<bool> bad{false};
      std::vector<int64_t> part(nt, 0);
      auto work = [&](int i) {
        int64_t sum = 0;
        for (size_t r = nreads * i / nt; r < nreads * (i + 1) / nt; ++r) {
          PyObject* rd = recs[r];
          if (Py_TYPE(rd) != tp || bad.load(std::memory_order_relaxed)) { bad = true; return; }
          Py_ssize_t m = 0;
          for (int x = 0; x < 5; ++x) {
            PyObject* a = rslots.get(rd, x);
            if (!a || Py_TYPE(a) != &PyArray_Type) { bad = true; return; }
            PyArrayObject* arr = reinterpret_cast<PyArrayObject*>(a);
            const Py_ssize_t n = PyArray_NDIM(arr) == 1 ? PyArray_DIM(arr, 0) : -1;
            if (n < 0 || PyArray_ITEMSIZE(arr) != 1 || !PyArray_IS_C_CONTIGUOUS(arr) || (x > 0 && n != m)) {
              bad = true;
              return;
            }
            m = n;
            rv.p[5 * r + x] = static_cast<const char*>(PyArray_DATA(arr));
            rv.n[5 * r + x] = n;
          }
          rlen[r] = m;
          sum += m;
        }
        part[i] = sum;
      };
      std::vector<std::thread> th;
      for (int i = 1; i < nt; ++i) th.emplace_back(work, i);
      work(0);
      for (auto& t : th) t.join();
      if (!bad) {
        fast = true;
        for (int64_t v : part) RL += v;
      } else {
        rv.p.clear();
        rv.n.clear();
        rlen.clear();
      }
    }
  }
  size_t gi = 0;                      // global read index
  constexpr size_t kAhead = 8;
  for (Py_ssize_t b = 0; ok && b < B; ++b) {
    PyObject* hs = keep[2 * b + 1];
    for (Py_ssize_t r = 0; ok && !fast && r < bre[b]; ++r, ++gi) {
      PyObject* rd = recs[gi];
      if (gi + 2 * kAhead < recs.size()) __builtin_prefetch(recs[gi + 2 * kAhead]);
      if (gi + kAhead < recs.size() && rslots.ok && Py_TYPE(recs[gi + kAhead]) == rslots.tp)
        for (int x = 0; x < 5; ++x) __builtin_prefetch(rslots.get(recs[gi + kAhead], x));
      const size_t first = rv.n.size();
      if (Py_TYPE(rd) != rslots.tp) rslots.resolve(Py_TYPE(rd), kNames, 5);
      if (rslots.ok) {                // slotted record: fields at fixed offsets
        for (int x = 0; ok && x < 5; ++x) {
          PyObject* a = rslots.get(rd, x);
          ok = a ? rv.take(a, kTracks[x]) : rv.get(rd, kNames[x], kTracks[x]);
        }
      } else {
        // instance __dict__ lookups (a frozen dataclass stores its fields there) instead of
        // five generic attribute lookups; anything else -> getattr
        PyObject* dict = PyObject_GenericGetDict(rd, nullptr);
        if (!dict) PyErr_Clear();
        for (int x = 0; ok && x < 5; ++x) {
          PyObject* a = dict ? PyDict_GetItemWithError(dict, kNames[x]) : nullptr;
          ok = a ? rv.take(a, kTracks[x]) : (!PyErr_Occurred() && rv.get(rd, kNames[x], kTracks[x]));
        }
        Py_XDECREF(dict);
      }
      if (!ok) break;
      const Py_ssize_t m = rv.n[first];
      for (int x = 1; ok && x < 5; ++x)
        if (rv.n[first + x] != m) {
          PyErr_Format(PyExc_ValueError, "%s track has length %zd, expected %zd", kTracks[x],
                       rv.n[first + x], m);
          ok = false;
        }
      rlen.push_back(m);
      RL += m;
    }
    for (Py_ssize_t h = 0; ok && h < bha[b]; ++h) {
      PyObject* hp = PySequence_Fast_GET_ITEM(hs, h);
      if (Py_TYPE(hp) != hslots.tp) hslots.resolve(Py_TYPE(hp), kNames, 1);
      PyObject* a = hslots.ok ? hslots.get(hp, 0) : nullptr;
      ok = a ? hv.take(a, kTracks[0]) : hv.get(hp, kNames[0], kTracks[0]);
      if (ok) {
        hlen.push_back(hv.n.back());
        HL += hlen.back();
      }
    }
  }
  t_pass2 = ms();
  PyObject* out = nullptr;
  if (ok) {
    PyObject* tr[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    PyObject* hb = nullptr;
    char* d[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    char* dh = nullptr;
    Py_buffer ab[6];
    int nab = 0;
    bool alloc = true;
    if (alloc_fn != Py_None) {        // caller's arena: already-faulted pages, no fresh allocation
      PyObject* got = PyObject_CallFunction(alloc_fn, "nn", (Py_ssize_t)RL, (Py_ssize_t)HL);
      PyObject* fast = got ? PySequence_Fast(got, "alloc must return a sequence") : nullptr;
      Py_XDECREF(got);
      alloc = fast && PySequence_Fast_GET_SIZE(fast) == 6;
      for (int x = 0; alloc && x < 6; ++x) {
        PyObject* o = PySequence_Fast_GET_ITEM(fast, x);
        alloc = PyObject_GetBuffer(o, &ab[x], PyBUF_WRITABLE | PyBUF_C_CONTIGUOUS) == 0;
        if (alloc) {
          ++nab;
          alloc = ab[x].len >= (x < 5 ? RL : HL);
          if (!alloc) PyErr_SetString(PyExc_ValueError, "alloc returned a buffer too small");
          Py_INCREF(o);
          if (x < 5) { tr[x] = o; d[x] = static_cast<char*>(ab[x].buf); }
          else { hb = o; dh = static_cast<char*>(ab[x].buf); }
        }
      }
      Py_XDECREF(fast);
    } else {
      for (int x = 0; x < 5; ++x) tr[x] = PyByteArray_FromStringAndSize(nullptr, RL);
      hb = PyByteArray_FromStringAndSize(nullptr, HL);
      alloc = hb != nullptr;
      for (int x = 0; x < 5; ++x) alloc = alloc && tr[x] != nullptr;
      if (alloc) {
        for (int x = 0; x < 5; ++x) d[x] = PyByteArray_AS_STRING(tr[x]);
        dh = PyByteArray_AS_STRING(hb);
      }
    }
    t_alloc = ms();
    if (alloc) {
      const size_t R = rlen.size();
      const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(8, (5 * RL + HL) >> 21));   // >= 2 MB per thread
      Py_BEGIN_ALLOW_THREADS
      // the copy (and the page faults of the fresh buffers) on a few threads, over read /
      // haplotype ranges; each range's destination offset is a prefix of the lengths
      std::vector<int64_t> roffs(R + 1, 0), hoffs(hlen.size() + 1, 0);
      for (size_t r = 0; r < R; ++r) roffs[r + 1] = roffs[r] + rlen[r];
      for (size_t h = 0; h < hlen.size(); ++h) hoffs[h + 1] = hoffs[h] + hlen[h];
      auto work = [&](int i) {
        for (size_t r = R * i / nt; r < R * (i + 1) / nt; ++r)
          for (int x = 0; x < 5; ++x) memcpy(d[x] + roffs[r], rv.p[5 * r + x], (size_t)rlen[r]);
        const size_t H = hlen.size();
        for (size_t h = H * i / nt; h < H * (i + 1) / nt; ++h) memcpy(dh + hoffs[h], hv.p[h], (size_t)hlen[h]);
      };
      std::vector<std::thread> th;
      for (int i = 1; i < nt; ++i) th.emplace_back(work, i);
      work(0);
      for (auto& t : th) t.join();
      Py_END_ALLOW_THREADS
      if (trace)
        fprintf(stderr, "[flatten] reads %zu haps %zu: batches %.3f views %.3f alloc %.3f copy %.3f ms (%d threads)\n",
                R, hlen.size(), t_pass1, t_pass2 - t_pass1, t_alloc - t_pass2, ms() - t_alloc, nt);
      out = Py_BuildValue("(NNNNNNNNNN)", tr[0], tr[1], tr[2], tr[3], tr[4],
                          new_bytes(rlen.data(), (Py_ssize_t)(rlen.size() * 8)), hb,
                          new_bytes(hlen.data(), (Py_ssize_t)(hlen.size() * 8)),
                          new_bytes(bre.data(), (Py_ssize_t)(bre.size() * 8)),
                          new_bytes(bha.data(), (Py_ssize_t)(bha.size() * 8)));
    } else {
      for (int x = 0; x < 5; ++x) Py_XDECREF(tr[x]);
      Py_XDECREF(hb);
      if (!PyErr_Occurred()) PyErr_NoMemory();
    }
    for (int x = 0; x < nab; ++x) PyBuffer_Release(&ab[x]);
  }
  for (PyObject* o : keep) Py_DECREF(o);
  Py_DECREF(seq);
  return out;
}

PyMethodDef kMethods[] = {
    {"flatten", flatten, METH_VARARGS,
     "flatten(batches, alloc=None) -> 10 buffers (see flatten.cpp); alloc(RL, HL) may supply the 6 data buffers"},
    {nullptr, nullptr, 0, nullptr}};

PyModuleDef kModule = {PyModuleDef_HEAD_INIT, "_phmm_flatten", "Batch list -> flat arrays", -1, kMethods};

}  // namespace

PyMODINIT_FUNC PyInit__phmm_flatten(void) {
  import_array();
  return PyModule_Create(&kModule);
}
