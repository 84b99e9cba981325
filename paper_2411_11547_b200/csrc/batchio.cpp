// batchio.cpp — host-only batch text format reader / writers (libphmm_host.so).
//
// The reference's line-oriented format (pkg/src/pairhmm/batchio.py:1-14):
//     BATCH <num_reads> <num_haps>
//     READ <bases> <baseQ> <insQ> <delQ> <gcpQ>      x num_reads (Phred+33)
//     HAP <bases>                                     x num_haps
// '#' comment lines and blank lines are skipped.  The reader parses straight into the
// flat arrays of the C-ABI (include/phmm.h phmm_input) -- one pass over the bytes, no
// per-read objects -- replacing parse_batch_file (batchio.py:50-108) on the engine path.
//
// Error policy: this reader is the FAST path only.  On any deviation from the canonical
// format (a syntax error, an illegal base or quality character, or bytes it does not
// interpret exactly like Python text mode: non-ASCII, a lone '\r', NUL) it returns
// PHMM_IO_SLOW and the Python restatement of the reference parser (batchio.py here)
// re-reads the file and raises the reference's ParseError with its message and line.
//
// Writers: the batch file (write_batch_file, batchio.py:111-123) and the score lines
// (format_score_lines / write_scores, batchio.py:126-159: "%d %d %d %.6f" per item or
// "%d %d %d ERROR:<kind>", then "# cells=%d seconds=%.6f gcups=%.6f").  glibc printf
// "%.6f" is correctly rounded, like CPython's float formatting.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace {

constexpr int kOk = 0, kSlow = 1, kIoError = 2;

struct Parsed {
  std::vector<int8_t> rb, hb;
  std::vector<uint8_t> q[4];
  std::vector<int64_t> read_off{0}, hap_off{0}, bro{0}, bho{0};
};

inline bool ws(unsigned char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

int8_t kBaseCode[256];
struct InitLut {
  InitLut() {
    memset(kBaseCode, -1, sizeof(kBaseCode));
    kBaseCode[(unsigned char)'A'] = 0; kBaseCode[(unsigned char)'C'] = 1; kBaseCode[(unsigned char)'G'] = 2;
    kBaseCode[(unsigned char)'T'] = 3; kBaseCode[(unsigned char)'N'] = 4;
  }
} init_lut;

struct Field { const char* p; int64_t n; };

// ASCII-whitespace split of one line (the line has no '\n'); at most `cap` fields kept,
// the true count returned
int split(const char* p, const char* e, Field* out, int cap) {
  int n = 0;
  while (p < e) {
    while (p < e && ws((unsigned char)*p)) ++p;
    if (p >= e) break;
    const char* s = p;
    while (p < e && !ws((unsigned char)*p)) ++p;
    if (n < cap) out[n] = Field{s, p - s};
    ++n;
  }
  return n;
}

bool eq(const Field& f, const char* lit) {
  const int64_t n = (int64_t)strlen(lit);
  return f.n == n && memcmp(f.p, lit, n) == 0;
}

// plain decimal digits only (anything CPython's int() accepts beyond that -> slow path)
bool to_int(const Field& f, int64_t* v) {
  if (f.n < 1 || f.n > 15) return false;
  int64_t x = 0;
  for (int64_t i = 0; i < f.n; ++i) {
    const char c = f.p[i];
    if (c < '0' || c > '9') return false;
    x = x * 10 + (c - '0');
  }
  *v = x;
  return true;
}

bool bases(const Field& f, std::vector<int8_t>& out) {
  const size_t o = out.size();
  out.resize(o + f.n);
  int8_t* d = out.data() + o;
  for (int64_t i = 0; i < f.n; ++i) {
    const int8_t c = kBaseCode[(unsigned char)f.p[i]];
    if (c < 0) return false;
    d[i] = c;
  }
  return true;
}

bool quals(const Field& f, std::vector<uint8_t>& out) {
  const size_t o = out.size();
  out.resize(o + f.n);
  uint8_t* d = out.data() + o;
  for (int64_t i = 0; i < f.n; ++i) {
    const int q = (unsigned char)f.p[i] - 33;
    if (q < 0 || q > 93) return false;
    d[i] = (uint8_t)q;
  }
  return true;
}

int parse_buffer(const char* buf, int64_t len, Parsed& P) {
  // bytes Python text mode would read differently: non-ASCII (UTF-8 decoding, Unicode
  // whitespace), control bytes other than \t \n \v \f \r (NUL; 0x1c-0x1f are str.split()
  // whitespace), and '\r' not followed by '\n' (universal newlines: a line break)
  for (int64_t i = 0; i < len; ++i) {
    const unsigned char c = (unsigned char)buf[i];
    if (c >= 0x80 || (c < 0x20 && !(c >= '\t' && c <= '\r')) || c == 0x7f ||
        (c == '\r' && (i + 1 >= len || buf[i + 1] != '\n')))
      return kSlow;
  }
  enum { kHeader, kRead, kHap } state = kHeader;
  int64_t need = 0, haps_left = 0;
  const char* p = buf;
  const char* end = buf + len;
  Field f[7];
  while (p < end) {
    const char* nl = (const char*)memchr(p, '\n', end - p);
    const char* le = nl ? nl : end;
    const char* s = p;
    p = nl ? nl + 1 : end;
    while (s < le && ws((unsigned char)*s)) ++s;
    if (s == le || *s == '#') continue;                     // blank / comment line
    const int nf = split(s, le, f, 7);
    if (state == kHeader) {
      int64_t r, h;
      if (nf != 3 || !eq(f[0], "BATCH") || !to_int(f[1], &r) || !to_int(f[2], &h) || r < 1 || h < 1)
        return kSlow;
      need = r;
      haps_left = h;
      state = kRead;
      P.bro.push_back(P.bro.back() + r);
      P.bho.push_back(P.bho.back() + h);
    } else if (state == kRead) {
      if (nf != 6 || !eq(f[0], "READ")) return kSlow;
      const int64_t m = f[1].n;
      for (int x = 2; x < 6; ++x)
        if (f[x].n != m) return kSlow;
      if (!bases(f[1], P.rb)) return kSlow;
      for (int x = 0; x < 4; ++x)
        if (!quals(f[2 + x], P.q[x])) return kSlow;
      P.read_off.push_back(P.read_off.back() + m);
      if (--need == 0) state = kHap;
    } else {
      if (nf != 2 || !eq(f[0], "HAP")) return kSlow;
      if (!bases(f[1], P.hb)) return kSlow;
      P.hap_off.push_back(P.hap_off.back() + f[1].n);
      if (--haps_left == 0) state = kHeader;
    }
  }
  return state == kHeader ? kOk : kSlow;                     // truncated batch: slow path
}

const char kAlphabet[5] = {'A', 'C', 'G', 'T', 'N'};

struct Out {
  FILE* f;
  std::vector<char> buf;
  size_t n = 0;
  explicit Out(FILE* fp) : f(fp), buf(1 << 20) {}
  bool flush() {
    if (n && fwrite(buf.data(), 1, n, f) != n) return false;
    n = 0;
    return true;
  }
  bool reserve(size_t k) {
    if (n + k > buf.size()) {
      if (!flush()) return false;
      if (k > buf.size()) buf.resize(k);
    }
    return true;
  }
  char* at() { return buf.data() + n; }
};

}  // namespace

extern "C" {

#define PHMM_IO_OK 0
#define PHMM_IO_SLOW 1
#define PHMM_IO_ERROR 2

// Parse a batch file.  Returns a handle (sizes / copy / free below) or null with *rc =
// PHMM_IO_SLOW (use the Python parser for the reference's error) or PHMM_IO_ERROR (I/O).
void* phmm_io_parse(const char* path, int* rc) {
  *rc = kIoError;
  FILE* fp = fopen(path, "rb");
  if (!fp) return nullptr;
  std::vector<char> data;
  if (fseek(fp, 0, SEEK_END) == 0) {
    const long sz = ftell(fp);
    if (sz > 0) {
      data.resize((size_t)sz);
      fseek(fp, 0, SEEK_SET);
      if (fread(data.data(), 1, (size_t)sz, fp) != (size_t)sz) { fclose(fp); return nullptr; }
    }
  }
  fclose(fp);
  // a UTF-8 byte-order mark is text Python keeps (it is not whitespace): slow path
  Parsed* P = new Parsed();
  const int r = parse_buffer(data.data(), (int64_t)data.size(), *P);
  if (r != kOk) {
    delete P;
    *rc = r;
    return nullptr;
  }
  *rc = kOk;
  return P;
}

void phmm_io_sizes(const void* h, int64_t* read_bases, int64_t* hap_bases, int64_t* reads, int64_t* haps,
                   int64_t* batches) {
  const Parsed* P = static_cast<const Parsed*>(h);
  *read_bases = (int64_t)P->rb.size();
  *hap_bases = (int64_t)P->hb.size();
  *reads = (int64_t)P->read_off.size() - 1;
  *haps = (int64_t)P->hap_off.size() - 1;
  *batches = (int64_t)P->bro.size() - 1;
}

void phmm_io_copy(const void* h, int8_t* rb, uint8_t* bq, uint8_t* iq, uint8_t* dq, uint8_t* gq, int64_t* read_off,
                  int8_t* hb, int64_t* hap_off, int64_t* bro, int64_t* bho) {
  const Parsed* P = static_cast<const Parsed*>(h);
  auto cp = [](void* d, const auto& v) {
    if (!v.empty()) memcpy(d, v.data(), v.size() * sizeof(v[0]));
  };
  cp(rb, P->rb); cp(bq, P->q[0]); cp(iq, P->q[1]); cp(dq, P->q[2]); cp(gq, P->q[3]);
  cp(read_off, P->read_off); cp(hb, P->hb); cp(hap_off, P->hap_off); cp(bro, P->bro); cp(bho, P->bho);
}

void phmm_io_free(void* h) { delete static_cast<Parsed*>(h); }

// write_batch_file (batchio.py:111-123) from flat arrays; 0 ok, PHMM_IO_ERROR on I/O failure
int phmm_io_write_batches(const char* path, const int8_t* rb, const uint8_t* bq, const uint8_t* iq,
                          const uint8_t* dq, const uint8_t* gq, const int64_t* read_off, const int8_t* hb,
                          const int64_t* hap_off, const int64_t* bro, const int64_t* bho, int64_t B) {
  FILE* fp = fopen(path, "wb");
  if (!fp) return kIoError;
  Out o(fp);
  bool ok = true;
  for (int64_t b = 0; ok && b < B; ++b) {
    ok = o.reserve(64);
    if (!ok) break;
    o.n += snprintf(o.at(), 64, "BATCH %lld %lld\n", (long long)(bro[b + 1] - bro[b]), (long long)(bho[b + 1] - bho[b]));
    for (int64_t r = bro[b]; ok && r < bro[b + 1]; ++r) {
      const int64_t s = read_off[r], m = read_off[r + 1] - s;
      ok = o.reserve(5 * m + 16);
      if (!ok) break;
      char* d = o.at();
      memcpy(d, "READ ", 5); d += 5;
      for (int64_t i = 0; i < m; ++i) *d++ = kAlphabet[(unsigned)rb[s + i] < 5 ? rb[s + i] : 4];
      for (const uint8_t* q : {bq, iq, dq, gq}) {
        *d++ = ' ';
        for (int64_t i = 0; i < m; ++i) *d++ = (char)(q[s + i] + 33);
      }
      *d++ = '\n';
      o.n = d - o.buf.data();
    }
    for (int64_t hh = bho[b]; ok && hh < bho[b + 1]; ++hh) {
      const int64_t s = hap_off[hh], n = hap_off[hh + 1] - s;
      ok = o.reserve(n + 8);
      if (!ok) break;
      char* d = o.at();
      memcpy(d, "HAP ", 4); d += 4;
      for (int64_t i = 0; i < n; ++i) *d++ = kAlphabet[(unsigned)hb[s + i] < 5 ? hb[s + i] : 4];
      *d++ = '\n';
      o.n = d - o.buf.data();
    }
  }
  ok = ok && o.flush();
  ok = (fclose(fp) == 0) && ok;
  return ok ? kOk : kIoError;
}

// write_scores (batchio.py:126-159): per item "<b> <r> <h> %.6f", or "<b> <r> <h> ERROR:<kind>"
// for items with kind[gid] >= 0 (kind_names[kind]) or a NaN score ("unscored"); then the
// report comment when footer != null.
int phmm_io_write_scores(const char* path, const int64_t* bro, const int64_t* bho, int64_t B, const double* scores,
                         const int8_t* kind, const char* const* kind_names, const char* footer) {
  FILE* fp = fopen(path, "wb");
  if (!fp) return kIoError;
  Out o(fp);
  bool ok = true;
  int64_t gid = 0;
  for (int64_t b = 0; ok && b < B; ++b) {
    const int64_t R = bro[b + 1] - bro[b], H = bho[b + 1] - bho[b];
    for (int64_t r = 0; ok && r < R; ++r)
      for (int64_t h = 0; h < H; ++h, ++gid) {
        if (!(ok = o.reserve(128))) break;
        const double v = scores[gid];
        const int k = kind[gid];
        int w;
        if (k >= 0 || v != v)
          w = snprintf(o.at(), 128, "%lld %lld %lld ERROR:%s\n", (long long)b, (long long)r, (long long)h,
                       k >= 0 ? kind_names[k] : "unscored");
        else
          w = snprintf(o.at(), 128, "%lld %lld %lld %.6f\n", (long long)b, (long long)r, (long long)h, v);
        o.n += (size_t)w;
      }
  }
  if (ok && footer) {
    const size_t n = strlen(footer);
    ok = o.reserve(n);
    if (ok) { memcpy(o.at(), footer, n); o.n += n; }
  }
  ok = ok && o.flush();
  ok = (fclose(fp) == 0) && ok;
  return ok ? kOk : kIoError;
}

}  // extern "C"
