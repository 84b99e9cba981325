// datagen.cpp — host-only synthetic input generator (libphmm_host.so).
//
// Re-implements, draw for draw, the numpy Generator stream that the reference's
// synthetic generator consumes (pkg/src/pairhmm/datagen.py:78-121, restated in
// paper_2411_11547_b200/datagen.py::_stream), so a c5-sized workload (10M pairs, 1.25M
// reads) is produced in about a second instead of minutes of per-read Python:
//   * PCG64 (XSL-RR 128/64; state / increment taken from numpy's SeedSequence seeding);
//   * next_uint32 with numpy's one-word carry (has_uint32 / uinteger) across calls;
//   * Generator.random():        (next_uint64 >> 11) * 2^-53;
//   * Generator.integers(lo, hi[, size]) for int64 results: Lemire's bounded multiply on
//     32-bit words with rejection (ranges < 2^32), no draw for an empty range;
//   * Generator.integers(0, 4, size, dtype=int8): the byte-buffered Lemire variant (a fresh
//     4-byte buffer per call).
// Inputs are validated by the Python caller; tests/test_datagen.py checks the arrays
// against the Python restatement element for element.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

namespace {

struct Pcg64 {
  unsigned __int128 state, inc;
  bool has32 = false;
  uint32_t u32 = 0;

  uint64_t next64() {
    static const unsigned __int128 kMul =
        ((unsigned __int128)2549297995355413924ULL << 64) | (unsigned __int128)4865540595714422341ULL;
    state = state * kMul + inc;
    const uint64_t x = (uint64_t)(state >> 64) ^ (uint64_t)state;
    const unsigned rot = (unsigned)(state >> 122);
    return (x >> rot) | (x << ((64 - rot) & 63));
  }
  uint32_t next32() {
    if (has32) {
      has32 = false;
      return u32;
    }
    const uint64_t v = next64();
    has32 = true;
    u32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }
  double uniform() { return (double)(next64() >> 11) * (1.0 / 9007199254740992.0); }
  // integers(lo, hi_inclusive) for int64 results with hi - lo < 2^32 - 1
  int64_t bounded(int64_t lo, int64_t hi) {
    const uint32_t rng = (uint32_t)(hi - lo);
    if (rng == 0) return lo;
    const uint32_t excl = rng + 1;
    uint64_t m = (uint64_t)next32() * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
      const uint32_t thr = (UINT32_MAX - rng) % excl;
      while (left < thr) {
        m = (uint64_t)next32() * excl;
        left = (uint32_t)m;
      }
    }
    return lo + (int64_t)(m >> 32);
  }
  // integers(0, 4, size=n, dtype=int8)
  void bases(int8_t* out, int64_t n) {
    uint32_t buf = 0;
    int bcnt = 0;
    for (int64_t i = 0; i < n; ++i) {
      if (!bcnt) {
        buf = next32();
        bcnt = 3;
      } else {
        buf >>= 8;
        --bcnt;
      }
      // rng_excl = 4 divides 256: Lemire's threshold is 0, no rejection
      out[i] = (int8_t)(((uint16_t)(uint8_t)buf * 4) >> 8);
    }
  }
};

struct Spec {                  // a length or quality spec: fixed value or inclusive range
  int64_t lo, hi;
  bool fixed;
};

struct Gen {
  std::vector<int8_t> rb, hb;
  std::vector<uint8_t> q[4];
  std::vector<int64_t> rlen, hlen;
};

int64_t draw_len(Pcg64& g, const Spec& s) { return s.fixed ? s.lo : g.bounded(s.lo, s.hi); }

void draw_quals(Pcg64& g, const Spec& s, int64_t m, std::vector<uint8_t>& out) {
  const size_t o = out.size();
  out.resize(o + m);
  for (int64_t i = 0; i < m; ++i) out[o + i] = (uint8_t)(s.fixed ? s.lo : g.bounded(s.lo, s.hi));
}

// _mutate: hits = random(n) < rate; count draws integers(1, 4, size=count); (b + k) % 4
void mutate(Pcg64& g, int8_t* b, int64_t n, double rate, std::vector<uint8_t>& hit) {
  hit.resize(n);
  int64_t count = 0;
  for (int64_t i = 0; i < n; ++i) {
    hit[i] = g.uniform() < rate;
    count += hit[i];
  }
  if (!count) return;
  for (int64_t i = 0; i < n; ++i)
    if (hit[i]) b[i] = (int8_t)((b[i] + g.bounded(1, 3)) % 4);
}

}  // namespace

extern "C" {

// Runs the generator; returns an opaque handle (nullptr on bad arguments).
//   mode 0 = independent, 1 = derived; len/qual specs: (lo, hi, fixed) triples
void* phmm_gen_run(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int has32,
                   uint32_t u32, int64_t num_batches, int64_t reads_per_batch, int64_t haps_per_batch,
                   const int64_t* read_len, const int64_t* hap_len, int mode, double rate,
                   const int64_t* base_q, const int64_t* indel_q, const int64_t* gcp_q) {
  if (num_batches < 0 || reads_per_batch < 1 || haps_per_batch < 1) return nullptr;
  Pcg64 g;
  g.state = ((unsigned __int128)state_hi << 64) | state_lo;
  g.inc = ((unsigned __int128)inc_hi << 64) | inc_lo;
  g.has32 = has32 != 0;
  g.u32 = u32;
  const Spec RL{read_len[0], read_len[1], read_len[2] != 0}, HLs{hap_len[0], hap_len[1], hap_len[2] != 0};
  const Spec BQ{base_q[0], base_q[1], base_q[2] != 0}, IQ{indel_q[0], indel_q[1], indel_q[2] != 0};
  const Spec GQ{gcp_q[0], gcp_q[1], gcp_q[2] != 0};
  Gen* out = new Gen();
  std::vector<int64_t> lengths(haps_per_batch);
  std::vector<int8_t> locus;
  std::vector<uint8_t> hit;
  for (int64_t b = 0; b < num_batches; ++b) {
    int64_t nmax = 0, nmin = INT64_MAX;
    for (int64_t h = 0; h < haps_per_batch; ++h) {
      lengths[h] = draw_len(g, HLs);
      nmax = std::max(nmax, lengths[h]);
      nmin = std::min(nmin, lengths[h]);
    }
    if (mode == 0) {
      for (int64_t h = 0; h < haps_per_batch; ++h) {
        const size_t o = out->hb.size();
        out->hb.resize(o + lengths[h]);
        g.bases(out->hb.data() + o, lengths[h]);
        out->hlen.push_back(lengths[h]);
      }
    } else {
      locus.resize(nmax);
      g.bases(locus.data(), nmax);
      for (int64_t h = 0; h < haps_per_batch; ++h) {
        const size_t o = out->hb.size();
        out->hb.insert(out->hb.end(), locus.begin(), locus.begin() + lengths[h]);
        mutate(g, out->hb.data() + o, lengths[h], rate, hit);
        out->hlen.push_back(lengths[h]);
      }
    }
    for (int64_t r = 0; r < reads_per_batch; ++r) {
      const int64_t m = draw_len(g, RL);
      const size_t o = out->rb.size();
      out->rb.resize(o + m);
      int8_t* dst = out->rb.data() + o;
      if (mode == 0) {
        g.bases(dst, m);
      } else {                                   // _read_from(rng, common = locus[:nmin], m)
        if (m <= nmin) {
          const int64_t start = g.bounded(0, nmin - m);
          memcpy(dst, locus.data() + start, m);
        } else {
          memcpy(dst, locus.data(), nmin);
          g.bases(dst + nmin, m - nmin);
        }
        mutate(g, dst, m, rate, hit);
      }
      draw_quals(g, BQ, m, out->q[0]);
      draw_quals(g, IQ, m, out->q[1]);
      draw_quals(g, IQ, m, out->q[2]);
      draw_quals(g, GQ, m, out->q[3]);
      out->rlen.push_back(m);
    }
  }
  return out;
}

void phmm_gen_sizes(const void* h, int64_t* read_bases, int64_t* hap_bases, int64_t* reads, int64_t* haps) {
  const Gen* G = static_cast<const Gen*>(h);
  *read_bases = (int64_t)G->rb.size();
  *hap_bases = (int64_t)G->hb.size();
  *reads = (int64_t)G->rlen.size();
  *haps = (int64_t)G->hlen.size();
}

// copies out: read bases, 4 quality tracks, read lengths, hap bases, hap lengths
void phmm_gen_copy(const void* h, int8_t* rb, uint8_t* bq, uint8_t* iq, uint8_t* dq, uint8_t* gq, int64_t* rlen,
                   int8_t* hb, int64_t* hlen) {
  const Gen* G = static_cast<const Gen*>(h);
  memcpy(rb, G->rb.data(), G->rb.size());
  memcpy(bq, G->q[0].data(), G->q[0].size());
  memcpy(iq, G->q[1].data(), G->q[1].size());
  memcpy(dq, G->q[2].data(), G->q[2].size());
  memcpy(gq, G->q[3].data(), G->q[3].size());
  memcpy(rlen, G->rlen.data(), G->rlen.size() * sizeof(int64_t));
  memcpy(hb, G->hb.data(), G->hb.size());
  memcpy(hlen, G->hlen.data(), G->hlen.size() * sizeof(int64_t));
}

void phmm_gen_free(void* h) { delete static_cast<Gen*>(h); }

}  // extern "C"
