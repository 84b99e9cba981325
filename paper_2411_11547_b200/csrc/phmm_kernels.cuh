// phmm_kernels.cuh — sm_100a kernels of the B200 Pair-HMM forward engine.
//
// Kernel family:
//   k_precompute      per read: degenerate-transition flag (prob.py:71-75) and the
//                     guard-band sensitivity sum Gsum used to decide when the fast
//                     FP32 result provably equals the reference's flushed FP32 result.
//   k_stream<MODE,P,K> read-stationary haplotype streaming wavefront (the hot kernel): one
//                     sub-warp of P threads owns one read and streams two LANES of the
//                     batch's haplotypes through an anti-diagonal wavefront (float2 lanes,
//                     FFMA2 with a scalar-broadcast coefficient); each thread owns K read
//                     positions; neighbour M/I/D cross threads by __shfl_up_sync
//                     (PAPER.md:186-218); emissions come from a per-read shared-memory
//                     table E[c][i].  Modes: fast FP32 / fast FP64
//                     (retries) / bit-exact FP32 / bit-exact FP64.  Reads longer than the
//                     tiling stripe over it with a boundary column.
//   k_exact_all / k_fast64_all  per-pair post-pass lists (bit-exact FP32/FP64 recursion:
//                     no FMA, per-store flush, j-ordered accumulation; FP64 retry).
//
// Read layout inside a kernel: Q stripes of W = P*K padded positions;
//   [L left-padding positions][m real read positions][1 accumulator position],
//   L = Q*W - m - 1.  Left padding carries the row-0 boundary D(0,j) = S/n down to the
//   first real position; the accumulator position turns the D recurrence into the
//   running sum  sum_j (M(m,j) + I(m,j))  (wavefront.py:156-160) so the result always
//   sits in fixed registers of the last thread.
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace phmm {

constexpr int kStatusOk = 0, kStatusOverflow = 1, kStatusTooSmall = 2, kStatusDegenerate = 3;
constexpr int kStatusExactF32 = 0x20, kStatusRetriedF64 = 0x40;
constexpr int kNumExactP = 4;            // exact kernels for P in {4, 8, 16, 32}
constexpr int kExactK = 8;

struct ExactItem {                        // one read x one haplotype
  int pair, read, hap, scale;
};

struct StreamUnit {                       // 32 B
  int read;
  int list;                               // StreamHap entries: lane A [list, list+cntA),
  int cntA, cntB;                         //                    lane B [list+cntA, +cntB)
  int rowsA, rowsB;                       // the lane's rows: haplotype lengths (+ separator rows, fast modes)
  int ro, m;                              // read offset / length (saves a dependent load)
};
struct StreamHap { int hap, pair, off, n; };   // haplotype, pair id, base offset, length

// Stream units appended on the device, one list per tiling (null units[0]: disabled)
struct RetryLists {
  StreamUnit* units[8];
  int* count;                             // [8] units per tiling
  StreamHap* haps;
  int* hap_count;
  int* overflow;
  int unit_cap[8];                        // per tiling: pairs that can land there
  int hap_cap;
  int enabled;
  int lane_haps;                          // haplotypes per lane of a built unit
};

struct EngineDev {
  const int8_t* rbases;
  const uint8_t *bq, *iq, *dq, *gq;
  const int64_t* roff;
  const int8_t* hbases;
  const int64_t* hoff;
  const int* read_m;
  const int* read_scale;
  const int* read_ncap;
  float* read_gsum;
  uint8_t* read_flags;                    // bit0: degenerate
  const double* lut;                      // PHRED_TO_PROB[94]
  double* acc;                            // per pair raw accumulator (scaled)
  uint8_t* status;                        // per pair status
  ExactItem* ex32[kNumExactP];            // exact-f32 work lists (host + device appended)
  int* ex32_count;                        // [kNumExactP]
  ExactItem* ex64[kNumExactP];            // f64 work lists
  int* ex64_count;                        // [kNumExactP]
  int list_cap[kNumExactP];              // per slot: pairs whose read maps to the slot
  int retry_f64;
  ExactItem* fx64[kNumExactP];            // FP64 retry lists (fast FP64 kernel)
  int* fx64_count;                        // [kNumExactP]
  int* band_inline;                       // guard-band pairs taken inline so far
  int band_budget;
  const int* invalid;                     // device input validation verdict: nonzero = skip
  RetryLists r64;                         // FP64 retry units (built by the FP32 stream kernel)
  RetryLists rx32;                        // bit-exact FP32 guard-band units (same)
  RetryLists r64b;                        // long reads: FP64 retries of guard-band pairs whose
                                          // exact rerun underflowed (built by the exact stream
                                          // kernel, run after the post-pass)
};

__device__ __forceinline__ int exact_slot_for(int m) {
  // smallest W = P*8 >= m + 1 among P in {4,8,16,32}; longer reads stripe at P = 32
  return (m + 1 <= 32) ? 0 : (m + 1 <= 64) ? 1 : (m + 1 <= 128) ? 2 : 3;
}

__device__ __forceinline__ void append_item(ExactItem* const* lists, int* counts, const int* caps,
                                            int slot, ExactItem it) {
  int pos = atomicAdd(&counts[slot], 1);
  if (pos < caps[slot]) lists[slot][pos] = it;
}

// Fast-path classification of a finished FP32 accumulator:
//   a < 2^-93                    -> every final-row term flushes in the reference: flagged
//   guard band                   -> rerun on the bit-exact kernel.  The reference's flushes
//                                   lower the accumulator by at most 2^-90 * n * Gsum, i.e.
//                                   |d log10| <= 2^-90 n Gsum / (a ln 10); that is <= 1e-5 |s|
//                                   (a tenth of the 1e-4 relative bar on the score s) iff
//                                   a |s| >= 2^-90 * 1e5 / ln 10 * n * Gsum = 2^-74.6 n Gsum
//   score > -1.5 (short pairs)   -> bit-exact kernel (relative tolerance near log10 = 0)
//   otherwise                    -> accept
__device__ __forceinline__ bool guard_band(float a, int n, float gsum, int scale) {
  const float hi = ldexpf(0.031622776f, scale);                   // 10^-1.5 * 2^scale
  const float s = fabsf(__log2f(a) - (float)scale) * 0.30103f;     // |log10 score| (a normal)
  return a * s < 0x1.6a09e6p-75f * (float)n * gsum || a > hi;     // 2^-74.5 (conservative)
}
// ---------------------------------------------------------------------------------
// k_exact<T, P, K>: bit-exact reference recursion (reference.py:106-122,
// wavefront.py:130-160) — no FMA, per-store flush, j-ordered accumulation.
// ---------------------------------------------------------------------------------

template <typename T> struct ExactTraits;
template <> struct ExactTraits<float> {
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float flush_thr() { return 0x1p-90f; }
};
template <> struct ExactTraits<double> {
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double flush_thr() { return 0x1p-970; }
};

__device__ inline bool retry64_unit(const EngineDev& E, int pair, int read, int hap, int m);

// One item (read x haplotype) on one sub-warp of P threads; `live` false = the
// sub-warp only takes part in the warp-wide shuffles.  Writes acc/status itself.
template <typename T, int P, int K>
__device__ __forceinline__ void exact_item(const EngineDev& E, const ExactItem& it, bool has,
                                           const double* s_lut, T* Et, T* colX, T* colY, int col_rows,
                                           int t) {
  using X = ExactTraits<T>;
  constexpr int W = P * K;
  constexpr bool kIsF32 = sizeof(T) == 4;
  const T thr = X::flush_thr();
  const T zero = (T)0;
  const int r = it.read, m = E.read_m[r];
  const int64_t ro = E.roff[r];
  const int n = (int)(E.hoff[it.hap + 1] - E.hoff[it.hap]);
  const bool degen = (E.read_flags[r] & 1) != 0;
  const bool live = has && !degen;
  int steps = live ? n + P - 1 : 0;
  steps = __reduce_max_sync(0xffffffffu, steps);
  if (has && degen && t == 0) { E.acc[it.pair] = 0.0; E.status[it.pair] = kStatusDegenerate; }
  const int Q = (m + 1 + W - 1) / W;
  const int Lp = Q * W - m - 1;
  const T bnd = (T)(ldexp(1.0, it.scale) / (double)n);     // wavefront.py:405-406
  const int8_t* h = E.hbases + E.hoff[it.hap];
  T res = zero;
  T* colPrev = colX;
  T* colNext = colY;

  // Q is per item; the warp iterates to the max over its sub-warps
  const int Qw = __reduce_max_sync(0xffffffffu, live ? Q : 0);
  for (int q = 0; q < Qw; ++q) {
    const bool sact = live && q < Q;
    T al[K], be[K], dl[K], ep[K], zt[K], M[K], I[K], D[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int p = q * W + t * K + k;
      T lam[5];
      M[k] = zero; I[k] = zero;
      if (p < Lp) {
        al[k] = zero; be[k] = zero; dl[k] = zero; ep[k] = (T)1; zt[k] = zero; D[k] = bnd;
#pragma unroll
        for (int c = 0; c < 5; ++c) lam[c] = zero;
      } else if (p < Lp + m) {
        const int i0 = p - Lp;
        const double d = s_lut[E.iq[ro + i0]], z = s_lut[E.dq[ro + i0]];
        const double e = s_lut[E.gq[ro + i0]], qe = s_lut[E.bq[ro + i0]];
        al[k] = (T)((1.0 - d) - z);
        be[k] = (T)(1.0 - e);
        dl[k] = (T)d;
        ep[k] = (T)e;
        zt[k] = (i0 + 1 < m) ? (T)z : zero;        // D(m, .) never reaches the score
        D[k] = zero;
        const int rc = E.rbases[ro + i0];
        const T lm = (T)(1.0 - qe), lx = (T)(qe / 3.0);
#pragma unroll
        for (int c = 0; c < 5; ++c) lam[c] = (rc == c || rc == 4 || c == 4) ? lm : lx;
      } else {
        al[k] = (T)1; be[k] = (T)1; dl[k] = zero; ep[k] = (T)1; zt[k] = (T)1; D[k] = zero;
#pragma unroll
        for (int c = 0; c < 5; ++c) lam[c] = (T)1;
      }
#pragma unroll
      for (int c = 0; c < 5; ++c) Et[(c * K + k) * P + t] = lam[c];
    }
    if (sact && t == P - 1 && q < Q - 1) {
      colNext[0] = M[K - 1]; colNext[col_rows] = I[K - 1]; colNext[2 * col_rows] = D[K - 1];
    }
    T nbM = zero, nbI = zero, nbD = zero;
    if (t == 0) {
      if (q == 0) { nbD = bnd; }
      else if (sact) { nbM = colPrev[0]; nbI = colPrev[col_rows]; nbD = colPrev[2 * col_rows]; }
    }
    __syncwarp();
    // one-row-ahead prefetch of thread 0's boundary column and of every thread's
    // haplotype character: global loads stay off the per-step dependency chain
    T pfM = zero, pfI = zero, pfD = zero;
    if (t == 0 && q > 0 && sact) {
      const int jj = min(1, n);
      pfM = colPrev[jj]; pfI = colPrev[col_rows + jj]; pfD = colPrev[2 * col_rows + jj];
    }
    int cpf = (sact && 1 - t >= 1 && 1 - t <= n) ? h[-t] : 0;
    for (int s = 1; s <= steps; ++s) {
      const int j = s - t;
      const T dgM = nbM, dgI = nbI, dgD = nbD;
      nbM = __shfl_up_sync(0xffffffffu, M[K - 1], 1, P);
      nbI = __shfl_up_sync(0xffffffffu, I[K - 1], 1, P);
      nbD = __shfl_up_sync(0xffffffffu, D[K - 1], 1, P);
      if (t == 0) {
        if (q == 0) { nbM = zero; nbI = zero; nbD = bnd; }
        else if (sact) {
          nbM = pfM; nbI = pfI; nbD = pfD;
          const int jj = min(s + 1, n);
          pfM = colPrev[jj]; pfI = colPrev[col_rows + jj]; pfD = colPrev[2 * col_rows + jj];
        }
      }
      const int c = cpf;
      cpf = (sact && j + 1 >= 1 && j + 1 <= n) ? h[j] : 0;
      if (sact && j >= 1 && j <= n) {
        const T* Ec = Et + (c * K) * P + t;
#pragma unroll
        for (int k = K - 1; k >= 0; --k) {
          // dv = zt*M(i,j-1) + ep*D(i,j-1)
          const T dv = X::add(X::mul(zt[k], M[k]), X::mul(ep[k], D[k]));
          D[k] = dv >= thr ? dv : zero;
          const T pm = (k > 0) ? M[k - 1] : dgM;
          const T pi = (k > 0) ? I[k - 1] : dgI;
          const T pd = (k > 0) ? D[k - 1] : dgD;
          // mv = lam*(al*M(i-1,j-1) + be*(I(i-1,j-1) + D(i-1,j-1)))
          const T mv = X::mul(Ec[k * P], X::add(X::mul(al[k], pm), X::mul(be[k], X::add(pi, pd))));
          M[k] = mv >= thr ? mv : zero;
        }
        T lM = nbM, lI = nbI;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          // iv = dl*M(i-1,j) + ep*I(i-1,j)
          const T iv = X::add(X::mul(dl[k], lM), X::mul(ep[k], lI));
          I[k] = iv >= thr ? iv : zero;
          lM = M[k];
          lI = I[k];
        }
        if (t == P - 1) {
          if (q == Q - 1) {
            if (j == n) res = X::add(X::add(D[K - 1], M[K - 1]), X::add(M[K - 2], I[K - 2]));
          } else {
            colNext[j] = M[K - 1]; colNext[col_rows + j] = I[K - 1]; colNext[2 * col_rows + j] = D[K - 1];
          }
        }
      }
    }
    __syncwarp();
    T* tmp = colPrev; colPrev = colNext; colNext = tmp;
  }
  if (live && t == P - 1) {
    const bool bad = !(res > zero) || !isfinite((double)res);
    if (kIsF32) {
      if (bad && E.retry_f64) {
        E.status[it.pair] = kStatusRetriedF64;
        if (!retry64_unit(E, it.pair, r, it.hap, m))
          append_item(E.fx64, E.fx64_count, E.list_cap, exact_slot_for(m), ExactItem{it.pair, r, it.hap, 0});
      } else {
        E.acc[it.pair] = (double)res;
        E.status[it.pair] = bad ? kStatusOverflow : kStatusExactF32;
      }
    } else {
      E.acc[it.pair] = (double)res;
      const uint8_t keep = E.status[it.pair] & kStatusRetriedF64;
      E.status[it.pair] = (uint8_t)((bad ? kStatusOverflow : kStatusOk) | keep);
    }
  }
}

// ---------------------------------------------------------------------------------
// k_stream<P, K>: read-stationary haplotype streaming (single-stripe reads).
//
// A StreamUnit is one read and two LANES of haplotypes (float2 .x = lane A, .y = lane B);
// each lane is the concatenation of several of the batch's haplotypes, scored one after
// the other without leaving the wavefront: the read's coefficients and emission table
// are set up once per unit, and the wavefront's fill/drain (P-1 steps) is paid once per
// unit instead of once per pair.  Haplotype boundaries travel down the sub-warp with the
// per-row code (the same shuffle that carries the haplotype characters):
//   FIRST(lane): the thread's row is row 1 of a new haplotype: its lane state is reset to
//                row 0 of that pair (M = I = 0, D' = S'/n in the left padding, else 0) and
//                the diagonal input becomes the matrix boundary;
//   LAST(lane):  the row is the pair's last: thread P-1 reads the accumulator position and
//                classifies the result (fast_finish).
// Rows outside a thread's stream (fill, drain, the shorter lane's tail) compute values
// that are never read: every pair starts with a FIRST reset.
// ---------------------------------------------------------------------------------

constexpr int kCodeFirst = 8, kCodeLast = 16;          // code byte: base | FIRST | LAST
// Row code of the rows before a thread's first row (the wavefront fill): emission 0 at
// every position, so a fill step maps the row-0 state onto itself (M stays 0, I stays 0,
// D keeps the boundary in the left padding and 0 elsewhere) -- every lane starts from its
// pre-initialised row 0 with no per-thread FIRST event.
constexpr int kCodeIdle = 5;
constexpr unsigned kIdle2 = kCodeIdle | (kCodeIdle << 8);
// window list entries: start row | kWinShort (a one-step window: the LAST event of a lane's
// final haplotype) -- otherwise P steps (the FIRST events of a haplotype boundary)
constexpr int kWinShort = 1 << 30;
// The fast modes (kFast32 = 0, kFast64 = 1) separate consecutive haplotypes of a lane by one
// kCodeIdle row: it leaves M = I = 0, so a FIRST event only resets D (a third of the event
// work inside the checked steps); the exact modes reset M, I and D and need no separators.
template <int MODE> struct SepRows { static constexpr bool value = MODE == 0 || MODE == 1; };
constexpr int kStreamCodeBytesPerCta = 32768;          // row-code staging, shared memory
constexpr int kStreamMaxLaneHaps = 15;                 // haplotypes per lane of one unit
constexpr int kStreamMaxWin = 2 * (kStreamMaxLaneHaps + 1);
template <int P> struct StreamCap {                    // max rows per lane of one unit
  static constexpr int bytes = kStreamCodeBytesPerCta / (4 * (32 / P));
  static constexpr int value = bytes / 2 - 2;
};
__host__ __device__ __forceinline__ int stream_cap_of(int P) {
  return kStreamCodeBytesPerCta / (4 * (32 / P)) / 2 - 2;
}

// Kernel modes of the streaming family:
//   kFast32   folded recurrence, FMA, packed float2 (FFMA2/FMUL2/FADD2), guard band
//   kFast64   folded recurrence, DFMA, two lanes (FP32-underflow retries, GATK behaviour)
//   kExact32  the reference's expressions, no FMA, per-store flush 2^-90 (packed FMUL2/FADD2
//             round each lane like scalar FMUL/FADD): guard-band pairs, exact mode
//   kExact64  the same in FP64 with flush 2^-970: f64 configs (bit-identical)
enum { kFast32 = 0, kFast64 = 1, kExact32 = 2, kExact64 = 3 };
template <int MODE> struct ModeOf {
  static constexpr bool F64 = MODE == kFast64 || MODE == kExact64;
  static constexpr bool EXACT = MODE == kExact32 || MODE == kExact64;
};
template <int MODE, int K> struct StreamOcc {
  static constexpr int value = ModeOf<MODE>::F64 ? (K <= 6 ? 3 : 2) : (K <= 8 ? 4 : (K <= (MODE == 0 ? 11 : 12) ? 3 : 2));
};

// Device-built stream units (one list per tiling): FP64 retries of FP32-underflowed pairs
// and bit-exact reruns of guard-band pairs, grouped per read by the FP32 stream kernel.
constexpr int kNumR64Geoms = 7;     // FP64 retry:  (8,4) (16,4) (16,6) (16,8) (32,6) (32,7) (32,8)
constexpr int kNumRX32Geoms = 8;    // exact FP32:  (8,4) (16,4) (16,6) (32,4) (32,6) (32,8) (32,12) (32,16)
// haplotypes per lane of a device-built unit: short units keep these small post-pass
// lists parallel (their count is unknown when the grid is sized)
constexpr int kRetryLaneHaps64 = 2, kRetryLaneHapsX32 = 1;   // defaults (RetryLists.lane_haps)
constexpr int kInlineBand = 4;      // guard-band pairs a warp may rerun inline per unit
// reads longer than the widest tiling stripe over it (k_stream handles Q > 1 stripes)
__host__ __device__ __forceinline__ int r64_geom_for(int m) {
  const int w = m + 1;
  return w <= 32 ? 0 : w <= 64 ? 1 : w <= 96 ? 2 : w <= 128 ? 3 : w <= 192 ? 4 : w <= 224 ? 5 : 6;
}
__host__ __device__ __forceinline__ int r64_geom_P(int g) { return g == 0 ? 8 : (g <= 3 ? 16 : 32); }

// A guard-band pair whose exact FP32 rerun ran per pair (inline or from the per-pair list)
// and underflowed: a one-haplotype second-stage FP64 stream unit, so every FP64 retry of a
// call runs on the FP64 stream kernel whichever path reran the pair (the per-pair FP64
// kernel rounds differently in the last ulp).  false: no second-stage list for this read.
__device__ inline bool retry64_unit(const EngineDev& E, int pair, int read, int hap, int m) {
  const RetryLists& L = E.r64b;
  const int g = r64_geom_for(m);
  if (!L.enabled || !L.units[g]) return false;
  const int n = (int)(E.hoff[hap + 1] - E.hoff[hap]);
  const int ui = atomicAdd(&L.count[g], 1);
  const int hi = atomicAdd(L.hap_count, 1);
  if (ui < L.unit_cap[g] && hi < L.hap_cap) {
    L.haps[hi] = StreamHap{hap, pair, (int)E.hoff[hap], n};
    L.units[g][ui] = StreamUnit{read, hi, 1, 0, n, 0, (int)E.roff[read], m};
  } else {
    atomicAdd(L.overflow, 1);                 // capacity is sized for every pair: never
  }
  return true;
}
__host__ __device__ __forceinline__ int rx32_geom_for(int m) {
  const int w = m + 1;
  return w <= 32 ? 0 : w <= 64 ? 1 : w <= 96 ? 2 : w <= 128 ? 3 : w <= 192 ? 4 : w <= 256 ? 5
       : w <= 384 ? 6 : 7;
}
__host__ __device__ __forceinline__ int rx32_geom_P(int g) { return g == 0 ? 8 : (g <= 2 ? 16 : 32); }

struct Dbl2 { double x, y; };

// Two-lane value algebra of the streaming kernel: FP32 = packed float2 (FFMA2/FMUL2/FADD2
// with a scalar-broadcast coefficient), FP64 = two independent DFMA chains.
template <bool F64> struct Lanes;
template <> struct Lanes<false> {
  using S = float;
  using V = float2;
  using EV = float4;                      // emission chunk: 4 positions (LDS.128)
  static constexpr int EW = 4;
  static __device__ __forceinline__ V zero() { return make_float2(0.f, 0.f); }
  static __device__ __forceinline__ V fma(S s, V a, V b) { return __ffma2_rn(make_float2(s, s), a, b); }
  static __device__ __forceinline__ V mul(S s, V a) { return __fmul2_rn(make_float2(s, s), a); }
  static __device__ __forceinline__ V add(V a, V b) { return __fadd2_rn(a, b); }
  static __device__ __forceinline__ S mul1(S a, S b) { return __fmul_rn(a, b); }
  // exact-mode ops: ptxas fuses packed multiplies into a following packed add (FFMA2) even
  // from explicit mul.rn.f32x2, so products are scalar __fmul_rn (never fused) and only
  // the adds are packed -- each lane rounds like the reference's separate mul and add
  static __device__ __forceinline__ V xmul(S s, V a) { return make_float2(__fmul_rn(s, a.x), __fmul_rn(s, a.y)); }
  static __device__ __forceinline__ V xadd(V a, V b) { return __fadd2_rn(a, b); }
  static __device__ __forceinline__ S comp(const EV& v, int i) {
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
  }
  static __device__ __forceinline__ EV pack(const S* l) { return make_float4(l[0], l[1], l[2], l[3]); }
  static __device__ __forceinline__ S thr() { return 0x1p-90f; }
};
template <> struct Lanes<true> {
  using S = double;
  using V = Dbl2;
  using EV = double2;                     // emission chunk: 2 positions (LDS.128)
  static constexpr int EW = 2;
  static __device__ __forceinline__ V zero() { return Dbl2{0.0, 0.0}; }
  static __device__ __forceinline__ V fma(S s, V a, V b) { return Dbl2{::fma(s, a.x, b.x), ::fma(s, a.y, b.y)}; }
  static __device__ __forceinline__ V mul(S s, V a) { return Dbl2{__dmul_rn(s, a.x), __dmul_rn(s, a.y)}; }
  static __device__ __forceinline__ V add(V a, V b) { return Dbl2{__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y)}; }
  static __device__ __forceinline__ S mul1(S a, S b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ V xmul(S s, V a) { return mul(s, a); }    // __dmul_rn: unfused
  static __device__ __forceinline__ V xadd(V a, V b) { return add(a, b); }
  static __device__ __forceinline__ S comp(const EV& v, int i) { return i == 0 ? v.x : v.y; }
  static __device__ __forceinline__ EV pack(const S* l) { return make_double2(l[0], l[1]); }
  static __device__ __forceinline__ S thr() { return 0x1p-970; }
};
template <int L, class V> __device__ __forceinline__ auto& lane_ref(V& v) { return L == 0 ? v.x : v.y; }
// emission-table chunks: float4 (4 positions, LDS.128) in FP32, double2 in FP64; the last
// chunk is padded when K is not a multiple of the width (K = 14: 4 LDS.128 per lane-step
// instead of 7 LDS.64, c5 FP32 phase -0.7 %)
__device__ __forceinline__ float ev_comp(const float4& v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }
__device__ __forceinline__ double ev_comp(const double2& v, int i) { return i == 0 ? v.x : v.y; }
__device__ __forceinline__ void ev_pack(float4& e, const float* l) { e = make_float4(l[0], l[1], l[2], l[3]); }
__device__ __forceinline__ void ev_pack(double2& e, const double* l) { e = make_double2(l[0], l[1]); }
template <bool F64, int K> struct EChunk {
  using type = typename std::conditional<F64, double2, float4>::type;
  static constexpr int width = F64 ? 2 : 4;
  static constexpr int chunks = (K + width - 1) / width;
};
// FP32 pairs: the flush as a packed multiply by {v >= thr} in {1, 0} (FSET + FSET + FMUL2
// instead of two compare-and-selects); exact because the values are finite and
// non-negative, and harmless when ptxas fuses the product into a later packed add
// (1*v + x and 0*v + x round like v + x and x)
__device__ __forceinline__ float2 flush2(float2 v, float thr) {
  float mx, my;
  asm("set.ge.f32.f32 %0, %1, %2;" : "=f"(mx) : "f"(v.x), "f"(thr));
  asm("set.ge.f32.f32 %0, %1, %2;" : "=f"(my) : "f"(v.y), "f"(thr));
  return __fmul2_rn(v, make_float2(mx, my));
}
template <class V, class S> __device__ __forceinline__ V flush2(V v, S thr) {
  v.x = v.x >= thr ? v.x : (S)0;            // reference store flush (wavefront.py:134-136)
  v.y = v.y >= thr ? v.y : (S)0;
  return v;
}

// Classification of a finished FP32 stream accumulator; returns 0 = written, 1 = guard
// band (caller queues the bit-exact rerun), 2 = FP32 underflow to retry in FP64 (caller).
__device__ __forceinline__ int stream_finish32(const EngineDev& E, float a, int pair, int n, float gsum, int scale) {
  if (a != a) { E.status[pair] = kStatusExactF32; return 1; }   // beta_i = 0 (gcp q = 0): exact
  if (!(a >= 0x1p-93f)) {
    if (E.retry_f64) { E.status[pair] = kStatusRetriedF64; return 2; }
    E.acc[pair] = 0.0;
    E.status[pair] = kStatusOverflow;
    return 0;
  }
  if (guard_band(a, n, gsum, scale)) { E.status[pair] = kStatusExactF32; return 1; }
  E.acc[pair] = (double)a;
  E.status[pair] = kStatusOk;
  return 0;
}

// Groups the flagged entries (bit e of mask[lane]) of a finished unit into new stream
// units of tiling g (row capacity cap) appended to L; thread-serial, rare.
__device__ __forceinline__ void emit_retry_units(const StreamUnit& U, const StreamHap* shaps, const unsigned* mask,
                                                 const RetryLists& L, int g, int cap, int m, int lane_haps,
                                                 int cap_w, bool sep) {
  int lanes_n[2] = {0, 0}, rows_n[2] = {0, 0};
  StreamHap buf[2][kStreamMaxLaneHaps];
  auto emit = [&]() {
    const int tot = lanes_n[0] + lanes_n[1];
    if (tot == 0) return;
    const int ui = atomicAdd(&L.count[g], 1);
    const int hi = atomicAdd(L.hap_count, tot);
    if (ui < L.unit_cap[g] && hi + tot <= L.hap_cap) {
      for (int x = 0; x < lanes_n[0]; ++x) L.haps[hi + x] = buf[0][x];
      for (int x = 0; x < lanes_n[1]; ++x) L.haps[hi + lanes_n[0] + x] = buf[1][x];
      L.units[g][ui] = StreamUnit{U.read, hi, lanes_n[0], lanes_n[1], rows_n[0], rows_n[1], U.ro, m};
    } else {
      atomicAdd(L.overflow, 1);                 // capacity is sized for every pair: never
    }
    lanes_n[0] = lanes_n[1] = 0;
    rows_n[0] = rows_n[1] = 0;
  };
  if (U.m + 1 > cap_w) lane_haps = 1;       // striped (long) reads: latency-bound, keep units short
  for (int ln = 0; ln < 2; ++ln) {
    unsigned msk = mask[ln];
    const int e0 = U.list + (ln ? U.cntA : 0);
    while (msk) {
      const int e = __ffs(msk) - 1;
      msk &= msk - 1;
      const StreamHap sh = shaps[e0 + e];
      int l2 = rows_n[0] <= rows_n[1] ? 0 : 1;
      const int gap = sep && rows_n[l2] > 0 ? 1 : 0;     // separator row before it (SepRows)
      if (rows_n[l2] + gap + sh.n > cap || lanes_n[l2] >= lane_haps) { emit(); l2 = 0; }
      rows_n[l2] += sh.n + (sep && lanes_n[l2] > 0 ? 1 : 0);
      buf[l2][lanes_n[l2]++] = sh;
    }
  }
  emit();
}

// cp.async (global -> shared, no registers): the striped kernels' boundary-column ring
template <int B> __device__ __forceinline__ void cp_async(unsigned dst, const void* src) {
  if constexpr (B == 16) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
  else asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(dst), "l"(src), "n"(B) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
constexpr int kColRing = 64;      // rows of a striped sub-warp's boundary-column ring (x3 states)

template <int MODE, int P, int K, bool STRIPES = false>
__global__ void __launch_bounds__(128, (STRIPES ? 2 : StreamOcc<MODE, K>::value))   // striped: <= 2
k_stream(const EngineDev E, const StreamUnit* __restrict__ units, const StreamHap* __restrict__ shaps,
         int num_units_arg, const int* __restrict__ num_units_dev, int* __restrict__ counter,
         void* __restrict__ colbuf_v, int col_rows) {
  constexpr bool F64 = ModeOf<MODE>::F64, EXACT = ModeOf<MODE>::EXACT;
  constexpr bool SEP = SepRows<MODE>::value;
  using A = Lanes<F64>;
  using S = typename A::S;
  using V = typename A::V;
  using EV = typename EChunk<F64, K>::type;
  constexpr int EW = EChunk<F64, K>::width;
  constexpr int W = P * K, G = 32 / P, KE = EChunk<F64, K>::chunks;
  constexpr int CB = kStreamCodeBytesPerCta / (4 * G);
  static_assert(K >= 4, "tiling");
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* s_lut = reinterpret_cast<double*>(smem_raw);
  EV* s_E = reinterpret_cast<EV*>(smem_raw + 96 * sizeof(double));
  unsigned char* s_code = smem_raw + 96 * sizeof(double) + (size_t)4 * G * 5 * KE * P * sizeof(EV);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int sw = lane / P, t = lane % P;
  const int slot = wib * G + sw;
  const int num_units = num_units_dev ? min(*num_units_dev, num_units_arg) : num_units_arg;
  if (num_units == 0 || *E.invalid) return;
  __shared__ EV s_zero[KE * P];                   // emission row of kCodeIdle (all 0)
  for (int i = threadIdx.x; i < 94; i += blockDim.x) s_lut[i] = E.lut[i];
  for (int i = threadIdx.x; i < KE * P * (int)(sizeof(EV) / sizeof(float)); i += blockDim.x)
    reinterpret_cast<float*>(s_zero)[i] = 0.f;
  __syncthreads();
  EV* Et = s_E + (size_t)(slot * 5 * KE) * P;
  unsigned char* cd = s_code + (size_t)slot * CB;
  const unsigned short* cd16 = reinterpret_cast<const unsigned short*>(cd);
  const V zero2 = A::zero();
  const S thr = A::thr();
  __shared__ StreamUnit s_unit[4 * G];
  __shared__ int s_win[4 * G * kStreamMaxWin];
  __shared__ S s_bs[4 * G * 2 * kStreamMaxLaneHaps];
  __shared__ int s_meta[4 * G * 4];
  __shared__ int s_nwin[4 * G];
  __shared__ unsigned s_flag[4 * G * 2];          // kFast32: lane entries that underflowed
  __shared__ unsigned s_band[4 * G * 2];          // kFast32: lane entries in the guard band
  __shared__ ExactItem s_inl[MODE == kFast32 ? 4 * G * kInlineBand : 1];
  __shared__ int s_ninl[4 * G];
  // Striped tilings, few units (<= 2 per CTA, latency bound: c4 and the long-read retry
  // lists): "team" mode -- the CTA's 4 warps share one unit, warp w running stripes
  // w, w+4, ... concurrently; stripe q's column goes to stripe q+1 through one of 8
  // per-CTA columns with a row-progress flag, so a unit takes ~(rows + Q x 64) steps
  // instead of Q x rows.
  __shared__ int s_team_unit;
  __shared__ int s_prog[STRIPES ? 8 : 1];          // team mode: column progress flags (atomics)
  const bool team = STRIPES && num_units * 2 <= (int)gridDim.x * 4;

  for (;;) {
    int g = 0;
    if (STRIPES && team) {
      __syncthreads();                                  // every warp is done with the last unit
      if (threadIdx.x == 0) s_team_unit = atomicAdd(counter, 1);
      if (threadIdx.x < 8) s_prog[threadIdx.x] = 0;
      __syncthreads();
      g = s_team_unit;
    } else {
      if (lane == 0) g = atomicAdd(counter, 1);
      g = __shfl_sync(FULL, g, 0);
    }
    if (g * G >= num_units) break;
    const int u = g * G + sw;
    const bool has = u < num_units;
    const StreamUnit U = units[has ? u : g * G];
    const int r = U.read, m = U.m;
    const int64_t ro = U.ro;
    const bool degen = (E.read_flags[r] & 1) != 0;
    const bool live = has && !degen;
    const int rows = live ? max(U.rowsA, U.rowsB) : 0;
    const int steps = __reduce_max_sync(FULL, rows) + P - 1;
    if (has && degen && !(team && wib > 0)) {
      for (int e = t; e < U.cntA + U.cntB; e += P) {
        const int pr = shaps[U.list + e].pair;
        E.acc[pr] = 0.0; E.status[pr] = kStatusDegenerate;
      }
    }
    // reads longer than W - 1 run in Q stripes of W positions: the stream is replayed per
    // stripe; thread P-1 hands its last position's (M, I, D) per row to the next stripe
    // through a column in global memory (L2-resident), read one row ahead by thread 0
    const int Q = STRIPES ? (m + 1 + W - 1) / W : 1;    // single-stripe instantiations: Q = 1
    const int Qw = STRIPES ? (int)__reduce_max_sync(FULL, (unsigned)(live ? Q : 1)) : 1;
    const int Lp = Q * W - m - 1;
    V* colX = nullptr;
    V* colY = nullptr;
    if (STRIPES && Qw > 1) {                            // team mode: the CTA's 8 columns
      const size_t gslot = ((size_t)blockIdx.x * 4 + (team ? 0 : wib)) * G + sw;
      colX = reinterpret_cast<V*>(colbuf_v) + gslot * 6 * (size_t)col_rows;
      colY = colX + 3 * (size_t)col_rows;
    }
    if (t == 0) {
      s_unit[slot] = U;
      s_flag[2 * slot] = 0u; s_flag[2 * slot + 1] = 0u;
      s_band[2 * slot] = 0u; s_band[2 * slot + 1] = 0u;
      s_ninl[slot] = 0;
    }
    __syncwarp();          // a team warp without a stripe of this unit reads these right away
#pragma unroll 1
    for (int q = team ? wib : 0; q < Qw; q += team ? 4 : 1) {
    const bool sq = live && q < Q;                      // this sub-warp has stripe q
    const bool first_q = q == (team ? wib : 0);         // this warp's first stripe of the unit
    const bool lastq = q == Q - 1;
    const int rows_q = sq ? rows : 0;

    // ---- per-position coefficients + emission table.  Fast modes: scaled
    //   state Mt(i) = alpha_{i+1} M(i), I(i) = d_i I''(i), beta_{i+1} D(i) = c_i D''(i) with
    //   d_i = beta_{i+1} delta_i / alpha_i, c_i = beta_{i+1} zeta_i / alpha_{i+1} (position
    //   after the read: beta = alpha = 1), so that
    //     D'' = eps D''(up) + Mt(up),   I'' = r I''(left) + Mt(left),
    //     Mt = lam (Mt + d_{i-1} I'' + c_{i-1} D'')(diag),   r = beta_{i+1} eps_i d_{i-1} / (beta_i d_i)
    //   -- 6 operations per cell (4 packed FMAs + the per-lane emission product); registers
    //   ep = eps, be = r, dl = d_{p-1}, zt = c_{p-1}.  Exact modes: the reference's al, be,
    //   dl, ep, zt with the f64 -> dtype casts of wavefront.py:347-355.
    S al[K], be[K], dl[K], ep[K], zt[K];
    V M[K], I[K], D[K];
    // the fast FP32 mode derives its coefficients in FP32 (a few ulp against the 1e-4 bar;
    // the FP64 retry keeps FP64 coefficients for its 1e-9 bar)
    using CT = typename std::conditional<MODE == kFast32, float, double>::type;
    CT dprev = 1, cprev = 1;                          // fast modes: d, c of position p - 1
    CT ia = -1;                                       // 1 / alpha of the next position, once known
    if constexpr (!EXACT) {
      const int pp = q * W + t * K - 1;
      if (pp >= Lp && pp < Lp + m) {
        const int i0 = pp - Lp;
        const CT d = (CT)s_lut[E.iq[ro + i0]], z = (CT)s_lut[E.dq[ro + i0]];
        CT anext = 1, bnext = 0, bI = 1;
        if (i0 + 1 < m) {
          anext = ((CT)1 - (CT)s_lut[E.iq[ro + i0 + 1]]) - (CT)s_lut[E.dq[ro + i0 + 1]];
          bnext = bI = (CT)1 - (CT)s_lut[E.gq[ro + i0 + 1]];
        }
        ia = (CT)1 / anext;
        dprev = bI * d / (((CT)1 - d) - z);
        cprev = bnext * z * ia;
      }
    }
#pragma unroll
    for (int ke = 0; ke < KE; ++ke) {
      S lam[5][EW];
#pragma unroll
      for (int kk = 0; kk < EW; ++kk) {
        const int k = ke * EW + kk;
        const int p = q * W + t * K + k;
        if (k >= K) {                                   // padding of the last chunk (odd K)
#pragma unroll
          for (int c = 0; c < 5; ++c) lam[c][kk] = 0;
          continue;
        }
        M[k] = zero2; I[k] = zero2; D[k] = zero2;
        if (p < Lp) {                                   // left padding
          if constexpr (EXACT) { al[k] = 0; be[k] = 0; dl[k] = 0; ep[k] = 1; zt[k] = 0; }
          else { be[k] = 0; dl[k] = (S)dprev; zt[k] = (S)cprev; ep[k] = 1; dprev = 1.0; cprev = 1.0; }
#pragma unroll
          for (int c = 0; c < 5; ++c) lam[c][kk] = 0;
        } else if (p < Lp + m) {                        // real read position
          const int i0 = p - Lp;
          const double d = s_lut[E.iq[ro + i0]], z = s_lut[E.dq[ro + i0]];
          const double e = s_lut[E.gq[ro + i0]], qe = s_lut[E.bq[ro + i0]];
          const int rc = E.rbases[ro + i0];
          S lm, lx;
          if constexpr (EXACT) {                        // prob.py:66-112, cast per dtype
            al[k] = (S)((1.0 - d) - z); be[k] = (S)(1.0 - e); dl[k] = (S)d; ep[k] = (S)e;
            zt[k] = (i0 + 1 < m) ? (S)z : (S)0;         // D(m, .) never reaches the score
            lm = (S)(1.0 - qe); lx = (S)(qe / 3.0);
          } else {                                      // fast modes (CT arithmetic)
            const CT cd = (CT)d, cz = (CT)z, ce = (CT)e, cqe = (CT)qe;
            CT anext = 1, bnext = 0, bI = 1;            // alpha, beta of position i+1
            if (i0 + 1 < m) {
              anext = ((CT)1 - (CT)s_lut[E.iq[ro + i0 + 1]]) - (CT)s_lut[E.dq[ro + i0 + 1]];
              bnext = bI = (CT)1 - (CT)s_lut[E.gq[ro + i0 + 1]];
            }
            // two divisions per position: 1/alpha carries to the next position
            const CT inv_alpha = ia >= 0 ? ia : (CT)1 / (((CT)1 - cd) - cz);
            const CT inv_anext = (CT)1 / anext;
            const CT dcur = bI * cd * inv_alpha;
            const CT ccur = bnext * cz * inv_anext;     // 0 for the last position
            // beta_i = 0 (gcp q = 0): r = inf -> NaN accumulator -> exact rerun
            be[k] = (S)(bI * ce * dprev / (((CT)1 - ce) * dcur));
            dl[k] = (S)dprev; zt[k] = (S)cprev; ep[k] = (S)ce;
            dprev = dcur; cprev = ccur; ia = inv_anext;
            lm = (S)(anext * ((CT)1 - cqe)); lx = (S)(anext * (cqe / (CT)3));
          }
#pragma unroll
          for (int c = 0; c < 5; ++c) lam[c][kk] = (rc == c || rc == 4 || c == 4) ? lm : lx;
        } else {                                        // accumulator position
          if constexpr (EXACT) { al[k] = 1; be[k] = 1; dl[k] = 0; ep[k] = 1; zt[k] = 1; }
          else { be[k] = 0; dl[k] = (S)dprev; zt[k] = (S)cprev; ep[k] = 1; dprev = 1.0; cprev = 1.0; }
#pragma unroll
          for (int c = 0; c < 5; ++c) lam[c][kk] = 1;
        }
      }
#pragma unroll
      for (int c = 0; c < 5; ++c) ev_pack(Et[(c * KE + ke) * P + t], lam[c]);
    }

    // ---- row codes of both lanes into shared memory (one uint16 per row: lane A | lane B,
    // each byte base | FIRST | LAST; rows outside a lane's stream read the idle code N).
    // A unit whose lanes fit the slot (rows < RS) is staged once; a longer one (a haplotype
    // longer than the slot: no length limit) runs in RING mode -- row i lives in slot
    // i & (RS - 1) and the sub-warp restages the next half-ring of rows every RS/2 steps,
    // once every thread has passed the rows it replaces (stage_rows / the step loop).
    constexpr int RS = CB / 2;                          // code slots per sub-warp (power of 2)
    static_assert((RS & (RS - 1)) == 0 && RS / 2 > P + 1, "code ring");
    const bool cring = rows >= RS;
    const unsigned rmask = cring ? (unsigned)(RS - 1) : 0xffffffffu;
    auto stage_rows = [&](int r0, int r1) {             // rows [r0, r1), r0 >= 1, both lanes
#pragma unroll 1
      for (int ln = 0; ln < 2; ++ln) {
        const int cnt = ln ? U.cntB : U.cntA;
        const int e0 = U.list + (ln ? U.cntA : 0);
        int start = 1;                                  // first row of haplotype e
#pragma unroll 1
        for (int e = 0; e < cnt && start < r1; ++e) {
          const StreamHap sh = shaps[e0 + e];
          const int lo = max(r0, start), hi = min(r1, start + sh.n);
          const int8_t* src = E.hbases + sh.off - start;   // src[row] = base of that row
          // coalesced 128-bit loads: thread t takes the aligned 16-byte chunks t, t + P, ...
          // of the segment (the device copy of the haplotype bases is padded by 16 bytes)
          const uintptr_t a_lo = reinterpret_cast<uintptr_t>(src + lo), a_hi = reinterpret_cast<uintptr_t>(src + hi);
#pragma unroll 1
          for (uintptr_t a = (a_lo & ~(uintptr_t)15) + 16 * (uintptr_t)t; a < a_hi; a += 16 * (uintptr_t)P) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(a));
            const int x0 = (int)(reinterpret_cast<const int8_t*>(a) - src);
            const unsigned w[4] = {v.x, v.y, v.z, v.w};
            if (x0 >= lo && x0 + 16 <= hi) {            // interior chunk (almost all)
#pragma unroll
              for (int b = 0; b < 16; ++b)
                cd[2 * ((x0 + b) & rmask) + ln] = (unsigned char)(w[b >> 2] >> (8 * (b & 3)));
            } else {
#pragma unroll
              for (int b = 0; b < 16; ++b)
                if (x0 + b >= lo && x0 + b < hi)
                  cd[2 * ((x0 + b) & rmask) + ln] = (unsigned char)(w[b >> 2] >> (8 * (b & 3)));
            }
            // event flags of the haplotype's first / last row, by the thread that wrote it
            const int fr = start > 1 ? start : -1, lr = start + sh.n - 1;
            if (fr >= max(x0, lo) && fr < min(x0 + 16, hi)) cd[2 * (fr & rmask) + ln] |= kCodeFirst;
            if (lr >= max(x0, lo) && lr < min(x0 + 16, hi)) cd[2 * (lr & rmask) + ln] |= kCodeLast;
          }
          // separator row after every haplotype but the lane's last: kCodeIdle (M -> 0, I -> 0)
          if (SEP && e + 1 < cnt && t == 0 && start + sh.n >= r0 && start + sh.n < r1)
            cd[2 * ((start + sh.n) & rmask) + ln] = kCodeIdle;
          start += sh.n + (SEP && e + 1 < cnt ? 1 : 0);
        }
        for (int x = max(r0, start) + t; x < r1; x += P) cd[2 * (x & rmask) + ln] = 4;
      }
    };
    // windows: every row b > 1 where a haplotype begins in either lane -- FIRST for thread
    // t at step b + t, the previous haplotype's LAST for thread P-1 at step b + P - 2: the
    // window [b, b + P), from b - 1 with separator rows (thread 0 reads the idle separator at
    // step b - 1) -- and each lane's final LAST, at step rows + P - 1 (one step).  The first
    // haplotype of each lane needs no window (pre-initialised row 0; the fill steps 1 .. P-1,
    // where threads still read the idle row 0, run checked).  Idle codes are only read in
    // checked steps and in the drain (rows past the stream, whose values no one reads), so
    // the plain step indexes the emission table without the idle-row select (clamped to N).
    // Built once per unit, sorted by start.
    if (first_q || cring) {
      if (live) stage_rows(1, min(rows + 1, RS));
    }
    if (first_q) {
    if (live) {
      if (t == 0) {                                   // merge the two lanes' windows by start
        int* wb = s_win + slot * kStreamMaxWin;
        // lane walk: entry x of a lane with c haplotypes: x < c - 1 -> start of haplotype
        // x + 1 (P steps); x == c - 1 -> the final LAST (one step, at rows + P - 1)
        int ia = 0, ib = 0, ra = 1, rb = 1, nw = 0;
        const int ca = U.cntA, cbn = U.cntB;
        auto entry = [&](int x, int c, int& row, int e0) -> int {
          if (x >= c) return 0x7fffffff;
          if (x == c - 1) return (row + shaps[U.list + e0 + x].n + P - 2) | kWinShort;   // last row + P - 1
          return row + shaps[U.list + e0 + x].n;      // next start b (SEP: b - 1, its separator row)
        };
        while (true) {
          const int va = entry(ia, ca, ra, 0), vb = entry(ib, cbn, rb, ca);
          const int sa = va & ~kWinShort, sbv = vb & ~kWinShort;
          if (va == 0x7fffffff && vb == 0x7fffffff) break;
          const bool takeA = vb == 0x7fffffff || (va != 0x7fffffff && sa <= sbv);
          const int v = takeA ? va : vb;
          if (nw == 0 || wb[nw - 1] != v) wb[nw++] = v;
          if (takeA) { ra += shaps[U.list + ia].n + (SEP ? 1 : 0); ++ia; }
          else { rb += shaps[U.list + ca + ib].n + (SEP ? 1 : 0); ++ib; }
        }
        s_nwin[slot] = nw;
      }
      // per-pair row-0 boundary: fast32 S*beta_1/n (folded), fast64 beta_1/n (scale 2^0),
      // exact fl_dtype(S/n) (wavefront.py:405-406)
      const double sd = ldexp(1.0, MODE == kFast64 ? 0 : E.read_scale[r]);
      const double sdf = EXACT ? sd : (1.0 - s_lut[E.gq[ro]]) * sd;
      for (int e = t; e < U.cntA + U.cntB; e += P)
        s_bs[slot * 2 * kStreamMaxLaneHaps + e] = (S)(sdf / (double)shaps[U.list + e].n);
      if (t == 0) {
        s_meta[slot * 4 + 0] = Lp;
        s_meta[slot * 4 + 1] = E.read_scale[r];
        s_meta[slot * 4 + 2] = __float_as_int(E.read_gsum[r]);
        s_meta[slot * 4 + 3] = m;
      }
    } else if (t == 0) {
      s_nwin[slot] = 0;
    }
    }                                                   // first_q
    int hcA = -1, hcB = -1;                             // current haplotype per lane
    __syncwarp();

    // ---- the stream
    V cb = zero2;                                       // thread 0: boundary D of row s
    V xM = zero2, xI = zero2, xD = zero2;               // neighbour values of the last step
    V yM = zero2, yI = zero2, yD = zero2;
    // every thread reads its own row's code from shared memory one step ahead (row 0 is
    // the idle code N|N: rows before, between and after this thread's stream)
    auto ld_code = [&](int s) -> unsigned {
      const int i = s - t;
      return (i >= 1 && i <= rows_q) ? (unsigned)cd16[(unsigned)i & rmask] : kIdle2;
    };
    // plain steps never read rows <= 0 (the fill runs checked) and ignore event bits, so
    // the drain's rows past the stream may read any entry of this slot: no bounds check
    auto ld_code_plain = [&](int s) -> unsigned { return (unsigned)cd16[(unsigned)(s - t) & (unsigned)(RS - 1)]; };
    unsigned code = kIdle2;
    unsigned pf1 = ld_code(1);
    // stripe q > 0: thread 0's left neighbour is the previous stripe's column
    V* colPrev = team ? colX + (size_t)((q - 1) & 7) * 3 * col_rows : (q & 1) ? colY : colX;
    V* colNext = team ? colX + (size_t)(q & 7) * 3 * col_rows : (q & 1) ? colX : colY;
    const bool col_in = STRIPES && q > 0 && sq;        // uniform over the sub-warp
    const bool from_col = col_in && t == 0;
    const bool to_col = STRIPES && !lastq && t == P - 1 && sq;
    // The column reaches thread 0 through a shared-memory ring of kColRing rows (M, I, D)
    // filled by the whole sub-warp with cp.async 32 rows ahead: an L2 round trip per step
    // (one row ahead in a register) was the striped kernels' bound.  Rows r0 .. r0+31 are
    // requested at step r0 - 32 (r0 = 1 before the stream) and waited for at step r0.
    V* ring = STRIPES ? reinterpret_cast<V*>(s_code + kStreamCodeBytesPerCta) + (size_t)slot * 3 * kColRing : nullptr;
    auto col_fill = [&](int r0) {
      static_assert(!STRIPES || P == 32, "striped tilings are 32 threads wide");
      if (team) {                                       // the rows must be written already
        // flags carry (writing stripe) << 16 | rows: a column reused by stripe q + 8 never
        // looks complete to stripe q + 9 early
        const int need = ((q - 1) << 16) | min(r0 + 31, rows_q);
        if (t == 0)
          while (atomicAdd(&s_prog[(q - 1) & 7], 0) < need) __nanosleep(64);   // acquire: + fence below
        __threadfence_block();
        __syncwarp();
      }
      const int r = min(r0 + t, col_rows - 1);
      const unsigned dst = (unsigned)__cvta_generic_to_shared(ring + ((r0 + t) & (kColRing - 1)));
      cp_async<sizeof(V)>(dst, colPrev + r);
      cp_async<sizeof(V)>(dst + kColRing * sizeof(V), colPrev + col_rows + r);
      cp_async<sizeof(V)>(dst + 2 * kColRing * sizeof(V), colPrev + 2 * col_rows + r);
      cp_async_commit();
    };
    if constexpr (STRIPES)
      if (col_in) col_fill(1);

    // threads whose FIRST needs the haplotype's boundary value: left padding, or thread 0
    const bool slow_first = (q * W + t * K <= s_meta[slot * 4 + 0]) || (t == 0 && q == 0);
    // FIRST(lane L): reset the lane to row 0 of its next haplotype (event paths only run
    // inside windows and read their inputs from shared memory)
    // FULL (the unit's pre-initialisation): M = I = 0, D = the boundary in the left padding.
    // Event (row 1 of a lane's next haplotype): the separator row before it (kCodeIdle)
    // already left M = I = 0 in this thread and in the neighbour's diagonal values, so only
    // D is reset.
    auto first_event = [&](auto lconst, auto full, V& dgM, V& dgI, V& dgD, V& nbM, V& nbI, V& nbD) {
      constexpr int L = decltype(lconst)::value;
      constexpr bool FULL = decltype(full)::value;
      const int hc = L == 0 ? hcA : hcB;                // incremented by the caller
      const int lp = s_meta[slot * 4 + 0];
      const int p0 = q * W + t * K;                     // global padded position of k = 0
      auto bval = [&]() { return s_bs[slot * 2 * kStreamMaxLaneHaps + (L == 0 ? 0 : s_unit[slot].cntA) + hc]; };
      if (p0 > lp) {                                    // no left padding here (most threads)
#pragma unroll
        for (int k = 0; k < K; ++k) {
          if (FULL) { lane_ref<L>(M[k]) = 0; lane_ref<L>(I[k]) = 0; }
          lane_ref<L>(D[k]) = 0;
        }
        lane_ref<L>(dgD) = 0;
      } else {
        const S b = bval();
#pragma unroll
        for (int k = 0; k < K; ++k) {
          if (FULL) { lane_ref<L>(M[k]) = 0; lane_ref<L>(I[k]) = 0; }
          lane_ref<L>(D[k]) = (p0 + k < lp) ? b : (S)0;
        }
        lane_ref<L>(dgD) = (p0 - 1 < lp) ? b : (S)0;    // (stripe 0, thread 0: the boundary)
      }
      if (FULL) { lane_ref<L>(dgM) = 0; lane_ref<L>(dgI) = 0; }
      if (t == 0 && q == 0) {
        const S b = bval();
        lane_ref<L>(cb) = b;
        lane_ref<L>(nbM) = 0; lane_ref<L>(nbI) = 0; lane_ref<L>(nbD) = b;
      }
    };
    // LAST(lane L), thread P-1: the accumulator position holds the pair's sum
    auto last_event = [&](auto lconst) {
      constexpr int L = decltype(lconst)::value;
      const StreamUnit& SU = s_unit[slot];
      const int hc = L == 0 ? hcA : hcB;
      const StreamHap sh = shaps[SU.list + (L == 0 ? 0 : SU.cntA) + hc];
      S res;
      if constexpr (EXACT)                              // j-ordered sum (wavefront.py:156-160)
        res = (lane_ref<L>(D[K - 1]) + lane_ref<L>(M[K - 1])) + (lane_ref<L>(M[K - 2]) + lane_ref<L>(I[K - 2]));
      else                                              // I(m) = d_m I''(m); d_m = dl[K - 1]
        res = (lane_ref<L>(D[K - 1]) + lane_ref<L>(M[K - 1])) + (lane_ref<L>(M[K - 2]) + dl[K - 1] * lane_ref<L>(I[K - 2]));
      const int mm = s_meta[slot * 4 + 3];
      if constexpr (MODE == kFast64) {
        // FP64 retry result; near/below the f64 flush floor -> bit-exact FP64 kernel
        if (res >= 0x1p-900 && isfinite(res)) {
          E.acc[sh.pair] = res;
          E.status[sh.pair] = kStatusOk | kStatusRetriedF64;
        } else {
          append_item(E.ex64, E.ex64_count, E.list_cap, exact_slot_for(mm), ExactItem{sh.pair, SU.read, sh.hap, 0});
        }
      } else if constexpr (MODE == kExact32) {
        const bool bad = !(res > 0.f) || !isfinite(res);
        if (bad && E.retry_f64) {
          E.status[sh.pair] = kStatusRetriedF64;
          const int g64 = r64_geom_for(mm);
          if (E.r64b.enabled && E.r64b.units[g64]) s_flag[2 * slot + L] |= 1u << hc;   // -> FP64 stream unit
          else append_item(E.fx64, E.fx64_count, E.list_cap, exact_slot_for(mm), ExactItem{sh.pair, SU.read, sh.hap, 0});
        } else {
          E.acc[sh.pair] = (double)res;
          E.status[sh.pair] = bad ? kStatusOverflow : kStatusExactF32;
        }
      } else if constexpr (MODE == kExact64) {
        const bool bad = !(res > 0.0) || !isfinite(res);
        E.acc[sh.pair] = res;
        const uint8_t keep = E.status[sh.pair] & kStatusRetriedF64;
        E.status[sh.pair] = (uint8_t)((bad ? kStatusOverflow : kStatusOk) | keep);
      } else {
        const int v = stream_finish32(E, res, sh.pair, sh.n, __int_as_float(s_meta[slot * 4 + 2]),
                                      s_meta[slot * 4 + 1]);
        if (v == 1) {                                   // guard band: bit-exact rerun
          const int c = s_ninl[slot];
          if (c < kInlineBand && s_meta[slot * 4 + 0] + mm + 1 <= W && atomicAdd(E.band_inline, 1) < E.band_budget) {
            // the first few per launch: rerun by this warp right after the unit (no
            // post-pass latency when band pairs are rare)
            s_inl[slot * kInlineBand + c] = ExactItem{sh.pair, SU.read, sh.hap, s_meta[slot * 4 + 1]};
            s_ninl[slot] = c + 1;
          } else if (E.rx32.enabled && rx32_geom_for(mm) >= 0) s_band[2 * slot + L] |= 1u << hc;
          else append_item(E.ex32, E.ex32_count, E.list_cap, exact_slot_for(mm),
                           ExactItem{sh.pair, SU.read, sh.hap, s_meta[slot * 4 + 1]});
        } else if (v == 2) {                            // FP32 underflow: FP64 retry unit
          if (E.r64.enabled && r64_geom_for(mm) >= 0) s_flag[2 * slot + L] |= 1u << hc;
          else append_item(E.fx64, E.fx64_count, E.list_cap, exact_slot_for(mm), ExactItem{sh.pair, SU.read, sh.hap, 0});
        }
      }
    };

    // One step; (dgM, dgI, dgD) holds the previous step's neighbour values (the diagonal
    // input of position 0) and the shuffle writes this step's into (nbM, nbI, nbD): the
    // caller alternates two register sets so no copy is needed between steps.
    auto step = [&](const int s, auto checked, V& dgM, V& dgI, V& dgD, V& nbM, V& nbI, V& nbD) {
      constexpr bool CHECK = decltype(checked)::value;
      {
        const V lm = M[K - 1], li = I[K - 1], ld = D[K - 1];
        nbM.x = __shfl_up_sync(FULL, lm.x, 1, P);
        nbM.y = __shfl_up_sync(FULL, lm.y, 1, P);
        nbI.x = __shfl_up_sync(FULL, li.x, 1, P);
        nbI.y = __shfl_up_sync(FULL, li.y, 1, P);
        nbD.x = __shfl_up_sync(FULL, ld.x, 1, P);
        nbD.y = __shfl_up_sync(FULL, ld.y, 1, P);
      }
      if constexpr (STRIPES)
        if (col_in && (s & 31) == 1) {                  // rows s .. s+31 landed; request the next 32
          cp_async_wait_all();
          __syncwarp();
          col_fill(s + 32);
        }
      if (t == 0) {
        if (from_col) {
          const int x = s & (kColRing - 1);
          nbM = ring[x]; nbI = ring[kColRing + x]; nbD = ring[2 * kColRing + x];
        } else {
          nbM = zero2; nbI = zero2; nbD = cb;
        }
      }
      code = pf1;
      pf1 = CHECK ? ld_code(s + 1) : ld_code_plain(s + 1);
      if constexpr (CHECK && SEP && F64) {
        // separator rows already zeroed M and I: a FIRST resets D and the diagonal D, done
        // predicated by every thread (no divergent branch between consecutive checked
        // steps); threads with left padding and thread 0 (the boundary) also take the
        // handler.  FP64 (32,8) / (32,7) -1.5 %; in FP32 the selects cost more than the
        // branch saves (c2 +4 %), so FP32 keeps the branchy handler.
        const bool fA = (code & kCodeFirst) != 0, fB = (code & (kCodeFirst << 8)) != 0;
        hcA += fA ? 1 : 0;
        hcB += fB ? 1 : 0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          if (fA) D[k].x = 0;
          if (fB) D[k].y = 0;
        }
        if (fA) dgD.x = 0;
        if (fB) dgD.y = 0;
        if (slow_first && (fA || fB)) {
          if (fA) first_event(std::integral_constant<int, 0>{}, std::false_type{}, dgM, dgI, dgD, nbM, nbI, nbD);
          if (fB) first_event(std::integral_constant<int, 1>{}, std::false_type{}, dgM, dgI, dgD, nbM, nbI, nbD);
        }
      } else if (CHECK && (code & ((kCodeFirst << 8) | kCodeFirst))) {
        using Full = std::integral_constant<bool, !SEP>;
        if (code & kCodeFirst) {
          ++hcA;
          first_event(std::integral_constant<int, 0>{}, Full{}, dgM, dgI, dgD, nbM, nbI, nbD);
        }
        if (code & (kCodeFirst << 8)) {
          ++hcB;
          first_event(std::integral_constant<int, 1>{}, Full{}, dgM, dgI, dgD, nbM, nbI, nbD);
        }
      }
      // plain steps read idle codes only in the drain (rows no one reads): they clamp to N
      // (one IMNMX instead of the select, and the table read stays in this slot)
      const int cA = CHECK ? (int)(code & 7) : min((int)(code & 7), 4);
      const int cB = CHECK ? (int)((code >> 8) & 7) : min((int)((code >> 8) & 7), 4);
      const EV* EA = (CHECK && cA == kCodeIdle) ? s_zero + t : Et + (cA * KE) * P + t;
      const EV* EB = (CHECK && cB == kCodeIdle) ? s_zero + t : Et + (cB * KE) * P + t;
      // fast FP32 at occupancy 2 (K = 14, 16) has the registers for the carried values
      constexpr bool FUSED = !EXACT && (F64 ? !STRIPES : K >= 12);
      if constexpr (FUSED) {
        // one ascending pass: position k's D'', M~ and I'' from position k's and k-1's
        // previous-step values (carried in pmo/pio/pdo) and k-1's new M~, I'' -- step s+1
        // at position k needs only step s up to k, so consecutive steps overlap
        V pmo = dgM, pio = dgI, pdo = dgD;
        V lM = nbM, lI = nbI;
#pragma unroll
        for (int ke = 0; ke < KE; ++ke) {
          const EV la = EA[ke * P];
          const EV lb = EB[ke * P];
#pragma unroll
          for (int kk = 0; kk < EW; ++kk) {
            const int k = ke * EW + kk;
            if (k >= K) continue;                       // padded chunk (odd K)
            const V mo = M[k], io = I[k], dold = D[k];
            D[k] = A::fma(ep[k], dold, mo);
            V x = A::fma(dl[k], pio, pmo);
            x = A::fma(zt[k], pdo, x);
            M[k].x = ev_comp(la, kk) * x.x;
            M[k].y = ev_comp(lb, kk) * x.y;
            I[k] = A::fma(be[k], lI, lM);
            lM = M[k];
            lI = I[k];
            pmo = mo; pio = io; pdo = dold;
          }
        }
      } else {
        // pass 1 (descending): D from the previous row, M from the previous-row diagonal
#pragma unroll
        for (int ke = KE - 1; ke >= 0; --ke) {
          const EV la = EA[ke * P];
          const EV lb = EB[ke * P];
#pragma unroll
          for (int kk = EW - 1; kk >= 0; --kk) {
            const int k = ke * EW + kk;
            if (k >= K) continue;                       // padded chunk (odd K)
            const V pm = (k > 0) ? M[k - 1] : dgM;
            const V pi = (k > 0) ? I[k - 1] : dgI;
            const V pd = (k > 0) ? D[k - 1] : dgD;
            if constexpr (EXACT) {
              // D = zt*M(i,j-1) + ep*D(i,j-1); M = lam*(al*M + be*(I + D)) (reference.py:111-113)
              D[k] = flush2(A::xadd(A::xmul(zt[k], M[k]), A::xmul(ep[k], D[k])), thr);
              V x = A::xadd(A::xmul(al[k], pm), A::xmul(be[k], A::xadd(pi, pd)));
              x.x = A::mul1(ev_comp(la, kk), x.x);
              x.y = A::mul1(ev_comp(lb, kk), x.y);
              M[k] = flush2(x, thr);
            } else {
              D[k] = A::fma(ep[k], D[k], M[k]);
              V x = A::fma(dl[k], pi, pm);
              x = A::fma(zt[k], pd, x);
              M[k].x = ev_comp(la, kk) * x.x;
              M[k].y = ev_comp(lb, kk) * x.y;
            }
          }
        }
        // pass 2 (ascending): I chain along the read within the current row
        {
          V lM = nbM, lI = nbI;
#pragma unroll
          for (int k = 0; k < K; ++k) {
            if constexpr (EXACT) I[k] = flush2(A::xadd(A::xmul(dl[k], lM), A::xmul(ep[k], lI)), thr);
            else I[k] = A::fma(be[k], lI, lM);
            lM = M[k];
            lI = I[k];
          }
        }
      }
      if (to_col) {
        const int j = s - (P - 1);
        if (j >= 1 && j <= rows_q) {
          colNext[j] = M[K - 1]; colNext[col_rows + j] = I[K - 1]; colNext[2 * col_rows + j] = D[K - 1];
          if (team && ((j & 31) == 0 || j == rows_q)) {   // publish the rows written so far
            __threadfence();
            atomicExch(&s_prog[q & 7], (q << 16) | j);   // release: after the fence above
          }
        }
      }
      if (CHECK && lastq && (code & ((kCodeLast << 8) | kCodeLast)) && t == P - 1) {
        if (code & kCodeLast) last_event(std::integral_constant<int, 0>{});
        if (code & (kCodeLast << 8)) last_event(std::integral_constant<int, 1>{});
      }
    };

    // row 0 of each lane's first haplotype: the fill steps (kCodeIdle) keep it until the
    // thread's first row, so no FIRST event is needed for it
    if (sq) {
      if (U.cntA > 0) { hcA = 0; first_event(std::integral_constant<int, 0>{}, std::true_type{}, xM, xI, xD, yM, yI, yD); }
      if (U.cntB > 0) { hcB = 0; first_event(std::integral_constant<int, 1>{}, std::true_type{}, xM, xI, xD, yM, yI, yD); }
    }

    // event-free stretches run the plain step; windows run the event-checking one, for as
    // long as any sub-warp of the warp is inside one of its windows; ring units restage a
    // half-ring of row codes at the (warp-uniform) refill steps nr: at step (b+1)H + P the
    // rows of block b (rows bH .. (b+1)H-1, last read at step (b+1)H + P - 2) are free and
    // block b+2 (first read at step (b+2)H - 1) is written
    const int nwin = s_nwin[slot];
    const int* wb = s_win + slot * kStreamMaxWin;
    // this sub-warp's earliest unfinished window [cur_s, cur_e), kept in registers; the
    // first is the fill [1, P)
    constexpr int WL = P + (SEP ? 1 : 0);               // window length (from the separator row)
    int wi = -1;
    int cur_s = 1, cur_e = P;
    int s = 1;
    auto advance = [&]() {
      while (cur_e <= s) {
        if (++wi < nwin) { cur_s = wb[wi] & ~kWinShort; cur_e = cur_s + ((wb[wi] & kWinShort) ? 1 : WL); }
        else { cur_s = 0x7fffffff; cur_e = 0x7fffffff; }
      }
    };
    constexpr int H = RS / 2;
    int nr = __any_sync(FULL, cring && sq) ? H + P : 0x7fffffff;
    // Steps always run in pairs (plain or checked) so the two register sets alternate with
    // no copies: a stretch that ends one step before a window starts the checked pair one
    // step early (a checked step is correct anywhere), and steps past `steps` compute rows
    // no one reads.  A refill may run one step after nr: block b + 2 is first read at step
    // (b + 2)H - 1, far ahead (H > P + 2).
#pragma unroll 1
    while (s <= steps) {
      if (s >= nr) {
        __syncwarp();
        if (cring && sq) stage_rows(nr - P + H, min(nr - P + 2 * H, rows + 1));
        __syncwarp();
        nr += H;
      }
      advance();
      const int e = max((int)__reduce_min_sync(FULL, (unsigned)cur_s), s);
      const int fend = min(min(e, nr), steps + 1);
#pragma unroll 1
      for (; s + 1 < fend; s += 2) {
        step(s, std::false_type{}, xM, xI, xD, yM, yI, yD);
        step(s + 1, std::false_type{}, yM, yI, yD, xM, xI, xD);
      }
      if (s > steps || (s >= nr && s == fend)) continue;
      // some sub-warp is inside a window (or one step before it): event-checking pairs
      pf1 = ld_code(s);                                 // the plain steps' prefetch is unchecked
#pragma unroll 1
      for (;;) {
        step(s, std::true_type{}, xM, xI, xD, yM, yI, yD);
        step(s + 1, std::true_type{}, yM, yI, yD, xM, xI, xD);
        s += 2;
        if (s > steps || s >= nr) break;
        advance();
        if (!__any_sync(FULL, cur_s <= s)) break;
      }
    }
    if constexpr (STRIPES) cp_async_wait_all();      // the ring is refilled by the next stripe
    __syncwarp();
    }                                                   // stripes
    if constexpr (MODE == kExact32) {
      // guard-band pairs whose exact rerun underflowed -> second-stage FP64 stream units
      // (long reads, and every read of a large call; otherwise the per-pair FP64 list)
      if (t == 0 && live && (s_flag[2 * slot] | s_flag[2 * slot + 1])) {
        const int g64 = r64_geom_for(m);
        emit_retry_units(U, shaps, s_flag + 2 * slot, E.r64b, g64, stream_cap_of(r64_geom_P(g64)), m,
                         E.r64b.lane_haps, 256, SepRows<kFast64>::value);
      }
    }
    if constexpr (MODE == kFast32) {
      // this unit's FP32-underflowed and guard-band pairs -> device-built stream units
      if (t == 0 && live) {
        if (s_flag[2 * slot] | s_flag[2 * slot + 1]) {
          const int g64 = r64_geom_for(m);
          emit_retry_units(U, shaps, s_flag + 2 * slot, E.r64, g64, stream_cap_of(r64_geom_P(g64)), m,
                           E.r64.lane_haps, 256, SepRows<kFast64>::value);
        }
        if (s_band[2 * slot] | s_band[2 * slot + 1]) {
          const int gx = rx32_geom_for(m);
          emit_retry_units(U, shaps, s_band + 2 * slot, E.rx32, gx, stream_cap_of(rx32_geom_P(gx)), m,
                           E.rx32.lane_haps, 512, SepRows<kExact32>::value);
        }
      }
      // inline guard-band reruns (same tiling; the emission-table slot is free again)
      const int nin = s_ninl[slot];
      const int nmax = __reduce_max_sync(FULL, (unsigned)nin);
#pragma unroll 1
      for (int x = 0; x < nmax; ++x) {
        const bool mine = x < nin;
        const ExactItem it = mine ? s_inl[slot * kInlineBand + x] : ExactItem{-1, U.read, shaps[U.list].hap, 0};
        exact_item<float, P, K>(E, it, mine, s_lut, reinterpret_cast<float*>(Et), nullptr, nullptr, 0, t);
        __syncwarp();
      }
    }
  }
}

// ---------------------------------------------------------------------------------
// k_fast64<P, K>: FP64 retry of pairs whose FP32 result underflowed (GATK behaviour).
// Same folded recurrence as k_fast (FMA, 7 DP operations per cell, no per-cell flush),
// one pair per sub-warp lane set, scale 2^0.  Accuracy vs the reference's f64 path is
// ~1e-13 relative (FMA/reassociation only); the reference's 2^-970 flush is provably
// irrelevant above 2^-900, and results below that are re-run on k_exact<double>.
// ---------------------------------------------------------------------------------
template <int P, int K>
__device__ __forceinline__ void
fast64_list(const EngineDev& E, int slot, int* __restrict__ counter, double* __restrict__ colbuf, int col_rows) {
  constexpr int W = P * K, G = 32 / P;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* s_lut = reinterpret_cast<double*>(smem_raw);
  double* s_E = reinterpret_cast<double*>(smem_raw + 96 * sizeof(double));
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int sw = lane / P, t = lane % P;
  const int count = min(E.fx64_count[slot], E.list_cap[slot]);
  if (count == 0) return;
  double* Et = s_E + (size_t)((wib * G + sw) * 5 * K) * P;   // Et[(c*K + k)*P + t]
  const int gwarp = blockIdx.x * (blockDim.x >> 5) + wib;
  double* colX = colbuf + (size_t)(gwarp * G + sw) * 2 * 3 * col_rows;
  double* colY = colX + 3 * col_rows;
  const ExactItem* items = E.fx64[slot];
  for (;;) {
    int g = 0;
    if (lane == 0) g = atomicAdd(counter, 1);
    g = __shfl_sync(FULL, g, 0);
    if (g * G >= count) break;
    const int u = g * G + sw;
    const bool has = u < count;
    const ExactItem it = items[has ? u : g * G];
    const int r = it.read, m = E.read_m[r];
    const int64_t ro = E.roff[r];
    const int n = (int)(E.hoff[it.hap + 1] - E.hoff[it.hap]);
    const bool live = has && !(E.read_flags[r] & 1);
    const int steps = __reduce_max_sync(FULL, live ? n + P - 1 : 0);
    const int Q = (m + 1 + W - 1) / W;
    const int Qw = __reduce_max_sync(FULL, live ? Q : 0);
    const int Lp = Q * W - m - 1;
    const double bfirst = 1.0 - s_lut[E.gq[ro]];
    const double bS = bfirst / (double)n;                    // scale 2^0 (f64 config)
    const int8_t* h = E.hbases + E.hoff[it.hap];
    double res = 0.0;
    double* colPrev = colX;
    double* colNext = colY;
    for (int q = 0; q < Qw; ++q) {
      const bool sact = live && q < Q;
      double be[K], dl[K], ep[K], zp[K], M[K], I[K], D[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int p = q * W + t * K + k;
        double lam[5];
        M[k] = 0.0; I[k] = 0.0;
        if (p < Lp) {
          be[k] = 0.0; dl[k] = 0.0; ep[k] = 1.0; zp[k] = 0.0; D[k] = bS;
#pragma unroll
          for (int c = 0; c < 5; ++c) lam[c] = 0.0;
        } else if (p < Lp + m) {
          const int i0 = p - Lp;
          const double d = s_lut[E.iq[ro + i0]], z = s_lut[E.dq[ro + i0]];
          const double e = s_lut[E.gq[ro + i0]], qe = s_lut[E.bq[ro + i0]];
          const double a = (1.0 - d) - z;
          double anext = 1.0, bnext = 0.0;
          if (i0 + 1 < m) {
            anext = (1.0 - s_lut[E.iq[ro + i0 + 1]]) - s_lut[E.dq[ro + i0 + 1]];
            bnext = 1.0 - s_lut[E.gq[ro + i0 + 1]];
          }
          be[k] = 1.0 - e; dl[k] = d / a; ep[k] = e; zp[k] = bnext * z / anext; D[k] = 0.0;
          const int rc = E.rbases[ro + i0];
          const double lm = anext * (1.0 - qe), lx = anext * (qe / 3.0);
#pragma unroll
          for (int c = 0; c < 5; ++c) lam[c] = (rc == c || rc == 4 || c == 4) ? lm : lx;
        } else {
          be[k] = 1.0; dl[k] = 0.0; ep[k] = 1.0; zp[k] = 1.0; D[k] = 0.0;
#pragma unroll
          for (int c = 0; c < 5; ++c) lam[c] = 1.0;
        }
#pragma unroll
        for (int c = 0; c < 5; ++c) Et[(c * K + k) * P + t] = lam[c];
      }
      if (sact && t == P - 1 && q < Q - 1) {
        colNext[0] = M[K - 1]; colNext[col_rows] = I[K - 1]; colNext[2 * col_rows] = D[K - 1];
      }
      double nbM = 0.0, nbI = 0.0, nbD = 0.0;
      if (t == 0) {
        if (q == 0) nbD = bS;
        else if (sact) { nbM = colPrev[0]; nbI = colPrev[col_rows]; nbD = colPrev[2 * col_rows]; }
      }
      __syncwarp();
      // one-row-ahead prefetch of the boundary column (thread 0) and the characters
      double pfM = 0.0, pfI = 0.0, pfD = 0.0;
      if (t == 0 && q > 0 && sact) {
        const int jj = min(1, n);
        pfM = colPrev[jj]; pfI = colPrev[col_rows + jj]; pfD = colPrev[2 * col_rows + jj];
      }
      int cpf = (sact && 1 - t >= 1 && 1 - t <= n) ? h[-t] : 0;
      for (int s = 1; s <= steps; ++s) {
        const int j = s - t;
        const double dgM = nbM, dgI = nbI, dgD = nbD;
        nbM = __shfl_up_sync(FULL, M[K - 1], 1, P);
        nbI = __shfl_up_sync(FULL, I[K - 1], 1, P);
        nbD = __shfl_up_sync(FULL, D[K - 1], 1, P);
        if (t == 0) {
          if (q == 0) { nbM = 0.0; nbI = 0.0; nbD = bS; }
          else if (sact) {
            nbM = pfM; nbI = pfI; nbD = pfD;
            const int jj = min(s + 1, n);
            pfM = colPrev[jj]; pfI = colPrev[col_rows + jj]; pfD = colPrev[2 * col_rows + jj];
          }
        }
        const int c = cpf;
        cpf = (sact && j + 1 >= 1 && j + 1 <= n) ? h[j] : 0;
        if (sact && j >= 1 && j <= n) {
          const double* Ec = Et + (c * K) * P + t;
#pragma unroll
          for (int k = K - 1; k >= 0; --k) {
            D[k] = fma(ep[k], D[k], zp[k] * M[k]);
            const double pm = (k > 0) ? M[k - 1] : dgM;
            const double pi = (k > 0) ? I[k - 1] : dgI;
            const double pd = (k > 0) ? D[k - 1] : dgD;
            M[k] = Ec[k * P] * (pm + fma(be[k], pi, pd));
          }
          double lM = nbM, lI = nbI;
#pragma unroll
          for (int k = 0; k < K; ++k) {
            I[k] = fma(ep[k], lI, dl[k] * lM);
            lM = M[k];
            lI = I[k];
          }
          if (t == P - 1) {
            if (q == Q - 1) {
              if (j == n) res = (D[K - 1] + M[K - 1]) + (M[K - 2] + I[K - 2]);
            } else {
              colNext[j] = M[K - 1]; colNext[col_rows + j] = I[K - 1]; colNext[2 * col_rows + j] = D[K - 1];
            }
          }
        }
      }
      __syncwarp();
      double* tmp = colPrev; colPrev = colNext; colNext = tmp;
    }
    if (live && t == P - 1) {
      if (res >= 0x1p-900 && isfinite(res)) {
        E.acc[it.pair] = res;
        E.status[it.pair] = kStatusOk | kStatusRetriedF64;
      } else {                                      // near/below the f64 flush floor: exact
        append_item(E.ex64, E.ex64_count, E.list_cap, exact_slot_for(m), it);
      }
    }
  }
}

// k_exact<T, P, K>: a complete work list (host-provided + appended before launch).
template <typename T, int P, int K>
__device__ __forceinline__ void
exact_list(const EngineDev& E, int slot, int* __restrict__ counter, T* __restrict__ colbuf, int col_rows) {
  constexpr int G = 32 / P;
  constexpr bool kIsF32 = sizeof(T) == 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* s_lut = reinterpret_cast<double*>(smem_raw);
  T* s_E = reinterpret_cast<T*>(smem_raw + 96 * sizeof(double));
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int sw = lane / P, t = lane % P;
  const int count = min(kIsF32 ? E.ex32_count[slot] : E.ex64_count[slot], E.list_cap[slot]);
  if (count == 0) return;
  T* Et = s_E + (size_t)((wib * G + sw) * 5 * K) * P;   // Et[(c*K + k)*P + t]
  const int gwarp = blockIdx.x * (blockDim.x >> 5) + wib;
  T* colX = colbuf + (size_t)(gwarp * G + sw) * 2 * 3 * col_rows;
  T* colY = colX + 3 * col_rows;
  const ExactItem* items = kIsF32 ? E.ex32[slot] : E.ex64[slot];
  for (;;) {
    int g = 0;
    if (lane == 0) g = atomicAdd(counter, 1);
    g = __shfl_sync(0xffffffffu, g, 0);
    if (g * G >= count) break;
    const int u = g * G + sw;
    const bool has = u < count;
    const ExactItem it = items[has ? u : g * G];
    exact_item<T, P, K>(E, it, has, s_lut, Et, colX, colY, col_rows, t);
  }
}

}  // namespace phmm
