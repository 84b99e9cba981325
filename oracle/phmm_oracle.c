/*
 * phmm_oracle.c — CPU restatement of the reference Pair-HMM forward recursion.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * engine and the CPU baseline of bench.py; it is never linked into, loaded by,
 * or called from the product path (paper_2411_11547_b200/).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * use it.
 *
 * What it restates (reference = /root/reference/pkg/src/pairhmm):
 *   - transitions      prob.py:66-78   delta=LUT[ins], zeta=LUT[del], eps=LUT[gcp],
 *                                      alpha=(1-delta)-zeta, beta=1-eps (f64), degenerate
 *                                      if delta+zeta >= 1.0 (f64)
 *   - emissions        prob.py:90-112  1-Q if r==c or r==N or c==N, else Q/3 (f64)
 *   - dtype cast       wavefront.py:347-355  tables built in f64 then cast to dtype
 *   - boundary         wavefront.py:405-406, reference.py:42-45  D(0,j)=dtype(2^s/n), j>=0
 *   - recurrence       reference.py:106-117 / wavefront.py:137-155 (no FMA anywhere)
 *                        M = lam*(al*M[i-1,j-1] + be*(I[i-1,j-1] + D[i-1,j-1]))
 *                        I = dl*M[i-1,j] + ep*I[i-1,j]
 *                        D = zt*M[i,j-1] + ep*D[i,j-1]
 *                      every store v >= flush ? v : 0 (flush 2^-90 f32, 2^-970 f64;
 *                      prob.py:38-39)
 *   - accumulation     reference.py:120-122 / wavefront.py:156-160  acc = acc + (M + I),
 *                      j increasing, in dtype
 * The f32 instance is the reference's wavefront f32 engine, which its docstring
 * (wavefront.py:14-18) and tests (test_acceptance.py:88-103) state is
 * bit-identical to the row-major linear-space order used here; the golden
 * fixtures under tests/golden/ pin that claim against the reference itself.
 *
 * Build (oracle/Makefile): gcc -O2 -ffp-contract=off -fno-fast-math -fPIC -shared.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { OR_OK = 0, OR_OVERFLOW = 1, OR_TOO_SMALL = 2, OR_DEGENERATE = 3 };

#define FLUSH_F32 0x1p-90f
#define FLUSH_F64 0x1p-970

/* Returns 1 if the read is degenerate (prob.py:71-75). */
static int degenerate(const uint8_t* iq, const uint8_t* dq, int m, const double* lut) {
  for (int i = 0; i < m; i++)
    if (lut[iq[i]] + lut[dq[i]] >= 1.0) return 1;
  return 0;
}

#define DEFINE_PAIR(NAME, T, FLUSH)                                                            \
  static T NAME(const int8_t* r, const uint8_t* bq, const uint8_t* iq, const uint8_t* dq,      \
                const uint8_t* gq, int m, const int8_t* h, int n, int scale_log2,              \
                const double* lut, T* work) {                                                  \
    T* Mp = work;                                                                              \
    T* Ip = Mp + (n + 1);                                                                      \
    T* Dp = Ip + (n + 1);                                                                      \
    T* Mc = Dp + (n + 1);                                                                      \
    T* Ic = Mc + (n + 1);                                                                      \
    T* Dc = Ic + (n + 1);                                                                      \
    const T zero = (T)0;                                                                       \
    const T flush = FLUSH;                                                                     \
    const T bnd = (T)(ldexp(1.0, scale_log2) / (double)n);                                     \
    for (int j = 0; j <= n; j++) { Mp[j] = zero; Ip[j] = zero; Dp[j] = bnd; }                  \
    for (int i = 1; i <= m; i++) {                                                             \
      const double dl64 = lut[iq[i - 1]], zt64 = lut[dq[i - 1]], ep64 = lut[gq[i - 1]];       \
      const double q64 = lut[bq[i - 1]];                                                       \
      const T al = (T)((1.0 - dl64) - zt64), be = (T)(1.0 - ep64);                             \
      const T dl = (T)dl64, ep = (T)ep64, zt = (T)zt64;                                        \
      const T lm = (T)(1.0 - q64), lx = (T)(q64 / 3.0);                                        \
      const int rc = r[i - 1];                                                                 \
      Mc[0] = zero; Ic[0] = zero; Dc[0] = zero;                                                \
      for (int j = 1; j <= n; j++) {                                                           \
        const int hc = h[j - 1];                                                               \
        const T lam = (rc == hc || rc == 4 || hc == 4) ? lm : lx;                              \
        const T a1 = al * Mp[j - 1];                                                           \
        const T s1 = Ip[j - 1] + Dp[j - 1];                                                    \
        const T b1 = be * s1;                                                                  \
        const T mv = lam * (a1 + b1);                                                          \
        const T i1 = dl * Mp[j];                                                               \
        const T i2 = ep * Ip[j];                                                               \
        const T iv = i1 + i2;                                                                  \
        const T d1 = zt * Mc[j - 1];                                                           \
        const T d2 = ep * Dc[j - 1];                                                           \
        const T dv = d1 + d2;                                                                  \
        Mc[j] = mv >= flush ? mv : zero;                                                       \
        Ic[j] = iv >= flush ? iv : zero;                                                       \
        Dc[j] = dv >= flush ? dv : zero;                                                       \
      }                                                                                        \
      T* t;                                                                                    \
      t = Mp; Mp = Mc; Mc = t;                                                                 \
      t = Ip; Ip = Ic; Ic = t;                                                                 \
      t = Dp; Dp = Dc; Dc = t;                                                                 \
    }                                                                                          \
    T acc = zero;                                                                              \
    for (int j = 1; j <= n; j++) acc = acc + (Mp[j] + Ip[j]);                                  \
    return acc;                                                                                \
  }

DEFINE_PAIR(pair_f32, float, FLUSH_F32)
DEFINE_PAIR(pair_f64, double, FLUSH_F64)

/*
 * Score one pair.  precision: 0 = f32, 1 = f64.  Returns an OR_* status; on
 * OR_OK / OR_OVERFLOW *acc_out holds the raw (scaled) accumulator widened to
 * double.  work must hold 6*(n+1) doubles.
 */
int oracle_pair(const int8_t* r, const uint8_t* bq, const uint8_t* iq, const uint8_t* dq,
                const uint8_t* gq, int m, const int8_t* h, int n, int precision, int scale_log2,
                const double* lut, double* acc_out, double* work) {
  if (degenerate(iq, dq, m, lut)) { *acc_out = NAN; return OR_DEGENERATE; }
  double acc;
  if (precision == 0)
    acc = (double)pair_f32(r, bq, iq, dq, gq, m, h, n, scale_log2, lut, (float*)work);
  else
    acc = pair_f64(r, bq, iq, dq, gq, m, h, n, scale_log2, lut, work);
  *acc_out = acc;
  return (acc <= 0.0 || !isfinite(acc)) ? OR_OVERFLOW : OR_OK;
}

/* ---- batch driver (pthreads), flat layout identical to the engine C-ABI ---- */

typedef struct {
  const int8_t* rb; const uint8_t *bq, *iq, *dq, *gq; const int64_t* roff;
  const int8_t* hb; const int64_t* hoff;
  const int64_t* pair_read; const int64_t* pair_hap; int64_t npairs;
  int precision; int scale_log2; int max_m; const double* lut;
  double* acc; uint8_t* status;
  int64_t next; pthread_mutex_t mu;
} job_t;

static void* worker(void* arg) {
  job_t* J = (job_t*)arg;
  size_t cap = 0; double* work = NULL;
  for (;;) {
    pthread_mutex_lock(&J->mu);
    int64_t lo = J->next; J->next += 64;
    pthread_mutex_unlock(&J->mu);
    if (lo >= J->npairs) break;
    int64_t hi = lo + 64 < J->npairs ? lo + 64 : J->npairs;
    for (int64_t p = lo; p < hi; p++) {
      int64_t ri = J->pair_read[p], hi_ = J->pair_hap[p];
      int64_t r0 = J->roff[ri], m = J->roff[ri + 1] - r0;
      int64_t h0 = J->hoff[hi_], n = J->hoff[hi_ + 1] - h0;
      if (m > J->max_m) { J->acc[p] = NAN; J->status[p] = OR_TOO_SMALL; continue; }
      size_t need = 6 * (size_t)(n + 1);
      if (need > cap) { free(work); cap = need; work = (double*)malloc(cap * sizeof(double)); }
      J->status[p] = (uint8_t)oracle_pair(J->rb + r0, J->bq + r0, J->iq + r0, J->dq + r0, J->gq + r0,
                                          (int)m, J->hb + h0, (int)n, J->precision, J->scale_log2,
                                          J->lut, &J->acc[p], work);
    }
  }
  free(work);
  return NULL;
}

/*
 * Score an explicit list of (read, hap) pairs over flat arrays.  max_m is the
 * largest registered p*k (reads longer than it are OR_TOO_SMALL, pipeline.py:94-96).
 * Returns 0 on success.
 */
int oracle_score_pairs(const int8_t* read_bases, const uint8_t* bq, const uint8_t* iq,
                       const uint8_t* dq, const uint8_t* gq, const int64_t* read_off,
                       const int8_t* hap_bases, const int64_t* hap_off,
                       const int64_t* pair_read, const int64_t* pair_hap, int64_t npairs,
                       int precision, int scale_log2, int max_m, const double* lut, int threads,
                       double* acc_out, uint8_t* status_out) {
  job_t J;
  memset(&J, 0, sizeof(J));
  J.rb = read_bases; J.bq = bq; J.iq = iq; J.dq = dq; J.gq = gq; J.roff = read_off;
  J.hb = hap_bases; J.hoff = hap_off; J.pair_read = pair_read; J.pair_hap = pair_hap;
  J.npairs = npairs; J.precision = precision; J.scale_log2 = scale_log2; J.max_m = max_m;
  J.lut = lut; J.acc = acc_out; J.status = status_out; J.next = 0;
  pthread_mutex_init(&J.mu, NULL);
  if (threads < 1) threads = 1;
  if (threads == 1) {
    worker(&J);
  } else {
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    for (int t = 0; t < threads; t++) pthread_create(&th[t], NULL, worker, &J);
    for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
    free(th);
  }
  pthread_mutex_destroy(&J.mu);
  return 0;
}
