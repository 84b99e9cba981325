// phmm_aux.cu — the engine's small kernels and their host launchers (libphmm.so):
//   k_l2_prefetch / k_precompute   per call: L2 warm-up of the per-unit inputs, per-read
//                                  degenerate flag + guard-band bound Gsum, counter reset
//   k_validate                     input content checks (16 B per thread-iteration)
//   k_exact_all<T> / k_fast64_all  per-pair post-pass lists (bit-exact FP32/FP64, FP64 retry)
// The stream kernels (k_stream<MODE,P,K>) are instantiated in k_stream_*.cu; every
// translation unit compiles on its own (no relocatable device code), in parallel.
#include "phmm_registry.h"

namespace phmm {

// ---------------------------------------------------------------------------------
// k_precompute: one warp per read.
// Gsum bounds sum over positions i of the backward sensitivities B_M(i)+B_I(i)+B_D(i)
// of the final accumulator w.r.t. a cell value, with every emission replaced by 1.
// Flushing a value v < 2^-90 changes the final accumulator by at most v*B, so
//   0 <= unflushed - flushed <= 2^-90 * n * Gsum        (guard band)
// ---------------------------------------------------------------------------------
__device__ __forceinline__ void prefetch_l2(const void* base, int64_t bytes, int64_t tid, int64_t nth) {
  const char* p = static_cast<const char*>(base);
  for (int64_t off = tid * 128; off < bytes; off += nth * 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(p + off));
}

// Pulls the inputs the stream kernels read once per unit (work units, haplotype lists
// and bases, read bases and base qualities) into L2; runs beside k_precompute.
__global__ void k_l2_prefetch(const void* pf0, int64_t pf0_bytes, const void* pf1, int64_t pf1_bytes,
                              const void* pf2, int64_t pf2_bytes, const void* pf3, const void* pf4,
                              int64_t read_bytes) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  prefetch_l2(pf0, pf0_bytes, tid, nth);
  prefetch_l2(pf1, pf1_bytes, tid, nth);
  prefetch_l2(pf2, pf2_bytes, tid, nth);
  prefetch_l2(pf3, read_bytes, tid, nth);
  prefetch_l2(pf4, read_bytes, tid, nth);
}

__global__ void k_precompute(EngineDev E, int num_reads, int* counters, int ncounters, int64_t num_pairs) {
  // One warp per read.  With X_i = max(B_M(i), B_I(i)) and g_i = min(n, 1/(1-eps_i)):
  //   B_D(i) <= g_i X_{i+1},  X_i <= (1 + zeta_i g_i) X_{i+1},  X_m = 1
  // so  sum_i (B_M + B_I + B_D) <= prod_{i<m}(1 + zeta_i g_i) * (2 + sum_{i<m}(2 + g_i)).
  // The grid also resets the work counters and the per-pair status.
  {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = tid; i < ncounters; i += nth) counters[i] = 0;
    uint4* st4 = reinterpret_cast<uint4*>(E.status);
    for (int64_t i = tid; i < num_pairs / 16; i += nth) st4[i] = make_uint4(0, 0, 0, 0);
    for (int64_t i = (num_pairs / 16) * 16 + tid; i < num_pairs; i += nth) E.status[i] = 0;
  }
  if (*E.invalid) return;
  const int lane = threadIdx.x & 31;
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= num_reads) return;
  const int m = E.read_m[r];
  const int64_t o = E.roff[r];
  const double ncap = (double)E.read_ncap[r];
  const double* lut = E.lut;
  bool degen = false;
  double logx = 0.0, sg = 0.0;
  for (int i = lane; i < m; i += 32) {
    const double d = lut[E.iq[o + i]], z = lut[E.dq[o + i]], e = lut[E.gq[o + i]];
    degen |= (d + z >= 1.0);
    if (i < m - 1) {
      const double g = (e >= 1.0) ? ncap : fmin(ncap, 1.0 / (1.0 - e));
      logx += log1p(z * g);
      sg += 2.0 + g;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    logx += __shfl_xor_sync(0xffffffffu, logx, off);
    sg += __shfl_xor_sync(0xffffffffu, sg, off);
  }
  degen = __any_sync(0xffffffffu, degen);
  if (lane == 0) {
    E.read_gsum[r] = (float)(exp(logx) * (2.0 + sg));
    E.read_flags[r] = degen ? 1 : 0;
  }
}

// ---------------------------------------------------------------------------------
// k_validate: input content checks of phmm_prepare on the device (model.py:14-18,47-52):
// base codes in 0..4, Phred qualities in 0..93.  16 B per thread-iteration, byte-wise
// SIMD compares; flag bit0 = bad base, bit1 = bad quality.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ unsigned over4(const uint4 v, unsigned lim) {
  return __vcmpgtu4(v.x, lim) | __vcmpgtu4(v.y, lim) | __vcmpgtu4(v.z, lim) | __vcmpgtu4(v.w, lim);
}
__global__ void k_validate(const uint8_t* rb, const uint8_t* bq, const uint8_t* iq, const uint8_t* dq,
                           const uint8_t* gq, int64_t RL, const uint8_t* hb, int64_t HL, int* flag) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  unsigned badb = 0, badq = 0;
  const int64_t RV = RL / 16, HV = HL / 16;
  for (int64_t v = tid; v < RV; v += nth) {
    badb |= over4(reinterpret_cast<const uint4*>(rb)[v], 0x04040404u);
    badq |= over4(reinterpret_cast<const uint4*>(bq)[v], 0x5d5d5d5du) |
            over4(reinterpret_cast<const uint4*>(iq)[v], 0x5d5d5d5du) |
            over4(reinterpret_cast<const uint4*>(dq)[v], 0x5d5d5d5du) |
            over4(reinterpret_cast<const uint4*>(gq)[v], 0x5d5d5d5du);
  }
  for (int64_t v = tid; v < HV; v += nth) badb |= over4(reinterpret_cast<const uint4*>(hb)[v], 0x04040404u);
  for (int64_t i = RV * 16 + tid; i < RL; i += nth) {
    badb |= rb[i] > 4;
    badq |= (bq[i] > 93) | (iq[i] > 93) | (dq[i] > 93) | (gq[i] > 93);
  }
  for (int64_t i = HV * 16 + tid; i < HL; i += nth) badb |= hb[i] > 4;
  if (badb || badq) atomicOr(flag, (badb ? 1 : 0) | (badq ? 2 : 0));
}


// Post-pass list kernels: one launch covers the four sub-warp widths P = 4, 8, 16, 32
// (slot lists filled by the host and by the fast kernels); empty lists cost nothing.
__device__ __forceinline__ bool post_lists_empty(const int* counts) {
  return counts[0] == 0 && counts[1] == 0 && counts[2] == 0 && counts[3] == 0;
}
template <typename T>
__global__ void __launch_bounds__(128)
k_exact_all(const EngineDev E, int* __restrict__ counters, T* __restrict__ colbuf, int col_rows) {
  constexpr bool kIsF32 = sizeof(T) == 4;
  if (*E.invalid || post_lists_empty(kIsF32 ? E.ex32_count : E.ex64_count)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* s_lut = reinterpret_cast<double*>(smem_raw);
  for (int i = threadIdx.x; i < 94; i += blockDim.x) s_lut[i] = E.lut[i];
  __syncthreads();
  exact_list<T, 4, kExactK>(E, 0, counters + 0, colbuf, col_rows);
  exact_list<T, 8, kExactK>(E, 1, counters + 1, colbuf, col_rows);
  exact_list<T, 16, kExactK>(E, 2, counters + 2, colbuf, col_rows);
  exact_list<T, 32, kExactK>(E, 3, counters + 3, colbuf, col_rows);
}
__global__ void __launch_bounds__(128)
k_fast64_all(const EngineDev E, int* __restrict__ counters, double* __restrict__ colbuf, int col_rows) {
  if (*E.invalid || post_lists_empty(E.fx64_count)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* s_lut = reinterpret_cast<double*>(smem_raw);
  for (int i = threadIdx.x; i < 94; i += blockDim.x) s_lut[i] = E.lut[i];
  __syncthreads();
  fast64_list<4, kExactK>(E, 0, counters + 0, colbuf, col_rows);
  fast64_list<8, kExactK>(E, 1, counters + 1, colbuf, col_rows);
  fast64_list<16, kExactK>(E, 2, counters + 2, colbuf, col_rows);
  fast64_list<32, kExactK>(E, 3, counters + 3, colbuf, col_rows);
}


// ---------------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------------
size_t exact_smem(int slot, size_t tsize) {
  const int P = 4 << slot;
  return 96 * sizeof(double) + (size_t)(kThreads / 32) * (32 / P) * 5 * kExactK * P * tsize;
}

cudaError_t aux_set_attributes() {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute((const void*)k_exact_all<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)exact_smem(0, 4))) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute((const void*)k_exact_all<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)exact_smem(0, 8))) != cudaSuccess) return e;
  return cudaFuncSetAttribute((const void*)k_fast64_all, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)exact_smem(0, 8));
}

void launch_l2_prefetch(int grid, cudaStream_t st, const void* pf0, int64_t pf0_bytes, const void* pf1,
                        int64_t pf1_bytes, const void* pf2, int64_t pf2_bytes, const void* pf3, const void* pf4,
                        int64_t read_bytes) {
  k_l2_prefetch<<<grid, 256, 0, st>>>(pf0, pf0_bytes, pf1, pf1_bytes, pf2, pf2_bytes, pf3, pf4, read_bytes);
}

void launch_precompute(int64_t num_reads, cudaStream_t st, const EngineDev& E, int* counters, int ncounters,
                       int64_t num_pairs) {
  const int threads = 128;
  const int64_t blocks = std::max<int64_t>(1, (num_reads * 32 + threads - 1) / threads);
  k_precompute<<<(unsigned)blocks, threads, 0, st>>>(E, (int)num_reads, counters, ncounters, num_pairs);
}

void launch_validate(int grid, cudaStream_t st, const uint8_t* rb, const uint8_t* bq, const uint8_t* iq,
                     const uint8_t* dq, const uint8_t* gq, int64_t RL, const uint8_t* hb, int64_t HL, int* flag) {
  k_validate<<<grid, 256, 0, st>>>(rb, bq, iq, dq, gq, RL, hb, HL, flag);
}

void launch_exact_all_f32(int grid, cudaStream_t st, const EngineDev& E, int* counters, float* col, int col_rows) {
  k_exact_all<float><<<grid, kThreads, exact_smem(0, 4), st>>>(E, counters, col, col_rows);
}
void launch_exact_all_f64(int grid, cudaStream_t st, const EngineDev& E, int* counters, double* col, int col_rows) {
  k_exact_all<double><<<grid, kThreads, exact_smem(0, 8), st>>>(E, counters, col, col_rows);
}
void launch_fast64_all(int grid, cudaStream_t st, const EngineDev& E, int* counters, double* col, int col_rows) {
  k_fast64_all<<<grid, kThreads, exact_smem(0, 8), st>>>(E, counters, col, col_rows);
}

}  // namespace phmm
