// phmm_registry.h — kernel tables and launchers shared by the translation units of
// libphmm.so.  Each k_stream_<mode>.cu instantiates one mode's tilings and exposes them
// as a StreamKernel table (launch function + attributes); phmm_aux.cu holds the small
// kernels; phmm_engine.cu (the host engine) only sees this header.
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdint>

#include "phmm_kernels.cuh"

namespace phmm {

constexpr int kThreads = 128;

// One k_stream<MODE, P, K, STRIPES> instantiation.
struct StreamKernel {
  int P, K, occ;
  size_t smem;
  const void* fn;
  void (*launch)(dim3, size_t, cudaStream_t, const EngineDev&, const StreamUnit*, const StreamHap*, int,
                 const int*, int*, void*, int);
};

template <int MODE, int P, int K, bool STRIPES>
void launch_stream_t(dim3 g, size_t smem, cudaStream_t s, const EngineDev& E, const StreamUnit* u,
                     const StreamHap* h, int nu, const int* nud, int* ctr, void* col, int col_rows) {
  k_stream<MODE, P, K, STRIPES><<<g, kThreads, smem, s>>>(E, u, h, nu, nud, ctr, col, col_rows);
}
template <int MODE, int P, int K, bool STRIPES = false>
StreamKernel SK() {
  const size_t elem = ModeOf<MODE>::F64 ? sizeof(double) : sizeof(float);   // 5*Kp*P entries per slot
  constexpr int Kp = EChunk<ModeOf<MODE>::F64, K>::chunks * EChunk<ModeOf<MODE>::F64, K>::width;   // K, padded
  // striped instantiations add the boundary-column ring: per sub-warp slot 3 x kColRing
  // two-lane values
  return StreamKernel{P, K, STRIPES ? 2 : StreamOcc<MODE, K>::value,
                      96 * sizeof(double) + (size_t)4 * (32 / P) * 5 * Kp * P * elem + kStreamCodeBytesPerCta +
                          (STRIPES ? (size_t)4 * (32 / P) * 3 * kColRing * 2 * elem : 0),
                      (const void*)k_stream<MODE, P, K, STRIPES>, launch_stream_t<MODE, P, K, STRIPES>};
}

// tiling tables per mode (k_stream_<mode>.cu); kFast32's first 13 entries are the
// geometry table PHMM_FAST_GEOM indexes
constexpr int kNumStreamFast32 = 23;
const StreamKernel* stream_table_fast32();
const StreamKernel* stream_table_fast64();     // kNumR64Geoms, indexed by r64_geom_for(m)
const StreamKernel* stream_table_exact32();    // kNumRX32Geoms, indexed by rx32_geom_for(m)
const StreamKernel* stream_table_exact64();    // kNumR64Geoms
// striped instantiation per mode (reads longer than the mode's widest tiling)
const StreamKernel& striped_fast32();
const StreamKernel& striped_fast64();
const StreamKernel& striped_exact32();
const StreamKernel& striped_exact64();

// phmm_aux.cu
size_t exact_smem(int slot, size_t tsize);
cudaError_t aux_set_attributes();
void launch_l2_prefetch(int grid, cudaStream_t st, const void* pf0, int64_t pf0_bytes, const void* pf1,
                        int64_t pf1_bytes, const void* pf2, int64_t pf2_bytes, const void* pf3, const void* pf4,
                        int64_t read_bytes);
void launch_precompute(int64_t num_reads, cudaStream_t st, const EngineDev& E, int* counters, int ncounters,
                       int64_t num_pairs);
void launch_validate(int grid, cudaStream_t st, const uint8_t* rb, const uint8_t* bq, const uint8_t* iq,
                     const uint8_t* dq, const uint8_t* gq, int64_t RL, const uint8_t* hb, int64_t HL, int* flag);
void launch_exact_all_f32(int grid, cudaStream_t st, const EngineDev& E, int* counters, float* col, int col_rows);
void launch_exact_all_f64(int grid, cudaStream_t st, const EngineDev& E, int* counters, double* col, int col_rows);
// phmm_matrices.cu
void launch_matrices(cudaStream_t st, const int8_t* rb, const uint8_t* bq, const uint8_t* iq, const uint8_t* dq,
                     const uint8_t* gq, int m, const int8_t* hb, int n, double boundary, const double* lut,
                     double* M, double* I, double* D);
void launch_fast64_all(int grid, cudaStream_t st, const EngineDev& E, int* counters, double* col, int col_rows);

}  // namespace phmm
