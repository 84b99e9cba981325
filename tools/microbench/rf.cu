// Register-file / operand-pattern throughput of packed FP32 on B200 (sm_100a):
// does FFMA2 with a scalar-broadcast operand + two distinct register pairs run at
// 1 warp-instruction / 2 cycles / SMSP, or is it limited by register-bank reads?
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned smid() { unsigned r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }
struct Rec { long long t0, t1; unsigned sm; };
constexpr int IT = 1024;

#define KERNEL(NAME, BODY, NINST)                                                          \
__global__ void NAME(float* out, float a, Rec* rec) {                                     \
  float2 x[8], y[8]; float s[8];                                                          \
  for (int i = 0; i < 8; i++) { x[i] = make_float2(threadIdx.x * 1e-3f + i, i); y[i] = make_float2(a + i, a - i); s[i] = a + i * 1e-6f + threadIdx.x * 1e-9f; } \
  __syncthreads(); long long t0 = clock64();                                              \
  _Pragma("unroll 2") for (int it = 0; it < IT; it++) { BODY }                            \
  __syncthreads(); long long t1 = clock64();                                              \
  float acc = 0; for (int i = 0; i < 8; i++) acc += x[i].x + x[i].y + y[i].x + s[i];      \
  if (acc == 1234.5f) out[0] = acc;                                                       \
  if (threadIdx.x == 0) rec[blockIdx.x] = {t0, t1, smid()};                               \
}

// A: distinct scalar per chain, 2 distinct pairs
KERNEL(k_ffma2_distinct, _Pragma("unroll") for (int i = 0; i < 8; i++) x[i] = __ffma2_rn(make_float2(s[i], s[i]), x[i], y[i]);, 8)
// B: one shared scalar (reuse-cacheable)
KERNEL(k_ffma2_shared, _Pragma("unroll") for (int i = 0; i < 8; i++) x[i] = __ffma2_rn(make_float2(s[0], s[0]), x[i], y[i]);, 8)
// C: FMUL2 distinct scalar
KERNEL(k_fmul2_distinct, _Pragma("unroll") for (int i = 0; i < 8; i++) x[i] = __fmul2_rn(make_float2(s[i], s[i]), x[i]);, 8)
// D: FADD2 pair + pair
KERNEL(k_fadd2, _Pragma("unroll") for (int i = 0; i < 8; i++) x[i] = __fadd2_rn(x[i], y[i]);, 8)
// E: scalar FFMA, 3 distinct registers
KERNEL(k_ffma_distinct, _Pragma("unroll") for (int i = 0; i < 8; i++) { x[i].x = fmaf(s[i], x[i].x, y[i].x); x[i].y = fmaf(s[i], x[i].y, y[i].y);}, 16)
// F: scalar FMUL distinct
KERNEL(k_fmul_distinct, _Pragma("unroll") for (int i = 0; i < 8; i++) { x[i].x = s[i] * x[i].x; x[i].y = s[i] * x[i].y;}, 16)

typedef void (*kfn)(float*, float, Rec*);
void run(kfn f, const char* name, double ninst) {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int T = 256, B = nsm * 4;
  float* out; Rec* rec; cudaMalloc(&out, 4); cudaMalloc(&rec, B * sizeof(Rec));
  f<<<B, T>>>(out, 1.0001f, rec); cudaDeviceSynchronize();
  f<<<B, T>>>(out, 1.0001f, rec); cudaDeviceSynchronize();
  std::vector<Rec> h(B); cudaMemcpy(h.data(), rec, B * sizeof(Rec), cudaMemcpyDeviceToHost);
  std::vector<long long> lo(nsm, -1), hi(nsm, -1); std::vector<int> cnt(nsm, 0);
  for (auto& r : h) { if (r.sm >= (unsigned)nsm) continue; if (lo[r.sm] < 0 || r.t0 < lo[r.sm]) lo[r.sm] = r.t0; if (r.t1 > hi[r.sm]) hi[r.sm] = r.t1; cnt[r.sm]++; }
  std::vector<double> rate;
  for (int s = 0; s < nsm; s++) if (cnt[s]) rate.push_back((double)cnt[s] * T * ninst * IT / (hi[s] - lo[s]));
  std::sort(rate.begin(), rate.end());
  printf("%-18s %7.2f thread-instr/clk/SM  (= %.2f warp-instr/clk/SMSP)\n", name, rate[rate.size() / 2], rate[rate.size() / 2] / 128.0);
  cudaFree(out); cudaFree(rec);
}
int main() {
  run(k_ffma2_distinct, "FFMA2 s_i,pair,pair", 8);
  run(k_ffma2_shared, "FFMA2 s,pair,pair", 8);
  run(k_fmul2_distinct, "FMUL2 s_i,pair", 8);
  run(k_fadd2, "FADD2 pair,pair", 8);
  run(k_ffma_distinct, "FFMA s_i,a,b", 16);
  run(k_fmul_distinct, "FMUL s_i,a", 16);
  return 0;
}
