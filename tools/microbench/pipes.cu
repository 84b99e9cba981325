// Pipe-throughput microbenchmarks for the Pair-HMM kernel design (B200, sm_100a).
// Measures per-SM per-clock throughput of FFMA, FFMA2 (with scalar-broadcast
// operand), FMUL2, FADD2, DFMA, LDS.128 and SHFL using in-kernel clock64()
// spans per SM, so the result is independent of the (DVFS) SM clock.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ unsigned smid() { unsigned r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }

struct Rec { long long t0, t1; unsigned sm; };

constexpr int ITERS = 2048;

// scalar FFMA, 8 independent chains, shared multiplier (reuse-friendly)
__global__ void k_ffma(float* out, float a, float b, Rec* rec) {
  float x[8];
  for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 0.001f + i;
  __syncthreads();
  long long t0 = clock64();
  #pragma unroll 4
  for (int it = 0; it < ITERS; it++) {
    #pragma unroll
    for (int i = 0; i < 8; i++) x[i] = fmaf(x[i], a, b);
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; i++) s += x[i];
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0) rec[blockIdx.x] = {t0, t1, smid()};
}

// scalar FFMA, 3 distinct per-chain register operands (bank-conflict prone)
__global__ void k_ffma3(float* out, float a, float b, Rec* rec) {
  float x[8], y[8], z[8];
  for (int i = 0; i < 8; i++) { x[i] = threadIdx.x * 0.001f + i; y[i] = a + i * 1e-3f; z[i] = b - i * 1e-3f; }
  __syncthreads();
  long long t0 = clock64();
  #pragma unroll 4
  for (int it = 0; it < ITERS; it++) {
    #pragma unroll
    for (int i = 0; i < 8; i++) x[i] = fmaf(x[i], y[i], z[i]);
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; i++) s += x[i];
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0) rec[blockIdx.x] = {t0, t1, smid()};
}

// packed FFMA2 with scalar broadcast multiplier + packed addend
__global__ void k_ffma2(float* out, float a, float b, Rec* rec) {
  float2 x[8], z[8];
  for (int i = 0; i < 8; i++) { x[i] = make_float2(threadIdx.x * 0.001f + i, i); z[i] = make_float2(b, b + i); }
  float ar = a + threadIdx.x * 1e-9f;
  __syncthreads();
  long long t0 = clock64();
  #pragma unroll 4
  for (int it = 0; it < ITERS; it++) {
    #pragma unroll
    for (int i = 0; i < 8; i++) x[i] = __ffma2_rn(make_float2(ar, ar), x[i], z[i]);
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; i++) s += x[i].x + x[i].y;
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0) rec[blockIdx.x] = {t0, t1, smid()};
}

// packed FFMA2, all three operands packed registers
__global__ void k_ffma2p(float* out, float a, float b, Rec* rec) {
  float2 x[8], y[8], z[8];
  for (int i = 0; i < 8; i++) { x[i] = make_float2(threadIdx.x * 0.001f + i, i); y[i] = make_float2(a, a + i * 1e-3f); z[i] = make_float2(b, b + i); }
  __syncthreads();
  long long t0 = clock64();
  #pragma unroll 4
  for (int it = 0; it < ITERS; it++) {
    #pragma unroll
    for (int i = 0; i < 8; i++) x[i] = __ffma2_rn(y[i], x[i], z[i]);
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; i++) s += x[i].x + x[i].y;
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0) rec[blockIdx.x] = {t0, t1, smid()};
}

__global__ void k_fmul2(float* out, float a, float b, Rec* rec) {
  float2 x[8], y[8];
  for (int i = 0; i < 8; i++) { x[i] = make_float2(threadIdx.x * 0.001f + i, i); y[i] = make_float2(a, a + i * 1e-7f); }
  __syncthreads();
  long long t0 = clock64();
  #pragma unroll 4
  for (int it = 0; it < ITERS; it++) {
    #pragma unroll
    for (int i = 0; i < 8; i++) x[i] = __fmul2_rn(x[i], y[i]);
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; i++) s += x[i].x + x[i].y;
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0) rec[blockIdx.x] = {t0, t1, smid()};
}

__global__ void k_fadd2(float* out, float a, float b, Rec* rec) {
  float2 x[8], y[8];
  for (int i = 0; i < 8; i++) { x[i] = make_float2(threadIdx.x * 0.001f + i, i); y[i] = make_float2(a, a + i * 1e-7f); }
  __syncthreads();
  long long t0 = clock64();
  #pragma unroll 4
  for (int it = 0; it < ITERS; it++) {
    #pragma unroll
    for (int i = 0; i < 8; i++) x[i] = __fadd2_rn(x[i], y[i]);
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; i++) s += x[i].x + x[i].y;
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0) rec[blockIdx.x] = {t0, t1, smid()};
}

// scalar FMUL + FADD mix (the exact kernel's op mix has no FMA)
__global__ void k_fmul(float* out, float a, float b, Rec* rec) {
  float x[8];
  for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 0.001f + i;
  __syncthreads();
  long long t0 = clock64();
  #pragma unroll 4
  for (int it = 0; it < ITERS; it++) {
    #pragma unroll
    for (int i = 0; i < 8; i++) x[i] = __fmul_rn(x[i], a);
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; i++) s += x[i];
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0) rec[blockIdx.x] = {t0, t1, smid()};
}

__global__ void k_dfma(float* out, float a, float b, Rec* rec) {
  double x[8];
  double ad = a, bd = b;
  for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 0.001 + i;
  __syncthreads();
  long long t0 = clock64();
  #pragma unroll 4
  for (int it = 0; it < ITERS / 4; it++) {
    #pragma unroll
    for (int i = 0; i < 8; i++) x[i] = fma(x[i], ad, bd);
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < 8; i++) s += x[i];
  if (s == 12345.0) out[0] = (float)s;
  if (threadIdx.x == 0) rec[blockIdx.x] = {t0, t1, smid()};
}


// DFMA with 3 distinct per-chain 64-bit operands (6 register reads per instruction)
__global__ void k_dfma3(float* out, float a, float b, Rec* rec) {
  double x[8], y[8], z[8];
  for (int i = 0; i < 8; i++) { x[i] = threadIdx.x * 0.001 + i; y[i] = a + i * 1e-3; z[i] = b - i * 1e-3; }
  __syncthreads();
  long long t0 = clock64();
  #pragma unroll 4
  for (int it = 0; it < ITERS / 4; it++) {
    #pragma unroll
    for (int i = 0; i < 8; i++) x[i] = fma(x[i], y[i], z[i]);
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < 8; i++) s += x[i];
  if (s == 12345.0) out[0] = (float)s;
  if (threadIdx.x == 0) rec[blockIdx.x] = {t0, t1, smid()};
}

// the k_stream FP64 pattern: two lanes share a per-position coefficient (x = c*x + y)
__global__ void k_dfma2l(float* out, float a, float b, Rec* rec) {
  double x[8], y[8], c[4];
  for (int i = 0; i < 8; i++) { x[i] = threadIdx.x * 0.001 + i; y[i] = b - i * 1e-3; }
  for (int i = 0; i < 4; i++) c[i] = a + i * 1e-3;
  __syncthreads();
  long long t0 = clock64();
  #pragma unroll 4
  for (int it = 0; it < ITERS / 4; it++) {
    #pragma unroll
    for (int i = 0; i < 8; i++) x[i] = fma(c[i >> 1], x[i], y[i]);
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < 8; i++) s += x[i];
  if (s == 12345.0) out[0] = (float)s;
  if (threadIdx.x == 0) rec[blockIdx.x] = {t0, t1, smid()};
}

__global__ void k_lds128(float* out, float a, float b, Rec* rec) {
  __shared__ float4 tab[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) tab[i] = make_float4(i, a, b, i + 1);
  __syncthreads();
  float4 acc = make_float4(0, 0, 0, 0);
  int idx = threadIdx.x;
  long long t0 = clock64();
  #pragma unroll 8
  for (int it = 0; it < ITERS; it++) {
    float4 v = tab[(idx + it) & 1023];
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  __syncthreads();
  long long t1 = clock64();
  if (acc.x + acc.y + acc.z + acc.w == 12345.f) out[0] = acc.x;
  if (threadIdx.x == 0) rec[blockIdx.x] = {t0, t1, smid()};
}

__global__ void k_shfl(float* out, float a, float b, Rec* rec) {
  float x[4];
  for (int i = 0; i < 4; i++) x[i] = threadIdx.x + i * a;
  __syncthreads();
  long long t0 = clock64();
  #pragma unroll 4
  for (int it = 0; it < ITERS; it++) {
    #pragma unroll
    for (int i = 0; i < 4; i++) x[i] = __shfl_up_sync(0xffffffffu, x[i], 1, 8);
  }
  __syncthreads();
  long long t1 = clock64();
  if (x[0] + x[1] + x[2] + x[3] == 12345.f) out[0] = x[0];
  if (threadIdx.x == 0) rec[blockIdx.x] = {t0, t1, smid()};
}

typedef void (*kfn)(float*, float, float, Rec*);

// returns thread-instructions (of the measured op) per SM per clock
static double measure(kfn f, const char* name, double ops_per_thread_per_iter, int iters, int threads, int blocks_per_sm,
                      int nsm) {
  int blocks = nsm * blocks_per_sm;
  float* out; Rec* rec;
  CK(cudaMalloc(&out, 4)); CK(cudaMalloc(&rec, blocks * sizeof(Rec)));
  for (int w = 0; w < 2; w++) f<<<blocks, threads>>>(out, 1.0000001f, 1e-7f, rec);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  f<<<blocks, threads>>>(out, 1.0000001f, 1e-7f, rec);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  std::vector<Rec> h(blocks);
  CK(cudaMemcpy(h.data(), rec, blocks * sizeof(Rec), cudaMemcpyDeviceToHost));
  std::vector<long long> lo(nsm, -1), hi(nsm, -1); std::vector<int> cnt(nsm, 0);
  for (auto& r : h) {
    if (r.sm >= (unsigned)nsm) continue;
    if (lo[r.sm] < 0 || r.t0 < lo[r.sm]) lo[r.sm] = r.t0;
    if (hi[r.sm] < 0 || r.t1 > hi[r.sm]) hi[r.sm] = r.t1;
    cnt[r.sm]++;
  }
  std::vector<double> rate;
  for (int s = 0; s < nsm; s++) if (cnt[s] > 0) {
    double ops = (double)cnt[s] * threads * ops_per_thread_per_iter * iters;
    rate.push_back(ops / (double)(hi[s] - lo[s]));
  }
  std::sort(rate.begin(), rate.end());
  double med = rate[rate.size() / 2];
  double total_ops = (double)blocks * threads * ops_per_thread_per_iter * iters;
  double clk_ghz = total_ops / med / nsm / (ms * 1e-3) / 1e9;   // implied average SM clock
  printf("%-10s %8.2f thread-instr/clk/SM (median over %zu SMs)  time %.3f ms  implied clk %.3f GHz\n",
         name, med, rate.size(), ms, clk_ghz);
  cudaFree(out); cudaFree(rec);
  return med;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int nsm = prop.multiProcessorCount;
  printf("device %s  SMs %d  cc %d.%d  clock %d kHz\n", prop.name, nsm, prop.major, prop.minor, prop.clockRate);
  int T = 512, B = 2;
  measure(k_ffma, "FFMA", 8, ITERS, T, B, nsm);
  measure(k_ffma3, "FFMA-3reg", 8, ITERS, T, B, nsm);
  measure(k_fmul, "FMUL", 8, ITERS, T, B, nsm);
  measure(k_ffma2, "FFMA2-bc", 8, ITERS, T, B, nsm);
  measure(k_ffma2p, "FFMA2-3p", 8, ITERS, T, B, nsm);
  measure(k_fmul2, "FMUL2", 8, ITERS, T, B, nsm);
  measure(k_fadd2, "FADD2", 8, ITERS, T, B, nsm);
  measure(k_dfma, "DFMA", 8, ITERS / 4, T, B, nsm);
  measure(k_dfma3, "DFMA-3reg", 8, ITERS / 4, T, B, nsm);
  measure(k_dfma2l, "DFMA-2lane", 8, ITERS / 4, T, B, nsm);
  measure(k_lds128, "LDS.128", 1, ITERS, T, B, nsm);
  measure(k_shfl, "SHFL", 4, ITERS, T, B, nsm);
  return 0;
}
