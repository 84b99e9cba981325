// phmm_matrices.cu — k_matrices: the complete (m+1) x (n+1) FP64 DP matrices of ONE pair
// (the reference's debugging oracle forward_matrices / _full_kernel, reference.py:36-75,
// 150-156), bit-identical to it:
//   M(i,j) = lam_ij * (alpha_i * M(i-1,j-1) + beta_i * (I(i-1,j-1) + D(i-1,j-1)))
//   I(i,j) = delta_i * M(i-1,j) + epsilon_i * I(i-1,j)
//   D(i,j) = zeta_i  * M(i,j-1) + epsilon_i * D(i,j-1)
// each product and sum rounded separately (__dmul_rn / __dadd_rn: no FMA, like numba's
// code), every store flushed below 2^-970 (prob.py:39), row 0: M = I = 0, D = 2^s / n
// (including j = 0), column 0 zero for i >= 1.
//
// One CTA sweeps the anti-diagonals d = i + j; thread t owns rows t+1, t+1+T, ...; cells
// of one diagonal are independent and read only diagonals d-1 and d-2 from the output
// matrices (global memory, L2/L1-resident at these sizes), with a CTA barrier per
// diagonal.  A debugging path: ~(m + n) barriers, sized for pairs up to a few thousand.
#include "phmm_registry.h"

namespace phmm {

__global__ void __launch_bounds__(1024) k_matrices(const int8_t* __restrict__ rb, const uint8_t* __restrict__ bq,
                                                   const uint8_t* __restrict__ iq, const uint8_t* __restrict__ dq,
                                                   const uint8_t* __restrict__ gq, int m,
                                                   const int8_t* __restrict__ hb, int n, double boundary,
                                                   const double* __restrict__ lut, double* __restrict__ M,
                                                   double* __restrict__ I, double* __restrict__ D) {
  const int T = blockDim.x;
  const size_t ld = (size_t)n + 1;
  const double zero = boundary - boundary;
  const double flush = 0x1p-970;
  for (int j = threadIdx.x; j <= n; j += T) {
    M[j] = zero; I[j] = zero; D[j] = boundary;
  }
  for (int i = 1 + threadIdx.x; i <= m; i += T) {
    M[i * ld] = zero; I[i * ld] = zero; D[i * ld] = zero;
  }
  __syncthreads();
  for (int d = 2; d <= m + n; ++d) {
    for (int i = 1 + threadIdx.x; i <= m; i += T) {
      const int j = d - i;
      if (j < 1 || j > n) continue;
      const double q = lut[bq[i - 1]];
      const double delta = lut[iq[i - 1]], zeta = lut[dq[i - 1]], eps = lut[gq[i - 1]];
      const double alpha = __dsub_rn(__dsub_rn(1.0, delta), zeta);
      const double beta = __dsub_rn(1.0, eps);
      const int r = rb[i - 1], h = hb[j - 1];
      const double lam = (r == h || r == 4 || h == 4) ? __dsub_rn(1.0, q) : __ddiv_rn(q, 3.0);
      const size_t c = (size_t)i * ld + j, up = c - ld, left = c - 1, diag = up - 1;
      const double mv = __dmul_rn(lam, __dadd_rn(__dmul_rn(alpha, M[diag]), __dmul_rn(beta, __dadd_rn(I[diag], D[diag]))));
      const double iv = __dadd_rn(__dmul_rn(delta, M[up]), __dmul_rn(eps, I[up]));
      const double dv = __dadd_rn(__dmul_rn(zeta, M[left]), __dmul_rn(eps, D[left]));
      M[c] = mv >= flush ? mv : zero;
      I[c] = iv >= flush ? iv : zero;
      D[c] = dv >= flush ? dv : zero;
    }
    __syncthreads();
  }
}

void launch_matrices(cudaStream_t st, const int8_t* rb, const uint8_t* bq, const uint8_t* iq, const uint8_t* dq,
                     const uint8_t* gq, int m, const int8_t* hb, int n, double boundary, const double* lut,
                     double* M, double* I, double* D) {
  const int threads = m >= 1024 ? 1024 : ((m + 31) / 32) * 32;
  k_matrices<<<1, threads, 0, st>>>(rb, bq, iq, dq, gq, m, hb, n, boundary, lut, M, I, D);
}

}  // namespace phmm
