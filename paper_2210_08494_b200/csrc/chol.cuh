// Cholesky factorisation and triangular inverse of the c x c Gram matrix G = R^T R,
// the small dense core of CholeskyQR2 (the orthonormalisation of the residual
// R = (I - U U^T) M, Alg 3 line 2 "QR_decomp(A_perp)"; footnote :451
// allows any orthonormal decomposition).  One CTA per factor.
//
// Storage: packed row-major lower triangle, idx(i,k) = i(i+1)/2 + k, in shared memory
// when c <= CHOL_SMEM_MAX (c(c+1)/2 floats <= 131.6 KB), else in a global scratch.
// Outputs: L (c x c col-major, zeros above the diagonal) and Linv = L^{-1} (same layout).
// A pivot <= tol * max_i G_ii (rank-deficient residual) is dropped: the column of L
// and the row of L^{-1} are set to zero, and ST_CHOL_DROP is OR-ed into the status.
#pragma once
#include "common.cuh"

namespace bkfac {

constexpr int CHOL_SMEM_MAX = 256;

struct CholProb {
  const float* G; int ldg;
  float* L; float* Linv;   // c x c col-major, ld = c
  float* scratch;          // packed c(c+1)/2 floats (global path only)
  int* status;
  int c;
};
constexpr int CHOL_MAXP = 100;
struct CholBatch { int nprob; CholProb p[CHOL_MAXP]; };

BKFAC_DEV long pidx(int i, int k) { return (long)i * (i + 1) / 2 + k; }

template <bool SMEM>
__global__ void __launch_bounds__(1024) chol_inv_kernel(const __grid_constant__ CholBatch b) {
  const CholProb& p = b.p[blockIdx.x];
  const int c = p.c;
  extern __shared__ __align__(16) float csm[];
  float* lj = csm;                                   // c floats: current column of L
  float* red = lj + c;                               // 32 floats
  float* P = SMEM ? (red + 32) : p.scratch;          // packed lower
  const int tid = threadIdx.x, nt = blockDim.x;
  const int tx = tid & 31, ty = tid >> 5;

  // load lower triangle of G, track max diagonal
  float dmax = 0.f;
  for (int i = ty; i < c; i += 32)
    for (int k = tx; k <= i; k += 32) {
      const float g = p.G[i + (long)k * p.ldg];
      P[pidx(i, k)] = g;
      if (k == i) dmax = fmaxf(dmax, g);
    }
  // block max via sum of squares trick is wrong; use warp max + smem
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dmax = fmaxf(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  if (tx == 0) red[ty] = dmax;
  __syncthreads();
  if (tid == 0) {
    float m = 0.f;
    for (int w = 0; w < (nt + 31) / 32; ++w) m = fmaxf(m, red[w]);
    red[0] = m;
  }
  __syncthreads();
  const float tol = 8.0f * (float)c * 1.1920929e-7f * red[0];
  __syncthreads();
  int dropped = 0;

  // right-looking Cholesky
  for (int j = 0; j < c; ++j) {
    const float piv = P[pidx(j, j)];
    const bool drop = !(piv > tol);
    const float ljj = drop ? 0.f : sqrtf(piv);
    const float inv = drop ? 0.f : 1.f / ljj;
    dropped |= drop;
    for (int i = j + tid; i < c; i += nt) {
      const float v = (i == j) ? ljj : P[pidx(i, j)] * inv;
      P[pidx(i, j)] = v;
      lj[i] = v;
    }
    __syncthreads();
    for (int i = j + 1 + ty; i < c; i += 32) {
      const float li = lj[i];
      for (int k = j + 1 + tx; k <= i; k += 32) P[pidx(i, k)] -= li * lj[k];
    }
    __syncthreads();
  }
  // write L (col-major, zeros above)
  for (int k = ty; k < c; k += 32)
    for (int i = tx; i < c; i += 32) p.L[i + (long)k * c] = (i >= k) ? P[pidx(i, k)] : 0.f;
  __syncthreads();

  // L^{-1} by right-looking forward substitution on packed accumulator (reuse P):
  // acc <- I; for i: X(i,:) = acc(i,:) / L(i,i); acc(i',k) -= L(i',i) X(i,k), i' > i, k <= i.
  for (int i = ty; i < c; i += 32)
    for (int k = tx; k <= i; k += 32) P[pidx(i, k)] = (i == k) ? 1.f : 0.f;
  __syncthreads();
  for (int i = 0; i < c; ++i) {
    const float lii = p.L[i + (long)i * c];
    const float inv = (lii > 0.f) ? 1.f / lii : 0.f;
    for (int k = tid; k <= i; k += nt) P[pidx(i, k)] *= inv;
    // column i of L below the diagonal
    for (int ip = i + 1 + tid; ip < c; ip += nt) lj[ip] = p.L[ip + (long)i * c];
    __syncthreads();
    for (int ip = i + 1 + ty; ip < c; ip += 32) {
      const float l = lj[ip];
      if (l != 0.f)
        for (int k = tx; k <= i; k += 32) P[pidx(ip, k)] -= l * P[pidx(i, k)];
    }
    __syncthreads();
  }
  for (int k = ty; k < c; k += 32)
    for (int i = tx; i < c; i += 32) p.Linv[i + (long)k * c] = (i >= k) ? P[pidx(i, k)] : 0.f;

  if (dropped && tid == 0 && p.status) atomicOr(p.status, ST_CHOL_DROP);
}

}  // namespace bkfac
