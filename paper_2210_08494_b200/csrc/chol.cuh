// Cholesky factorisation and triangular inverse of the c x c Gram matrix G = R^T R,
// the small dense core of CholeskyQR2 (the orthonormalisation of the residual
// R = (I - U U^T) M, Alg 3 line 2 "QR_decomp(A_perp)"; footnote :451
// allows any orthonormal decomposition).  One CTA (32 warps) per factor.
//
// Storage: packed row-major lower triangle, idx(i,k) = i(i+1)/2 + k, in shared memory
// when c <= CHOL_SMEM_MAX (c(c+1)/2 floats <= 131.6 KB), else in a global scratch.
//   phase 1  right-looking Cholesky, one column per step (2 barriers per column);
//   phase 2  L^{-1} by forward substitution, one column of L^{-1} per warp, the
//            running column kept in a per-warp shared vector (no block barriers).
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
  float shift;             // shifted CholeskyQR: G_ii += shift * trace(G) (0 = plain)
};
constexpr int CHOL_MAXP = 100;
struct CholBatch { int nprob; CholProb p[CHOL_MAXP]; };

BKFAC_DEV int pidx(int i, int k) { return i * (i + 1) / 2 + k; }

// smem layout: [lj: c][red: 32][xw: 32 warps * c][P (SMEM path): c(c+1)/2]
template <bool SMEM>
__global__ void __launch_bounds__(1024) chol_inv_kernel(const __grid_constant__ CholBatch b) {
  const CholProb& p = b.p[blockIdx.x];
  const int c = p.c;
  extern __shared__ __align__(16) float csm[];
  float* lj = csm;
  float* red = lj + c;
  float* xw = red + 32;
  float* P = SMEM ? (xw + 32 * c) : p.scratch;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int tx = tid & 31, ty = tid >> 5;

  float dsum = 0.f, dmax = 0.f;
  for (int i = ty; i < c; i += 32)
    for (int k = tx; k <= i; k += 32) {
      const float g = p.G[i + (long)k * p.ldg];
      P[pidx(i, k)] = g;
      if (k == i) { dsum += g; dmax = fmaxf(dmax, g); }
    }
  const float trace = block_sum(dsum, red);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dmax = fmaxf(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  if (tx == 0) red[ty] = dmax;
  __syncthreads();
  float gmax = 0.f;
  for (int w = 0; w < (nt + 31) / 32; ++w) gmax = fmaxf(gmax, red[w]);
  // shifted first pass (sCQR, Fukaya et al. 2020): keeps the factorisation defined
  // for ill-conditioned inputs; R = Q R_Q stays exact, later passes restore Q^T Q = I.
  const float sh = (p.shift > 0.f) ? p.shift * trace : 0.f;
  __syncthreads();
  if (sh > 0.f)
    for (int i = tid; i < c; i += nt) P[pidx(i, i)] += sh;
  __syncthreads();
  // pivots at the rounding level of the largest diagonal entry = rank deficiency
  const float tol = 4.0f * 1.1920929e-7f * (gmax + sh);
  int dropped = 0;

  // ---- phase 1: right-looking Cholesky
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
      float* row = P + pidx(i, 0);
      for (int k = j + 1 + tx; k <= i; k += 32) row[k] -= li * lj[k];
    }
    __syncthreads();
  }
  for (int k = ty; k < c; k += 32)
    for (int i = tx; i < c; i += 32) p.L[i + (long)k * c] = (i >= k) ? P[pidx(i, k)] : 0.f;

  // ---- phase 2: columns of L^{-1}; warp ty owns columns ty, ty+32, ...
  float* x = xw + ty * c;
  for (int j = ty; j < c; j += 32) {
    const float ljj = P[pidx(j, j)];
    if (tx == 0) x[j] = (ljj > 0.f) ? 1.f / ljj : 0.f;
    __syncwarp();
    for (int i = j + 1; i < c; ++i) {
      const float* row = P + pidx(i, 0);
      float s = 0.f;
      for (int k = j + tx; k < i; k += 32) s = fmaf(row[k], x[k], s);
      s = warp_sum(s);
      const float lii = row[i];
      if (tx == 0) x[i] = (lii > 0.f) ? -s / lii : 0.f;
      __syncwarp();
    }
    for (int i = tx; i < c; i += 32) p.Linv[i + (long)j * c] = (i >= j) ? x[i] : 0.f;
    __syncwarp();
  }
  if (dropped && tid == 0 && p.status) atomicOr(p.status, ST_CHOL_DROP);
}

inline size_t chol_smem_bytes(int cmax, bool smem_path) {
  size_t f = (size_t)cmax + 32 + 32 * (size_t)cmax;
  if (smem_path) f += (size_t)cmax * (cmax + 1) / 2;
  return f * sizeof(float);
}

}  // namespace bkfac
