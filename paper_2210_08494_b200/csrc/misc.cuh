// Small fused elementwise kernels of the hot path (epilogue-class work).
#pragma once
#include "common.cuh"

namespace bkfac {

// ---- generic batched "axpy-like" ops on col-major blocks -----------------------------
struct EwProb {
  float* Y; int ldy;          // destination block (rows x cols)
  const float* X; int ldx;    // source block
  const float* vec;           // optional per-column (or diagonal) vector
  int rows, cols;
  float a, b;
  int op;
};
enum : int {
  EW_ADD = 0,        // Y += a * X
  EW_SCALE_COLS = 1, // Y(:,j) = X(:,j) * vec[j]
  EW_ADD_DIAG = 2,   // Y(i,i) += a * vec[i], i < rows
  EW_COPY = 3,       // Y = X
  EW_SCALE_ROWSCOLS = 4, // Y(i,j) = X(i,j) * a * vec[i]... (unused)
  EW_ZERO_UPPER = 5, // Y(i,j) = 0 for i < j (X unused)
};
constexpr int EW_MAXP = 100;
struct EwBatch { int nprob; EwProb p[EW_MAXP]; };

__global__ void ew_kernel(const __grid_constant__ EwBatch b) {
  const EwProb& p = b.p[blockIdx.y];
  if (p.op == EW_ADD_DIAG) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p.rows; i += gridDim.x * blockDim.x)
      p.Y[i + (long)i * p.ldy] += p.a * p.vec[i];
    return;
  }
  // columns over blocks, rows over threads (coalesced, no index division)
  if (p.op == EW_ZERO_UPPER) {
    for (int j = blockIdx.x; j < p.cols; j += gridDim.x)
      for (int i = threadIdx.x; i < min(j, p.rows); i += blockDim.x) p.Y[i + (long)j * p.ldy] = 0.f;
    return;
  }
  for (int j = blockIdx.x; j < p.cols; j += gridDim.x) {
    float* yc = p.Y + (long)j * p.ldy;
    const float* xc = p.X + (long)j * p.ldx;
    const float sj = (p.op == EW_SCALE_COLS) ? p.vec[j] : 1.f;
    for (int i = threadIdx.x; i < p.rows; i += blockDim.x) {
      const float x = xc[i];
      switch (p.op) {
        case EW_ADD: yc[i] += p.a * x; break;
        case EW_SCALE_COLS: yc[i] = x * sj; break;
        case EW_COPY: yc[i] = x; break;
        default: break;
      }
    }
  }
}

// ---- inf/NaN guard for inputs that reach the tensor cores only as MMA operands (the MMA
// does not propagate NaN reliably): one pass, OR into the factor's status word.
struct NfProb { const float* X; int rows, cols, ld; int* status; };
constexpr int NF_MAXP = 100;
struct NfBatch { int nprob; NfProb p[NF_MAXP]; };
__global__ void nonfinite_kernel(const __grid_constant__ NfBatch b) {
  const NfProb& p = b.p[blockIdx.y];
  const long total = (long)p.rows * p.cols;
  int bad = 0;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x)
    bad |= !isfinite(p.X[(e % p.rows) + (e / p.rows) * (long)p.ld]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(p.status, ST_NONFINITE);
}

// ---- column gather / scatter by an index array (light correction, Algorithm 6) ------------
//   mode 0: dst(:, j) = src(:, idx[j])                      j < n
//   mode 1: dst(:, idx[j]) = src(:, j), ddst[idx[j]] = dsrc[j]
// An index outside [0, r) is skipped and reported (ST_BAD_INDEX).
struct ColIdxProb {
  const float* src; int lds; float* dst; int ldd; int rows;
  const int* idx; int n; int r; int mode;
  const float* dsrc; float* ddst; int* status;
};
struct ColIdxBatch { int nprob; ColIdxProb p[NF_MAXP]; };
__global__ void colidx_kernel(const __grid_constant__ ColIdxBatch b) {
  const ColIdxProb& p = b.p[blockIdx.y];
  const long total = (long)p.rows * p.n;
  int bad = 0;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    const int j = (int)(e / p.rows), i = (int)(e % p.rows);
    const int c = p.idx[j];
    if (c < 0 || c >= p.r) { bad = 1; continue; }
    if (p.mode == 0) {
      p.dst[i + (long)j * p.ldd] = p.src[i + (long)c * p.lds];
    } else {
      p.dst[i + (long)c * p.ldd] = p.src[i + (long)j * p.lds];
      if (i == 0 && p.ddst) p.ddst[c] = p.dsrc[j];
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0 && p.status) atomicOr(p.status, ST_BAD_INDEX);
}

// ---- preconditioner scalars (Alg 1 lines 16-17) ---------------------
// One CTA per layer.  For each side: effective lambda (relative mode :940, continuation
// :711) and s_i = (D_i + lambda)^{-1} - 1/lambda; then the coefficient of J in S,
// 1 / (lambda_G lambda_A).  Writes s_A, s_G and lam_out[0..4] = {lambda_A, lambda_G, coef,
// 1 / lambda_A, 1 / lambda_G}.
struct PrecScalProb {
  const float* D[2]; int r[2]; float lam[2]; float* s[2];   // [0] = A side, [1] = Gamma side
  int flags;
  float* lam_out;
};
constexpr int PS_MAXP = 200;
struct PrecScalBatch { int nprob; PrecScalProb p[PS_MAXP]; };

__global__ void prec_scalars_kernel(const __grid_constant__ PrecScalBatch b) {
  const PrecScalProb& p = b.p[blockIdx.x];
  __shared__ float s_min[2], s_max[2];
  if (threadIdx.x < 2) {
    const int q = threadIdx.x;
    float mn = 3.4e38f, mx = 0.f;
    for (int i = 0; i < p.r[q]; ++i) { mn = fminf(mn, p.D[q][i]); mx = fmaxf(mx, p.D[q][i]); }
    if (p.r[q] == 0) mn = 0.f;
    s_min[q] = mn; s_max[q] = mx;
  }
  __syncthreads();
  float lam[2];
  for (int q = 0; q < 2; ++q) {
    float l = p.lam[q];
    if (p.flags & 2) l = l * s_max[q];          // relative: lambda = phi * max D
    float shift = 0.f;
    if (p.flags & 1) { shift = s_min[q]; l += shift; }  // continuation
    for (int i = threadIdx.x; i < p.r[q]; i += blockDim.x) {
      const float dd = p.D[q][i] - shift;
      p.s[q][i] = 1.f / (dd + l) - 1.f / l;
    }
    lam[q] = l;
  }
  if (threadIdx.x == 0) {
    p.lam_out[0] = lam[0];
    p.lam_out[1] = lam[1];
    p.lam_out[2] = 1.f / (lam[1] * lam[0]);
    p.lam_out[3] = 1.f / lam[0];
    p.lam_out[4] = 1.f / lam[1];
  }
}

// ---- Philox4x32-10 Gaussian sketch -------------------------------------
// Omega (n x l col-major), element e = j*n + i; counter block e/4, word pair by e%4;
// uniforms (x + 0.5) 2^-32; Box-Muller in fp64; rounded to fp32.
BKFAC_DEV void philox_round(unsigned& c0, unsigned& c1, unsigned& c2, unsigned& c3,
                            unsigned k0, unsigned k1) {
  const unsigned long long p0 = 0xD2511F53ull * c0;
  const unsigned long long p1 = 0xCD9E8D57ull * c2;
  const unsigned hi0 = (unsigned)(p0 >> 32), lo0 = (unsigned)p0;
  const unsigned hi1 = (unsigned)(p1 >> 32), lo1 = (unsigned)p1;
  const unsigned n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
  c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
}

BKFAC_DEV void philox4x32_10(unsigned c[4], unsigned k0, unsigned k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    philox_round(c[0], c[1], c[2], c[3], k0, k1);
  }
}

__global__ void philox_sketch_kernel(float* Om, long total, unsigned long long seed,
                                     unsigned long long counter) {
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total;
       e += (long)gridDim.x * blockDim.x) {
    const unsigned long long blk = (unsigned long long)e >> 2;
    unsigned c[4] = {(unsigned)blk, (unsigned)(blk >> 32), (unsigned)counter,
                     (unsigned)(counter >> 32)};
    philox4x32_10(c, (unsigned)seed, (unsigned)(seed >> 32));
    const int t = (int)(e & 3);
    const int pp = t >> 1;
    const double ua = ((double)c[2 * pp] + 0.5) * 2.3283064365386963e-10;
    const double ub = ((double)c[2 * pp + 1] + 0.5) * 2.3283064365386963e-10;
    const double rad = sqrt(-2.0 * log(ua));
    const double th = 6.283185307179586 * ub;
    const double z = (t & 1) ? rad * sin(th) : rad * cos(th);
    Om[e] = (float)z;
  }
}

}  // namespace bkfac
