// Grouped fp32 SIMT GEMM (CUDA cores), the correctness baseline of every contraction
// on the hot path.  C = alpha * op(A) op(B) + beta * C0, all col-major (BLAS style):
//   TA = false: A(i,k) = A[i + k*lda]      TA = true: A(i,k) = A[k + i*lda]
//   TB = false: B(k,j) = B[k + j*ldb]      TB = true: B(k,j) = B[j + k*ldb]
// The K range may be split in two segments (k < k1 reads A/B, k >= k1 reads A2/B2):
// this expresses [U Q] V and [U_A | X'] [Y'; U_G]^T without packing.
// Split-K writes fp32 partials to a workspace; a second kernel reduces them in a
// fixed order (deterministic, so results do not depend on the GPU count).
#pragma once
#include "common.cuh"

namespace bkfac {

struct GemmProb {
  const float* A; const float* A2; const float* B; const float* B2;
  float* C; const float* C0; float* ws;
  int lda, lda2, ldb, ldb2, ldc, ldc0;
  int M, N, K, k1;
  float alpha, beta;
  const float* beta_dev;   // if non-null, beta = *beta_dev (device scalar)
  int splits, kchunk, tiles_m, tiles_n, tile_start;
  int sym;                 // tcgen05 path: 1: C = C^T known (e.g. M M^T): lower tiles only, mirrored;
                           // 2: lower tiles only, the upper triangle beyond them left untouched
  int tbm;                 // tcgen05 path: square tile edge of a symmetric problem (split-K reduce)
  int nfast;               // tcgen05 path: consecutive tiles walk N first (A row blocks read
                           // once, B re-read from L2) instead of M first
  int stream_c;            // C0 read / C written once (evict-first: keeps the operands in L2)
  int vec;                 // tcgen05 path: bit 0 A (and A2), bit 1 B (and B2) 16-byte aligned
  int promo;               // tcgen05 path: K chunks per TMEM accumulation block (0: TC_PROMO)
  int* status;             // if set: ST_NONFINITE is OR-ed in when C0 (beta != 0) holds
                           // inf/NaN -- the tensor core does not propagate NaN reliably, so
                           // inputs are checked where an epilogue reads them anyway
  // fused epilogue scalings (all optional):
  //   C(i, j) = alpha * (*alpha_dev) * row_scale[i] * col_scale[j] * (AB)(i, j)
  //             + beta * C0(i, j) + [i == j < diag_n] diag_a * diag_vec[i]
  const float* alpha_dev;
  const float* row_scale;
  const float* col_scale;
  const float* diag_vec; float diag_a; int diag_n;
};

// output multiplier of row i (alpha, device alpha, row scale); the column scale is applied per
// element by the epilogues
BKFAC_DEV float gemm_row_alpha(const GemmProb& p, int i) {
  float a = p.alpha;
  if (p.alpha_dev) a *= *p.alpha_dev;
  if (p.row_scale && i < p.M) a *= p.row_scale[i];
  return a;
}
BKFAC_DEV float gemm_out(const GemmProb& p, int i, int j, float ra, float acc, float beta) {
  float v = (p.col_scale ? ra * p.col_scale[j] : ra) * acc;
  if (beta != 0.f) {
    const float c0 = p.C0[i + (long)j * p.ldc0];
    if (p.status && !isfinite(c0)) atomicOr(p.status, ST_NONFINITE);
    v += beta * c0;
  }
  if (p.diag_vec && i == j && i < p.diag_n) v += p.diag_a * p.diag_vec[i];
  return v;
}

constexpr int GEMM_MAXP = 100;
struct GemmBatch {
  int nprob;
  int total_tiles;
  GemmProb p[GEMM_MAXP];
};

constexpr int SG_BM = 64, SG_BN = 64, SG_BK = 16;

template <bool TA>
BKFAC_DEV float gemm_a(const GemmProb& p, int i, int k) {
  if (k < p.k1) return TA ? p.A[k + (long)i * p.lda] : p.A[i + (long)k * p.lda];
  const int kk = k - p.k1;
  return TA ? p.A2[kk + (long)i * p.lda2] : p.A2[i + (long)kk * p.lda2];
}
template <bool TB>
BKFAC_DEV float gemm_b(const GemmProb& p, int k, int j) {
  if (k < p.k1) return TB ? p.B[j + (long)k * p.ldb] : p.B[k + (long)j * p.ldb];
  const int kk = k - p.k1;
  return TB ? p.B2[j + (long)kk * p.ldb2] : p.B2[kk + (long)j * p.ldb2];
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const __grid_constant__ GemmBatch b) {
  const int t = blockIdx.x;
  int pi = 0;
  while (pi + 1 < b.nprob && b.p[pi + 1].tile_start <= t) ++pi;
  const GemmProb& p = b.p[pi];
  const int lt = t - p.tile_start;
  const int per_split = p.tiles_m * p.tiles_n;
  const int s = lt / per_split;
  const int rem = lt - s * per_split;
  const int row0 = (rem % p.tiles_m) * SG_BM;
  const int col0 = (rem / p.tiles_m) * SG_BN;
  const int kbeg = s * p.kchunk;
  const int kend = min(p.K, kbeg + p.kchunk);

  __shared__ __align__(16) float As[2][SG_BK][SG_BM + 4];
  __shared__ __align__(16) float Bs[2][SG_BK][SG_BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;

  float ra[4], rb[4];
  auto load = [&](int k0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int i, k;
      if (!TA) { i = row0 + (tid & 63); k = k0 + (tid >> 6) + 4 * q; }
      else     { k = k0 + (tid & 15);   i = row0 + (tid >> 4) + 16 * q; }
      ra[q] = (i < p.M && k < kend) ? gemm_a<TA>(p, i, k) : 0.f;
      int j;
      if (!TB) { k = k0 + (tid & 15);   j = col0 + (tid >> 4) + 16 * q; }
      else     { j = col0 + (tid & 63); k = k0 + (tid >> 6) + 4 * q; }
      rb[q] = (j < p.N && k < kend) ? gemm_b<TB>(p, k, j) : 0.f;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (!TA) As[buf][(tid >> 6) + 4 * q][tid & 63] = ra[q];
      else     As[buf][tid & 15][(tid >> 4) + 16 * q] = ra[q];
      if (!TB) Bs[buf][tid & 15][(tid >> 4) + 16 * q] = rb[q];
      else     Bs[buf][(tid >> 6) + 4 * q][tid & 63] = rb[q];
    }
  };

  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  int buf = 0;
  if (kbeg < kend) {
    load(kbeg);
    store(0);
    __syncthreads();
    for (int k0 = kbeg; k0 < kend; k0 += SG_BK) {
      const bool more = k0 + SG_BK < kend;
      if (more) load(k0 + SG_BK);
#pragma unroll
      for (int kk = 0; kk < SG_BK; ++kk) {
        const float4 a = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
        const float4 bb = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
        const float av[4] = {a.x, a.y, a.z, a.w};
        const float bv[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      if (more) {
        store(buf ^ 1);
        __syncthreads();
        buf ^= 1;
      }
    }
  }

  const float beta = p.beta_dev ? *p.beta_dev : p.beta;
  if (p.splits == 1) {
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int j = col0 + tx * 4 + jj;
      if (j >= p.N) continue;
#pragma unroll
      for (int ii = 0; ii < 4; ++ii) {
        const int i = row0 + ty * 4 + ii;
        if (i >= p.M) continue;
        p.C[i + (long)j * p.ldc] = gemm_out(p, i, j, gemm_row_alpha(p, i), acc[ii][jj], beta);
      }
    }
  } else {
    float* w = p.ws + (long)s * p.M * p.N;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int j = col0 + tx * 4 + jj;
      if (j >= p.N) continue;
#pragma unroll
      for (int ii = 0; ii < 4; ++ii) {
        const int i = row0 + ty * 4 + ii;
        if (i < p.M) w[i + (long)j * p.M] = acc[ii][jj];
      }
    }
  }
}

// Deterministic split-K reduction: fixed summation order over splits.
__global__ void gemm_splitk_reduce_kernel(const __grid_constant__ GemmBatch b) {
  const GemmProb& p = b.p[blockIdx.y];
  if (p.splits <= 1) return;
  const long total = (long)p.M * p.N;
  const float beta = p.beta_dev ? *p.beta_dev : p.beta;
  if ((p.M & 3) == 0) {
    // 4 consecutive rows of one column per thread (a symmetric problem's tile edge is a
    // multiple of 4, so a group never straddles a tile): 16-byte partial loads, the splits'
    // loads in flight together; the same per-element summation order as the scalar path
    // (0 + w_0 + w_1 + ...), so results are bitwise those of the scalar loop.
    const int M4 = p.M >> 2;
    const long items = (long)M4 * p.N;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < items;
         e += (long)gridDim.x * blockDim.x) {
      const int i = (int)(e % M4) * 4, j = (int)(e / M4);
      const bool mir = p.sym && i / p.tbm < j / p.tbm;   // upper tile
      if (mir && p.sym == 2) continue;                   // left untouched
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      if (!mir) {
        const float* w = p.ws + i + (long)j * p.M;
#pragma unroll 8
        for (int s = 0; s < p.splits; ++s) {
          const float4 q = __ldg(reinterpret_cast<const float4*>(w + (long)s * total));
          acc[0] += q.x; acc[1] += q.y; acc[2] += q.z; acc[3] += q.w;
        }
      } else {                                           // mirrored: C(i, j) = C(j, i)
        const float* w = p.ws + j + (long)i * p.M;
#pragma unroll 4
        for (int s = 0; s < p.splits; ++s)
#pragma unroll
          for (int t = 0; t < 4; ++t) acc[t] += __ldg(w + (long)s * total + (long)t * p.M);
      }
#pragma unroll
      for (int t = 0; t < 4; ++t)
        p.C[i + t + (long)j * p.ldc] = gemm_out(p, i + t, j, gemm_row_alpha(p, i + t), acc[t], beta);
    }
    return;
  }
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total;
       e += (long)gridDim.x * blockDim.x) {
    const int i = (int)(e % p.M), j = (int)(e / p.M);
    long src = e;
    if (p.sym && i / p.tbm < j / p.tbm) {   // upper tile: not computed
      if (p.sym == 2) continue;               // left untouched
      src = j + (long)i * p.M;                // mirrored: C(i, j) = C(j, i), a lower tile
    }
    float acc = 0.f;
    for (int s = 0; s < p.splits; ++s) acc += p.ws[(long)s * total + src];
    p.C[i + (long)j * p.ldc] = gemm_out(p, i, j, gemm_row_alpha(p, i), acc, beta);
  }
}

}  // namespace bkfac
