// Blocked Cholesky factorisation and triangular inverse of the c x c Gram matrix
// G = R^T R of CholeskyQR (Alg 3 line 2 "QR_decomp(A_perp)"; footnote :451
// allows any orthonormal decomposition) -- one CTA per factor (or, with few factors per
// GPU, a cluster of up to 8 CTAs sharing the global tiles), 32 x 32 register tiles.
//
// G is split into NB = ceil(c/32) block rows/columns (padding: identity), tiles packed
// lower-triangular in a global scratch (L1/L2 resident):
//   L tiles  col-major (element (i,j) at j*32 + i),  T(I,J) = I(I+1)/2 + J, I >= J
//   X tiles  row-major (element (i,j) at i*32 + j),  X = L^{-1}
// Right-looking Cholesky, for each block column J:
//   (1) one warp factors the diagonal tile (lane = row, rows in registers, shuffles)
//       and inverts it (lane = column);                                         barrier
//   (2) every warp takes below-diagonal tiles: L_IJ = G_IJ X_JJ^T;              barrier
//   (3) every warp takes trailing tiles (I >= K > J): G_IK -= L_IJ L_KJ^T;     barrier
// then X = L^{-1} right-looking by block rows K (X_KJ = X_KK A_KJ, then A_IJ -= L_IK X_KJ
// for all I > K in parallel), A_IJ = -sum_{M<I} L_IM X_MJ accumulated in place.
// The tile products run on FP32 FFMA with the B tile read as broadcast float4 loads.
// A pivot <= tol * max_i G_ii (rank-deficient residual) is dropped: its column of L and
// row of X are zero and ST_CHOL_DROP is reported (informational, as before).
// Outputs: L and Linv = L^{-1} (c x c col-major, zeros above the diagonal).
#pragma once
#include <cooperative_groups.h>
#include "chol.cuh"
#include "common.cuh"

namespace bkfac {

constexpr int CT_THREADS = 512;

BKFAC_DEV int ctix(int I, int J) { return I * (I + 1) / 2 + J; }

// acc[j] -= (or +=) sum_k A(lane, k) * B(j, k); A, B col-major 32 x 32 tiles.  The FMAs run
// on column pairs (FFMA2: half the FP instructions; same per-element rounding as FFMA).
template <bool SUB>
BKFAC_DEV void tile_abt(float (&acc)[32], const float* A, const float* B, int lane) {
  float2* acc2 = reinterpret_cast<float2*>(acc);
#pragma unroll 2
  for (int k = 0; k < 32; ++k) {
    const float a = SUB ? -A[k * 32 + lane] : A[k * 32 + lane];
    const float2 a2 = make_float2(a, a);
    const float4* b4 = reinterpret_cast<const float4*>(B + k * 32);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 bb = b4[q];
      acc2[2 * q] = __ffma2_rn(a2, make_float2(bb.x, bb.y), acc2[2 * q]);
      acc2[2 * q + 1] = __ffma2_rn(a2, make_float2(bb.z, bb.w), acc2[2 * q + 1]);
    }
  }
}
// acc[j] += sum_k A(lane, k) * B(k, j); A col-major, B row-major 32 x 32 tiles
BKFAC_DEV void tile_ab(float (&acc)[32], const float* A, const float* Brm, int lane) {
  float2* acc2 = reinterpret_cast<float2*>(acc);
#pragma unroll 2
  for (int k = 0; k < 32; ++k) {
    const float a = A[k * 32 + lane];
    const float2 a2 = make_float2(a, a);
    const float4* b4 = reinterpret_cast<const float4*>(Brm + k * 32);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 bb = b4[q];
      acc2[2 * q] = __ffma2_rn(a2, make_float2(bb.x, bb.y), acc2[2 * q]);
      acc2[2 * q + 1] = __ffma2_rn(a2, make_float2(bb.z, bb.w), acc2[2 * q + 1]);
    }
  }
}

// Copy one 32 x 32 tile (1024 floats, 16-byte aligned) global -> this warp's shared
// buffer with all loads in flight at once (one L2 round trip instead of one per column).
BKFAC_DEV void tile_stage(float* dst, const float* src, int lane) {
  float4 r[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) r[q] = reinterpret_cast<const float4*>(src)[q * 32 + lane];
#pragma unroll
  for (int q = 0; q < 8; ++q) reinterpret_cast<float4*>(dst)[q * 32 + lane] = r[q];
}

// ---- 32 x 32 diagonal tile on one warp, fully unrolled by templates (compile-time
// register indices: no local memory).  Factor: lane = row i, a[j] = A(i, j).  Step K
// publishes column K of L to shared memory (col-major scratch D) and every lane reads it
// back as broadcast float4 loads (8 loads instead of 31 shuffles per step).
template <int K, int Q>
BKFAC_DEV void ct_upd4(float (&a)[32], float lik, const float* D, int lane) {
  if constexpr (Q < 8) {
    if constexpr (4 * Q + 3 > K) {
      const float4 l4 = reinterpret_cast<const float4*>(D + K * 32)[Q];
      const float lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int j = 4 * Q + t;
        if (j > K && lane >= j) a[j] = fmaf(-lik, lv[t], a[j]);
      }
    }
    ct_upd4<K, Q + 1>(a, lik, D, lane);
  }
}
template <int K>
BKFAC_DEV void ct_factor(float (&a)[32], float* D, int lane, int nreal, float tol, int& dropped) {
  if constexpr (K < 32) {
    const float akk = __shfl_sync(0xffffffffu, a[K], K);
    const bool drop = (K < nreal) && !(akk > tol);
    const float rs = drop ? 0.f : rsqrtf(fmaxf(akk, 1e-38f));   // 1 / l_kk (MUFU)
    const float lkk = drop ? 0.f : fmaxf(akk, 1e-38f) * rs;
    dropped |= drop;
    const float lik = (lane > K) ? a[K] * rs : (lane == K ? lkk : 0.f);
    a[K] = lik;
    if constexpr (K < 31) {
      D[K * 32 + lane] = lik;
      __syncwarp();
      ct_upd4<K, 0>(a, lik, D, lane);
    }
    ct_factor<K + 1>(a, D, lane, nreal, tol, dropped);
  }
}
// Inverse of the lower-triangular tile: R (row-major copy of L in shared memory) is read
// row by row as broadcast float4 loads; lane j computes column j of X = L^{-1}:
// x[i] = X(i, j) = (delta_ij - sum_{k<i} L(i,k) x[k]) / L(i,i).
template <int I, int Q>
BKFAC_DEV void ct_inv_dot4(const float* R, const float (&x)[32], float& s) {
  if constexpr (4 * Q < I) {
    const float4 l4 = reinterpret_cast<const float4*>(R + I * 32)[Q];
    const float lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (4 * Q + t < I) s = fmaf(lv[t], x[4 * Q + t], s);
    ct_inv_dot4<I, Q + 1>(R, x, s);
  }
}
template <int I>
BKFAC_DEV void ct_inverse(const float* R, float (&x)[32], int lane) {
  if constexpr (I < 32) {
    float s = 0.f;
    ct_inv_dot4<I, 0>(R, x, s);          // terms with x[k] = 0 (k < lane) add zero
    const float lii = R[I * 32 + I];
    const float rinv = (lii > 0.f) ? __frcp_rn(lii) : 0.f;
    x[I] = (I < lane) ? 0.f : (I == lane ? rinv : -s * rinv);
    ct_inverse<I + 1>(R, x, lane);
  }
}

struct CholTiledProb {
  const float* G; int ldg;
  float* L; float* Linv;   // c x c col-major, ld = ldl (0: c)
  float* tiles;            // chol_tiled_scratch_floats(c) floats of scratch
  int* status;
  int c;
  float shift;
  int ldl;                 // leading dimension of L / Linv (0: c); chol_smem_kernel only
  const float* gref;       // optional device scalar: pivot-drop tolerance reference (the whole
                           // matrix's max diagonal when this problem is a diagonal block of it)
};
constexpr int CT_MAXP = 100;
struct CholTiledBatch { int nprob; CholTiledProb p[CT_MAXP]; };

constexpr size_t CT_SMEM_BYTES = (size_t)(CT_THREADS / 32) * 2048 * sizeof(float);
inline size_t chol_tiled_scratch_floats(int c) {
  const size_t NB = (size_t)(c + 31) / 32;
  return 2 * NB * (NB + 1) / 2 * 1024 + NB * 1024;
}

#ifdef BKFAC_CHOL_TIMING
__device__ unsigned long long g_chol_dbg[8];   // tuning builds: per-phase cycle sums (CTA 0)
#define CT_T(ph) do { if (threadIdx.x == 0 && blockIdx.x == 0) { const unsigned long long tn = clock64(); g_chol_dbg[ph] += tn - ct_prev; ct_prev = tn; } } while (0)
#else
#define CT_T(ph) do {} while (0)
#endif
// C > 1: a cluster of C CTAs per factor (tiles in global memory / L2 are shared; every
// tile loop is dealt over the cluster's C * 16 warps, the phase barriers are cluster
// barriers, the diagonal tiles are factored by CTA 0) -- for few factors per GPU (an 8-GPU
// rank's share of configs[4]), where one CTA per factor leaves most SMs idle.
__global__ void __launch_bounds__(CT_THREADS, 1) chol_tiled_kernel(const __grid_constant__ CholTiledBatch b, int C) {
#ifdef BKFAC_CHOL_TIMING
  unsigned long long ct_prev = clock64();
#endif
  cooperative_groups::cluster_group cluster = cooperative_groups::this_cluster();
  const int q = C > 1 ? (int)cluster.block_rank() : 0;
  const CholTiledProb& p = b.p[blockIdx.x / C];
  const int c = p.c, NB = (c + 31) >> 5;
  const int ntile = NB * (NB + 1) / 2;
  float* Lt = p.tiles;                       // L tiles (col-major)
  float* Xt = Lt + (size_t)ntile * 1024;     // X tiles (row-major)
  float* Xd = Xt + (size_t)ntile * 1024;     // col-major copies of the diagonal X_JJ
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = CT_THREADS / 32;
  const int gw = q * NW + warp, NWC = NW * C;   // warp index / count over the cluster
  auto csync = [&]() { if (C > 1) cluster.sync(); else __syncthreads(); };
  __shared__ float red[32];
  __shared__ float s_part[2];
  __shared__ int s_drop;
  extern __shared__ __align__(16) float ctsm[];
  float* sA = ctsm + warp * 2048;     // per-warp staging: A tile, B tile
  float* sB = sA + 1024;

  // ---- load G (lower) into tiles, identity padding; trace and max diagonal
  float dsum = 0.f, dmax = 0.f;
  for (int t = gw; t < ntile; t += NWC) {
    int I = 0;
    while ((I + 1) * (I + 2) / 2 <= t) ++I;
    const int J = t - I * (I + 1) / 2;
    float* T = Lt + (size_t)t * 1024;
    float gv[32];   // all 32 loads in flight before the stores
    const int i = 32 * I + lane;
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) {
      const int j = 32 * J + jj;
      gv[jj] = (i < c && j < c && i >= j) ? p.G[i + (long)j * p.ldg] : 0.f;
    }
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) {
      const int j = 32 * J + jj;
      float g = gv[jj];
      if (!(i < c && j < c)) g = (i == j) ? 1.f : 0.f;
      T[jj * 32 + lane] = g;
      if (i == j && i < c) { dsum += g; dmax = fmaxf(dmax, g); }
    }
  }
  float trace = block_sum(dsum, red);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dmax = fmaxf(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  if (lane == 0) red[warp] = dmax;
  __syncthreads();
  float gmax = 0.f;
  for (int w = 0; w < NW; ++w) gmax = fmaxf(gmax, red[w]);
  if (tid == 0) s_drop = 0;
  if (C > 1) {                       // the cluster's trace and max diagonal, in rank order
    if (tid == 0) { s_part[0] = trace; s_part[1] = gmax; }
    cluster.sync();                  // also: every CTA's tiles of G are loaded
    float tr = 0.f, gm = 0.f;
    for (int r = 0; r < C; ++r) {
      const float* rp = cluster.map_shared_rank(s_part, r);
      tr += rp[0];
      gm = fmaxf(gm, rp[1]);
    }
    trace = tr;
    gmax = gm;
    cluster.sync();                  // no CTA reuses / leaves s_part while it is read
  }
  // shifted first pass (sCQR, Fukaya et al. 2020): G_ii += shift * tr(G)
  const float sh = (p.shift > 0.f) ? p.shift * trace : 0.f;
  const float tol = 4.0f * 1.1920929e-7f * (gmax + sh);
  __syncthreads();
  CT_T(0);

  for (int J = 0; J < NB; ++J) {
    // (1) diagonal tile: one warp factors it (lane = row, register rows, shuffles; fully
    //     unrolled by templates) and inverts it (lane = column).
    if (q == 0 && warp == 0) {
      float* T = Lt + (size_t)ctix(J, J) * 1024;
      float a[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) a[j] = T[j * 32 + lane];
      const bool real = 32 * J + lane < c;
      if (sh > 0.f && real) {
#pragma unroll
        for (int j = 0; j < 32; ++j) if (j == lane) a[j] += sh;
      }
      int dropped = 0;
      ct_factor<0>(a, sA, lane, c - 32 * J, tol, dropped);
      // write L_JJ (lower), zero the upper part; row-major copy (lane = row) for the
      // inverse, rows 16-byte aligned: element (i, j) at i*32 + j
#pragma unroll
      for (int j = 0; j < 32; ++j) T[j * 32 + lane] = (lane >= j) ? a[j] : 0.f;
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 8; ++q)
        reinterpret_cast<float4*>(sB + lane * 32)[q] =
            make_float4(lane >= 4 * q ? a[4 * q] : 0.f, lane >= 4 * q + 1 ? a[4 * q + 1] : 0.f,
                        lane >= 4 * q + 2 ? a[4 * q + 2] : 0.f, lane >= 4 * q + 3 ? a[4 * q + 3] : 0.f);
      __syncwarp();
      float x[32];
      ct_inverse<0>(sB, x, lane);
      // X_JJ: row-major into the X tiles, col-major copy into Xd
      float* XJ = Xt + (size_t)ctix(J, J) * 1024;
      float* XJc = Xd + (size_t)J * 1024;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        XJ[i * 32 + lane] = x[i];       // element (i, lane)
        XJc[lane * 32 + i] = x[i];      // col-major: column lane
      }
      if (dropped && lane == 0) s_drop = 1;
    }
    csync();
    CT_T(1);
    // (2) L_IJ = G_IJ X_JJ^T for I > J (X_JJ^T(k, j) = X_JJ(j, k) -> col-major copy as B)
    for (int I = J + 1 + gw; I < NB; I += NWC) {
      float* T = Lt + (size_t)ctix(I, J) * 1024;
      float acc[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = 0.f;
      // acc(i, j) = sum_k G(i, k) X_JJ(j, k): B = X_JJ col-major
      tile_stage(sA, T, lane);
      tile_stage(sB, Xd + (size_t)J * 1024, lane);
      __syncwarp();
      tile_abt<false>(acc, sA, sB, lane);
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 32; ++j) T[j * 32 + lane] = acc[j];
    }
    csync();
    CT_T(2);
    // (3) trailing update G_IK -= L_IJ L_KJ^T for I >= K > J
    {
      const int n = NB - J - 1;
      const int npairs = n * (n + 1) / 2;
      for (int t = gw; t < npairs; t += NWC) {
        int a = 0;
        while ((a + 1) * (a + 2) / 2 <= t) ++a;
        const int I = J + 1 + a, K = J + 1 + (t - a * (a + 1) / 2);
        float* T = Lt + (size_t)ctix(I, K) * 1024;
        float acc[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = T[j * 32 + lane];
        // B(j, k) = L_KJ(j, k): col-major L tile is element (j,k) at k*32 + j -- we need
        // B rows contiguous in j for fixed k: that is exactly the col-major layout.
        tile_stage(sA, Lt + (size_t)ctix(I, J) * 1024, lane);
        tile_stage(sB, Lt + (size_t)ctix(K, J) * 1024, lane);
        __syncwarp();
        tile_abt<true>(acc, sA, sB, lane);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 32; ++j) T[j * 32 + lane] = acc[j];
      }
    }
    csync();
    CT_T(3);
  }
  // ---- X = L^{-1}, right-looking by block rows K: the off-diagonal X tiles first hold
  // the accumulators A_IJ = -sum_{M<I} L_IM X_MJ (zero-initialised), then
  //   (1) X_KJ = X_KK A_KJ for J < K;     (2) A_IJ -= L_IK X_KJ for I > K, J <= K.
  for (int t = gw; t < ntile; t += NWC) {
    int I = 0;
    while ((I + 1) * (I + 2) / 2 <= t) ++I;
    if (t - I * (I + 1) / 2 == I) continue;            // diagonal X_II already set
    float4* T4 = reinterpret_cast<float4*>(Xt + (size_t)t * 1024);
#pragma unroll
    for (int q = 0; q < 8; ++q) T4[q * 32 + lane] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  csync();
  for (int K = 0; K < NB; ++K) {
    for (int J = gw; J < K; J += NWC) {                // (1)
      float* XK = Xt + (size_t)ctix(K, J) * 1024;
      float acc[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = 0.f;
      tile_stage(sA, Xd + (size_t)K * 1024, lane);     // X_KK col-major
      tile_stage(sB, XK, lane);                        // A_KJ row-major
      __syncwarp();
      tile_ab(acc, sA, sB, lane);
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 32; ++j) XK[lane * 32 + j] = acc[j];
    }
    csync();
    CT_T(5);
    const int nI = NB - K - 1, nJ = K + 1;
    for (int t = gw; t < nI * nJ; t += NWC) {          // (2)
      const int I = K + 1 + t / nJ, J = t % nJ;
      float* XI = Xt + (size_t)ctix(I, J) * 1024;
      float acc[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = 0.f;
      tile_stage(sA, Lt + (size_t)ctix(I, K) * 1024, lane);   // L_IK col-major
      tile_stage(sB, Xt + (size_t)ctix(K, J) * 1024, lane);   // X_KJ row-major
      __syncwarp();
      tile_ab(acc, sA, sB, lane);
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 32; ++j) XI[lane * 32 + j] -= acc[j];
    }
    csync();
    CT_T(6);
  }
  // ---- outputs: L and Linv, c x c col-major, zeros above the diagonal
  for (int t = gw; t < NB * NB; t += NWC) {
    const int I = t % NB, J = t / NB;
    const int i = 32 * I + lane;
    float lv[32], xv[32];   // all loads in flight before the stores
    if (I >= J) {
      const float* LT = Lt + (size_t)ctix(I, J) * 1024;
      const float4* XT = reinterpret_cast<const float4*>(Xt + (size_t)ctix(I, J) * 1024 + lane * 32);
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) lv[jj] = LT[jj * 32 + lane];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 x4 = XT[q];
        xv[4 * q] = x4.x; xv[4 * q + 1] = x4.y; xv[4 * q + 2] = x4.z; xv[4 * q + 3] = x4.w;
      }
    } else {
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) { lv[jj] = 0.f; xv[jj] = 0.f; }
    }
    if (i < c) {
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) {
        const int j = 32 * J + jj;
        if (j >= c) break;
        const bool up = (I == J && lane < jj);
        p.L[i + (long)j * c] = up ? 0.f : lv[jj];
        p.Linv[i + (long)j * c] = up ? 0.f : xv[jj];
      }
    }
  }
  if (tid == 0 && s_drop && p.status) atomicOr(p.status, ST_CHOL_DROP);
  CT_T(7);
}

// ---- c <= 256: every tile resident in shared memory -------------------------------------
// Same right-looking factorisation as chol_tiled_kernel with the NB(NB+1)/2 L tiles
// (col-major) in shared memory and products read straight from it (no staging).  The
// inverse is formed IN PLACE, right-looking by block rows K:
//   (1) X_KJ = X_KK A_KJ            for J < K       (A_KJ row-major accumulator at (K, J))
//   (2a) A_IJ -= L_IK X_KJ          for I > K, J < K
//   (2b) A_IK  = -L_IK X_KK         for I > K        (position (I, K): L_IK -> accumulator)
// so a position holds L_IJ (col-major) until step K = J, then the row-major accumulator /
// X_IJ.  X_KK = L_KK^{-1} comes from the diagonal step (col-major copy in Xd).
constexpr int CS_MAXNB = 8;
inline size_t chol_smem_bytes(int c) {
  const size_t NB = (size_t)(c + 31) / 32;
  return sizeof(float) * (NB * (NB + 1) / 2 * 1024 + 2 * NB * 1024 + 2 * 1024);
}

__global__ void __launch_bounds__(CT_THREADS, 1) chol_smem_kernel(const __grid_constant__ CholTiledBatch b) {
  const CholTiledProb& p = b.p[blockIdx.x];
  const int c = p.c, NB = (c + 31) >> 5;
  const int ntile = NB * (NB + 1) / 2;
  extern __shared__ __align__(16) float cssm[];
  float* Lt = cssm;                              // ntile tiles
  float* Xd = Lt + (size_t)ntile * 1024;         // NB col-major X_KK
  float* Xr = Xd + (size_t)NB * 1024;            // NB row-major X_KK
  float* sD = Xr + (size_t)NB * 1024;            // warp-0 scratch: columns of L_JJ
  float* sR = sD + 1024;                         //                 row-major L_JJ
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = CT_THREADS / 32;
  __shared__ float red[32];
  __shared__ int s_drop;
  auto tile = [&](int I, int J) { return Lt + (size_t)ctix(I, J) * 1024; };

  // ---- load G (lower) into tiles, identity padding; trace and max diagonal
  float dsum = 0.f, dmax = 0.f;
  for (int t = warp; t < ntile; t += NW) {
    int I = 0;
    while ((I + 1) * (I + 2) / 2 <= t) ++I;
    const int J = t - I * (I + 1) / 2;
    float* T = Lt + (size_t)t * 1024;
    float gv[32];
    const int i = 32 * I + lane;
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) {
      const int j = 32 * J + jj;
      gv[jj] = (i < c && j < c && i >= j) ? p.G[i + (long)j * p.ldg] : 0.f;
    }
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) {
      const int j = 32 * J + jj;
      float g = gv[jj];
      if (!(i < c && j < c)) g = (i == j) ? 1.f : 0.f;
      T[jj * 32 + lane] = g;
      if (i == j && i < c) { dsum += g; dmax = fmaxf(dmax, g); }
    }
  }
  const float trace = block_sum(dsum, red);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dmax = fmaxf(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  if (lane == 0) red[warp] = dmax;
  __syncthreads();
  float gmax = 0.f;
  for (int w = 0; w < NW; ++w) gmax = fmaxf(gmax, red[w]);
  if (p.gref) gmax = fmaxf(gmax, *p.gref);
  if (tid == 0) s_drop = 0;
  const float sh = (p.shift > 0.f) ? p.shift * trace : 0.f;   // shifted CholeskyQR
  const float tol = 4.0f * 1.1920929e-7f * (gmax + sh);
  const long ldl = p.ldl ? p.ldl : c;
  __syncthreads();

  for (int J = 0; J < NB; ++J) {
    // (1) diagonal tile on warp 0: factor (lane = row) and invert (lane = column)
    if (warp == 0) {
      float* T = tile(J, J);
      float a[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) a[j] = T[j * 32 + lane];
      const bool real = 32 * J + lane < c;
      if (sh > 0.f && real) {
#pragma unroll
        for (int j = 0; j < 32; ++j) if (j == lane) a[j] += sh;
      }
      int dropped = 0;
      ct_factor<0>(a, sD, lane, c - 32 * J, tol, dropped);
#pragma unroll
      for (int j = 0; j < 32; ++j) T[j * 32 + lane] = (lane >= j) ? a[j] : 0.f;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        reinterpret_cast<float4*>(sR + lane * 32)[q] =
            make_float4(lane >= 4 * q ? a[4 * q] : 0.f, lane >= 4 * q + 1 ? a[4 * q + 1] : 0.f,
                        lane >= 4 * q + 2 ? a[4 * q + 2] : 0.f, lane >= 4 * q + 3 ? a[4 * q + 3] : 0.f);
      __syncwarp();
      float x[32];
      ct_inverse<0>(sR, x, lane);
      float* XJc = Xd + (size_t)J * 1024;      // col-major: lane = column
      float* XJr = Xr + (size_t)J * 1024;      // row-major
#pragma unroll
      for (int q = 0; q < 8; ++q)
        reinterpret_cast<float4*>(XJc + lane * 32)[q] = make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
#pragma unroll
      for (int i = 0; i < 32; ++i) XJr[i * 32 + lane] = x[i];
      if (dropped && lane == 0) s_drop = 1;
    }
    __syncthreads();
    // (2) L_IJ = G_IJ X_JJ^T for I > J, in place (B(j, k) = X_JJ(j, k): col-major X_JJ)
    for (int I = J + 1 + warp; I < NB; I += NW) {
      float* T = tile(I, J);
      float acc[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = 0.f;
      tile_abt<false>(acc, T, Xd + (size_t)J * 1024, lane);
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 32; ++j) T[j * 32 + lane] = acc[j];
    }
    __syncthreads();
    // (3) trailing update G_IK -= L_IJ L_KJ^T for I >= K > J
    {
      const int n = NB - J - 1;
      const int npairs = n * (n + 1) / 2;
      for (int t = warp; t < npairs; t += NW) {
        int a = 0;
        while ((a + 1) * (a + 2) / 2 <= t) ++a;
        const int I = J + 1 + a, K = J + 1 + (t - a * (a + 1) / 2);
        float* T = tile(I, K);
        float acc[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = T[j * 32 + lane];
        tile_abt<true>(acc, tile(I, J), tile(K, J), lane);
#pragma unroll
        for (int j = 0; j < 32; ++j) T[j * 32 + lane] = acc[j];
      }
    }
    __syncthreads();
  }
  // ---- L out (c x c col-major, zeros above the diagonal)
  for (int t = warp; t < NB * NB; t += NW) {
    const int I = t % NB, J = t / NB;
    const int i = 32 * I + lane;
    if (i >= c) continue;
    const float* T = I >= J ? tile(I, J) : nullptr;
    for (int jj = 0; jj < 32; ++jj) {
      const int j = 32 * J + jj;
      if (j >= c) break;
      p.L[i + (long)j * ldl] = (T && !(I == J && lane < jj)) ? T[jj * 32 + lane] : 0.f;
    }
  }
  __syncthreads();
  // ---- in-place inverse
  for (int K = 0; K < NB; ++K) {
    for (int J = warp; J < K; J += NW) {                 // (1) X_KJ = X_KK A_KJ
      float* T = tile(K, J);
      float acc[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = 0.f;
      tile_ab(acc, Xd + (size_t)K * 1024, T, lane);
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 8; ++q)
        reinterpret_cast<float4*>(T + lane * 32)[q] = make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
    }
    __syncthreads();
    const int nI = NB - K - 1;
    for (int t = warp; t < nI * K; t += NW) {             // (2a) A_IJ -= L_IK X_KJ, J < K
      const int I = K + 1 + t / K, J = t % K;
      float* T = tile(I, J);
      float acc[32];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 v4 = reinterpret_cast<const float4*>(T + lane * 32)[q];
        acc[4 * q] = v4.x; acc[4 * q + 1] = v4.y; acc[4 * q + 2] = v4.z; acc[4 * q + 3] = v4.w;
      }
      float prod[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) prod[j] = 0.f;
      tile_ab(prod, tile(I, K), tile(K, J), lane);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        reinterpret_cast<float4*>(T + lane * 32)[q] =
            make_float4(acc[4 * q] - prod[4 * q], acc[4 * q + 1] - prod[4 * q + 1],
                        acc[4 * q + 2] - prod[4 * q + 2], acc[4 * q + 3] - prod[4 * q + 3]);
    }
    __syncthreads();
    for (int I = K + 1 + warp; I < NB; I += NW) {          // (2b) A_IK = -L_IK X_KK
      float* T = tile(I, K);
      float acc[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = 0.f;
      tile_ab(acc, T, Xr + (size_t)K * 1024, lane);      // L_IK X_KK (X_KK row-major)
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = -acc[j];
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 8; ++q)
        reinterpret_cast<float4*>(T + lane * 32)[q] = make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
    }
    __syncthreads();
  }
  // ---- Linv out: off-diagonal X tiles row-major in place, diagonal X_KK col-major in Xd
  for (int t = warp; t < NB * NB; t += NW) {
    const int I = t % NB, J = t / NB;
    const int i = 32 * I + lane;
    float xv[32];
    if (I > J) {
      const float4* X4 = reinterpret_cast<const float4*>(tile(I, J) + lane * 32);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 x4 = X4[q];
        xv[4 * q] = x4.x; xv[4 * q + 1] = x4.y; xv[4 * q + 2] = x4.z; xv[4 * q + 3] = x4.w;
      }
    } else if (I == J) {
      const float* XJc = Xd + (size_t)J * 1024;
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) xv[jj] = (lane >= jj) ? XJc[jj * 32 + lane] : 0.f;
    } else {
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) xv[jj] = 0.f;
    }
    if (i < c) {
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) {
        const int j = 32 * J + jj;
        if (j >= c) break;
        p.Linv[i + (long)j * ldl] = xv[jj];
      }
    }
  }
  if (tid == 0 && s_drop && p.status) atomicOr(p.status, ST_CHOL_DROP);
}

// Blocked Cholesky for c > 256 (host side: run_chol_blocked in bkfac_api.cu): 256 x 256
// diagonal blocks on chol_smem_kernel, the panel solve L21 = A21 L11^{-T} and the trailing
// update A22 -= L21 L21^T (SYRK), and the off-diagonal blocks of L^{-1}, on the tcgen05 GEMM.
// This kernel starts it: A = lower(G) + shift * trace(G) I into L (upper zero), L^{-1} = 0,
// and the tolerance reference max_i G_ii + shift trace(G) into *gref.
// grid (nprob, 32), block 256.
__global__ void __launch_bounds__(256) chol_blocked_prep_kernel(const __grid_constant__ CholTiledBatch b) {
  const CholTiledProb& p = b.p[blockIdx.x];
  const int c = p.c;
  __shared__ float red[32];
  float ds = 0.f, dm = 0.f;
  for (int i = threadIdx.x; i < c; i += blockDim.x) {
    const float g = p.G[i + (long)i * p.ldg];
    ds += g;
    dm = fmaxf(dm, g);
  }
  const float trace = block_sum(ds, red);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dm = fmaxf(dm, __shfl_xor_sync(0xffffffffu, dm, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dm;
  __syncthreads();
  float gmax = 0.f;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) gmax = fmaxf(gmax, red[w]);
  const float sh = (p.shift > 0.f) ? p.shift * trace : 0.f;
  if (blockIdx.y == 0 && threadIdx.x == 0) *const_cast<float*>(p.gref) = gmax + sh;
  const long tot = (long)c * c;
  for (long e = blockIdx.y * (long)blockDim.x + threadIdx.x; e < tot; e += (long)gridDim.y * blockDim.x) {
    const int i = (int)(e % c), j = (int)(e / c);
    float v = 0.f;
    if (i >= j) v = p.G[i + (long)j * p.ldg] + (i == j ? sh : 0.f);
    p.L[e] = v;
    p.Linv[e] = 0.f;
  }
}

}  // namespace bkfac
