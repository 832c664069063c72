// Two-stage Householder tridiagonalisation for the large eigenproblems of the path (the
// Brand cores of order m = r + c = 1536 at configs[4]): "EVD(M_S)" of Alg 3 line 4
// (PAPER.md:505).  The one-stage reduction (sytrd_tiled.cuh) streams the whole trailing
// matrix once per column -- 4/3 m^3 bytes per factor, HBM-bound when 96 such factors run
// at once.  Here the reduction is split:
//
// Stage 1, dense -> band (bandwidth SBR_B = 32), panel by panel j (columns c0 = 32 j ..
// c0 + 31, rows below the band r0 = c0 + 32 .. m - 1, L = m - r0):
//   sbr_panel_kernel  Householder QR of P = K[r0:, c0:c0+32] in shared memory: R stays in
//                     K (it is the band part of those columns), the reflectors' tails go
//                     below it (geqrf layout: reflector of column k has its unit at row
//                     k + 32), the explicit unit-lower V into Vp and the compact-WY factor T
//                     (Q = I - V T V^T, dlarft recurrence) into Tp.
//   GEMM  X = A22 V                 (A22 = K[r0:, r0:], full symmetric storage; tcgen05)
//   sbr_w_kernel      Y = X T,  W = Y - 1/2 V (T^T (V^T Y))
//   GEMM  A22 -= V W^T + W V^T      (symmetric: lower tiles computed and mirrored; tcgen05)
// which is the two-sided block update Q^T A22 Q = A22 - V W^T - W V^T.  All O(m^3) work of
// the reduction is in the two GEMMs per panel: m / 32 synchronisation points instead of m.
//
// Stage 2, band -> tridiagonal (sbr_chase_kernel, one CTA per problem): bulge chasing.
// Sweep j annihilates column j below the subdiagonal (task 0: reflector on rows j+1 ..
// j+32, applied two-sidedly to that diagonal block); task k >= 1 right-applies the
// previous reflector to the block below (rows R_k = [j+1+32k, +32), columns R_{k-1}),
// which fills it, computes a reflector from its first column, applies it from the left and
// two-sidedly to the diagonal block R_k.  The fill beyond the band (at most 2b - 1 below the
// diagonal) is removed by the following sweeps.  One warp per sweep (lane = row of the
// 32-row block), sweeps pipelined over the CTA's warps: task (j, k) starts once sweep j - 1
// has finished task k + 1 (the last task whose rows meet those of (j, k)).  The band with
// its bulge space (2b diagonals) lives in global memory (L2-resident; ld/st.cg).
//
// Back-transform V = Q1 Q2 Y of the tridiagonal's eigenvectors Y (eig.cuh 2-4):
//   sbr_q2_kernel  applies the chase reflectors: in reverse order, grouped into "diamonds"
//                  (the reflectors of 32 consecutive sweeps at the same task index touch a
//                  63-row window, applied in one pass with the window in registers, lane =
//                  eigenvector column; diamonds run group by group, last group first, task
//                  index ascending inside a group -- the order the overlaps require).
//   then the blocked compact-WY back-transform of eig.cuh with reflector offset 32 (Q1).
#pragma once
#include "common.cuh"
#include "eig.cuh"

namespace bkfac {

constexpr int SBR_B = 32;                 // band width (= warp size: lane = row of a block)
constexpr int SBR_LDB = 2 * SBR_B;        // band storage: diagonals 0 .. 2b-1 (bulge included)
#ifndef BKFAC_PANEL_THREADS
#define BKFAC_PANEL_THREADS 512
#endif
constexpr int SBR_PANEL_THREADS = BKFAC_PANEL_THREADS;
constexpr int SBR_W_WARPS = 16;
#ifndef BKFAC_CHASE_WARPS
#define BKFAC_CHASE_WARPS 16
#endif
constexpr int SBR_CHASE_WARPS = BKFAC_CHASE_WARPS;
#ifndef BKFAC_SBR_G
#define BKFAC_SBR_G 32
#endif
constexpr int SBR_G = BKFAC_SBR_G;        // sweeps per diamond
constexpr int SBR_MAX_L = 1600;           // panel rows held in shared memory (m <= 1632)

__host__ __device__ inline int sbr_panels(int m) { return m - 2 >= SBR_B ? (m - 2) / SBR_B : 0; }
__host__ __device__ inline int sbr_tasks(int m) { return (m + SBR_B - 1) / SBR_B + 1; }   // KT
inline bool sbr_supported(int m) { return m - SBR_B <= SBR_MAX_L && sbr_panels(m) > 0; }
inline size_t sbr_panel_smem_bytes(int m) {
  return sizeof(float) * ((size_t)(m - SBR_B) * (SBR_B + 1) + SBR_B * (SBR_B + 1) +
                          2 * (SBR_PANEL_THREADS / 32) * SBR_B + 3 * SBR_B);
}
inline size_t sbr_w_smem_bytes() {
  return sizeof(float) * (3 * SBR_B * (SBR_B + 1) + SBR_W_WARPS * 3 * SBR_B * (SBR_B + 1));
}
inline size_t sbr_chase_smem_bytes() {
  return sizeof(float) * SBR_CHASE_WARPS * (2 * SBR_B * (SBR_B + 1) + 3 * SBR_B) + 64 * sizeof(int);
}

// ---------------------------------------------------------------------- stage 1: panel QR
// grid (nprob), block SBR_PANEL_THREADS; panel j of every problem that has one.
// The panel lives row-major in shared memory (row l at P[l * 33], conflict-free for a thread
// walking its own row); thread t owns rows t, t + 512, ...  Column step i needs one block
// barrier: every thread forms, over its rows below i, the 32 partial sums
//   value[i] = sum x_l^2,  value[c] = sum x_l P(l, c) (c > i),  value[a] = sum x_l V(l, a) (a < i)
// (x = column i), reduced across the warp by a 31-shuffle transpose-reduce (lane c ends with
// value[c]) and across warps through shared memory (double-buffered by step parity); then
// every thread has beta, tau, the update coefficients w_c = tau (P(i, c) + s_c / (alpha -
// beta)) and applies the reflector to its own rows, warp 0 extends T (dlarft:
// T(0:i, i) = -tau T(0:i, 0:i) g, g_a = V(i, a) + u_a / (alpha - beta)), and the owner of
// row i + 1 publishes that row for the next step.
BKFAC_DEV float sbr_transpose_reduce(float (&v)[32], int lane) {
  // after the 5 rounds lane c holds sum over the warp of v[c]
#pragma unroll
  for (int h = 16; h >= 1; h >>= 1) {
    const bool upper = (lane & h) != 0;
#pragma unroll
    for (int q = 0; q < h; ++q) {
      // keep half of the 2h values: lanes with bit h set keep the upper half
      const float send = upper ? v[q] : v[q + h];
      const float keep = upper ? v[q + h] : v[q];
      v[q] = keep + __shfl_xor_sync(0xffffffffu, send, h);
    }
  }
  return v[0];
}

#if defined(BKFAC_CHASE_TIMING) || defined(BKFAC_Q2_TIMING) || defined(BKFAC_PANEL_TIMING)
__device__ unsigned long long g_chase_dbg[8];   // tuning builds: phase cycle sums
#endif
#ifdef BKFAC_PANEL_TIMING
#define PN_T(x) const unsigned long long x = clock64()
#define PN_ACC(k, a, b) if (blockIdx.x == 0 && tid == 0) atomicAdd(&g_chase_dbg[k], (b) - (a))
#else
#define PN_T(x)
#define PN_ACC(k, a, b)
#endif
__global__ void __launch_bounds__(SBR_PANEL_THREADS, 1)
sbr_panel_kernel(const __grid_constant__ EigBatch b, int j) {
  const EigProb& p = b.p[blockIdx.x];
  const int m = p.m, ld = p.ldk;
  if (p.sbr == 0 || j >= sbr_panels(m)) return;
  constexpr int B = SBR_B, NT = SBR_PANEL_THREADS, NW = NT / 32, LDP = B + 1, LDT = B + 1;
  const int c0 = j * B, r0 = c0 + B, L = m - r0;
  extern __shared__ __align__(16) float ps[];
  float* P = ps;                          // L x B row-major, ld 33
  float* T = P + (size_t)L * LDP;         // B x B upper triangular, T[a*LDT + c]
  float* red = T + B * LDT;               // [2][NW][B] partial sums by step parity
  float* rowb = red + 2 * NW * B;         // [2][B] row i of the panel by step parity
  float* taus = rowb + 2 * B;             // B
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float* K = p.K;
  {   // the panel into shared memory: every element's copy in flight at once (cp.async)
    const uint32_t pb = (uint32_t)__cvta_generic_to_shared(P);
    for (int e = tid; e < L * B; e += NT) {
      const int l = e % L, i = e / L;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(pb + 4u * (uint32_t)(l * LDP + i)),
                   "l"(K + (r0 + l) + (long)(c0 + i) * ld) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int e = tid; e < B * LDT; e += NT) T[e] = 0.f;
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  if (tid < B) rowb[tid] = P[tid];        // row 0 for step 0
  __syncthreads();
  for (int i = 0; i < B; ++i) {
    const int par = i & 1;
    PN_T(pa);
    // ---- partial sums over this thread's rows l > i
    float v[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) v[c] = 0.f;
    for (int l = tid; l < L; l += NT) {
      if (l <= i) continue;
      const float* pr = P + l * LDP;
      const float x = pr[i];
#pragma unroll
      for (int c = 0; c < 32; ++c) v[c] = fmaf(x, c == i ? x : pr[c], v[c]);
    }
    const float mine = sbr_transpose_reduce(v, lane);   // lane c: warp total of value[c]
    red[(par * NW + warp) * B + lane] = mine;
    PN_T(pb);
    __syncthreads();
    PN_T(pc);
    float tot = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) tot += red[(par * NW + w) * B + lane];
    // lane c of every warp: value[c] (c == i: ||x||^2 below row i; c > i: s_c; c < i: u_c)
    const float xn2 = __shfl_sync(0xffffffffu, tot, i);
    const float* ri = rowb + par * B;     // row i (published by its owner before the barrier)
    const float alpha = ri[i];
    float tau = 0.f, beta = alpha, sc = 0.f;
    if (L - i > 1 && xn2 > 0.f && i < L) {
      beta = -copysignf(sqrtf(fmaf(alpha, alpha, xn2)), alpha);
      tau = (beta - alpha) / beta;
      sc = 1.f / (alpha - beta);
    }
    // w_c = tau (P(i, c) + s_c sc) for c > i (lane c)
    const float wc = (lane > i) ? tau * fmaf(tot, sc, ri[lane]) : 0.f;
    // T column i (warp 0): g_a = V(i, a) + u_a sc, a < i
    if (warp == 0) {
      const float g = (lane < i) ? fmaf(tot, sc, ri[lane]) : 0.f;
      float tcol = 0.f;
      for (int e = 0; e < i; ++e) {
        const float ge = __shfl_sync(0xffffffffu, g, e);
        if (lane <= e) tcol = fmaf(T[lane * LDT + e], ge, tcol);
      }
      if (lane < i) T[lane * LDT + i] = -tau * tcol;
      if (lane == i) { T[i * LDT + i] = tau; taus[i] = tau; }
    }
    PN_T(pd);
    // ---- apply H_i to this thread's rows (scale x into v, update the later columns)
    float wl[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) wl[c] = __shfl_sync(0xffffffffu, wc, c);
    for (int l = tid; l < L; l += NT) {
      if (l < i) continue;
      float* pr = P + l * LDP;
      if (l == i) {
        if (tau != 0.f) {
          pr[i] = beta;
#pragma unroll
          for (int c = 0; c < 32; ++c) if (c > i) pr[c] -= wl[c];
        }
      } else if (tau != 0.f) {
        const float vx = pr[i] * sc;
        pr[i] = vx;
#pragma unroll
        for (int c = 0; c < 32; ++c) if (c > i) pr[c] = fmaf(-wl[c], vx, pr[c]);
      }
    }
    // publish row i + 1 (after this step's update) for the next step: its owner's warp copies
    // it lane by lane (one element each) instead of the owner alone, 32 copies in a row
    if (i + 1 < L && warp == ((i + 1) % NT) >> 5) {
      __syncwarp();
      rowb[(par ^ 1) * B + lane] = P[(i + 1) * LDP + lane];
    }
    PN_T(pe);
    PN_ACC(0, pa, pb); PN_ACC(1, pb, pc); PN_ACC(2, pc, pd); PN_ACC(3, pd, pe);
    if (blockIdx.x == 0 && tid == 0) { PN_ACC(5, 0ull, 1ull); }
#ifdef BKFAC_PANEL_TIMING
    if (blockIdx.x == 0 && tid == 256) {   // a warp without the T column
      atomicAdd(&g_chase_dbg[7], pb - pa); atomicAdd(&g_chase_dbg[6], pc - pb); atomicAdd(&g_chase_dbg[4], pe - pd);
    }
#endif
  }
  __syncthreads();
  // write back: K panel (R above / on the diagonal, reflector tails below), explicit V, T, tau
  for (int e = tid; e < L * B; e += NT) {
    const int l = e % L, i = e / L;
    const float x = P[l * LDP + i];
    K[(r0 + l) + (long)(c0 + i) * ld] = x;
    p.Vp[(r0 + l) + (long)i * m] = (l < i) ? 0.f : (l == i ? 1.f : x);
  }
  for (int e = tid; e < L * B; e += NT) {   // row-major copy for the X and update kernels' tiles
    const int l = e / B, i = e % B;
    p.Vt[(long)(r0 + l) * B + i] = (l < i) ? 0.f : (l == i ? 1.f : P[l * LDP + i]);
  }
  for (int e = tid; e < B * B; e += NT) {
    const int a = e % B, c = e / B;
    p.Tp[a + c * B] = T[a * LDT + c];
  }
  if (tid < B) p.tau[c0 + tid] = taus[tid];
}

// ---------------------------------------------------------------------- stage 1: W
// grid (nprob), block SBR_W_WARPS*32:  Y = X T;  Z = V^T Y;  M2 = T^T Z;  W = Y - 1/2 V M2
// (rows r0 .. m-1 of the m x B buffers Xp, Vp, Wp, col-major ld m).  Each warp walks 32-row
// blocks staged through shared memory (coalesced loads, lane = column in the arithmetic).
__global__ void __launch_bounds__(SBR_W_WARPS * 32)
sbr_w_kernel(const __grid_constant__ EigBatch b, int j) {
  const EigProb& p = b.p[blockIdx.x];
  const int m = p.m;
  if (p.sbr == 0 || j >= sbr_panels(m)) return;
  constexpr int B = SBR_B, LDT = B + 1, NW = SBR_W_WARPS;
  const int r0 = (j + 1) * B, L = m - r0;
  extern __shared__ __align__(16) float wsm[];
  float* T = wsm;                    // T[a*LDT + c]
  float* Zs = T + B * LDT;           // Z, then M2 (in place after a sync)
  float* M2 = Zs + B * LDT;
  float* tiles = M2 + B * LDT;       // per warp: xs, vs, ys (B x LDT each); also the Z reduction
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float* xs = tiles + warp * 3 * B * LDT;
  float* vs = xs + B * LDT;
  float* ys = vs + B * LDT;
  for (int e = tid; e < B * B; e += NW * 32) {
    const int a = e % B, c = e / B;
    T[a * LDT + c] = p.Tp[a + c * B];
  }
  __syncthreads();
  const float* X = p.Xp;
  const float* V = p.Vp;
  float* W = p.Wp;
  float zacc[B];
#pragma unroll
  for (int a = 0; a < B; ++a) zacc[a] = 0.f;
  const int nblk = (L + B - 1) / B;
  for (int blk = warp; blk < nblk; blk += NW) {
    const int rb = r0 + blk * B;
    const bool ok = rb + lane < m;
#pragma unroll 4
    for (int a = 0; a < B; ++a) {
      xs[lane * LDT + a] = ok ? X[(rb + lane) + (long)a * m] : 0.f;
      vs[lane * LDT + a] = ok ? V[(rb + lane) + (long)a * m] : 0.f;
    }
    __syncwarp();
    for (int i = 0; i < B; ++i) {
      float y = 0.f;
#pragma unroll
      for (int a = 0; a < B; ++a) y = fmaf(xs[i * LDT + a], T[a * LDT + lane], y);
      ys[i * LDT + lane] = y;
#pragma unroll
      for (int a = 0; a < B; ++a) zacc[a] = fmaf(vs[i * LDT + a], y, zacc[a]);
    }
    __syncwarp();
#pragma unroll 4
    for (int a = 0; a < B; ++a)
      if (ok) W[(rb + lane) + (long)a * m] = ys[lane * LDT + a];   // Y, finished below
    __syncwarp();
  }
  __syncthreads();
  // Z = sum over warps (reduction space: the tiles)
  float* zr = tiles;                 // [NW][B][LDT]
#pragma unroll
  for (int a = 0; a < B; ++a) zr[(warp * B + a) * LDT + lane] = zacc[a];
  __syncthreads();
  for (int e = tid; e < B * B; e += NW * 32) {
    const int a = e / B, c = e % B;
    float s = 0.f;
    for (int w = 0; w < NW; ++w) s += zr[(w * B + a) * LDT + c];
    Zs[a * LDT + c] = s;
  }
  __syncthreads();
  for (int e = tid; e < B * B; e += NW * 32) {    // M2 = T^T Z  (T upper: e <= a)
    const int a = e / B, c = e % B;
    float s = 0.f;
    for (int q = 0; q <= a; ++q) s = fmaf(T[q * LDT + a], Zs[q * LDT + c], s);
    M2[a * LDT + c] = 0.5f * s;
  }
  __syncthreads();
  for (int blk = warp; blk < nblk; blk += NW) {
    const int rb = r0 + blk * B;
    const bool ok = rb + lane < m;
#pragma unroll 4
    for (int a = 0; a < B; ++a) {
      ys[lane * LDT + a] = ok ? W[(rb + lane) + (long)a * m] : 0.f;
      vs[lane * LDT + a] = ok ? V[(rb + lane) + (long)a * m] : 0.f;
    }
    __syncwarp();
    for (int i = 0; i < B; ++i) {
      float w = ys[i * LDT + lane];
#pragma unroll
      for (int a = 0; a < B; ++a) w = fmaf(-vs[i * LDT + a], M2[a * LDT + lane], w);
      xs[i * LDT + lane] = w;
    }
    __syncwarp();
#pragma unroll 4
    for (int a = 0; a < B; ++a)
      if (ok) W[(rb + lane) + (long)a * m] = xs[lane * LDT + a];
#pragma unroll 4
    for (int i = 0; i < B; ++i)   // row-major copy for the update kernel's tiles
      if (rb + i < m) p.Wt[(long)(rb + i) * B + lane] = xs[i * LDT + lane];
    __syncwarp();
  }
}

// ---------------------------------------------------------------------- stage 1: X = A22 V
// grid (row blocks of SBR_X_ROWS, nprob), block SBR_X_THREADS.  Only the lower triangle of
// A22 is kept current (the block update writes lower tiles only), so element (i, k) of the
// symmetric A22 is read from K(i, k) when i >= k and from K(k, i) otherwise.  The CTA walks
// the 32-deep k tiles of its 128 rows through a SBR_X_STAGES-deep cp.async ring (the next
// tiles in flight while one is multiplied, no staging registers):
//   below the diagonal  16-byte copies along i (4 rows of a stored column): As[k][i], pitch 136;
//   above it            16-byte copies along k (4 k of a stored column i, the stored block
//                       read transposed): At[i][k], pitch 36;
//   crossing it         4-byte copies into At, each element by the pattern that reads it
//                       from the lower triangle; zero-filled out of range;
//   V                   16-byte copies of the row-major V tile (Vt, written by the panel
//                       kernel): Vs[k][c], pitch 40.
// (pitches: every fragment load below is bank-conflict-free).  The products run on the
// warp-level tensor-core MMA (mma.sync m16n8k8 tf32) in 3xTF32 -- hi = rna_tf32(x), lo = x -
// hi, hi_A lo_B + lo_A hi_B + hi_A hi_B, the split done in registers -- each warp 32 rows x 32
// columns; every k tile is accumulated in fresh fragments and added into a running fp32 sum
// (round-to-nearest FADDs: the MMA accumulate's bias stays bounded by 32 terms, as the
// tcgen05 GEMM's promotion does).  Measured on configs[4]: the CUDA-core FFMA2 version (8 x 8
// register tiles) was bound by the FMA pipes at 6.4 ms per step for the products alone (the
// 3-register FFMA/FFMA2 issue at half the nominal FP32 rate); the tcgen05 GEMM reached 1.6
// TB/s here (its loaders' memory parallelism); one 1-D bulk copy (cp.async.bulk) per 512- /
// 128-byte run made the loads alone 10.3 ms (the copy engine's per-copy cost).
#ifndef BKFAC_SBRX_STAGES
#define BKFAC_SBRX_STAGES 2   // 2 stages, 4 CTAs per SM: 6.45 ms per configs[4] step (3: 6.94, 4: 7.11)
#endif
constexpr int SBR_X_ROWS = 128, SBR_X_THREADS = 128, SBR_X_STAGES = BKFAC_SBRX_STAGES;
constexpr int SBR_X_LDK = 136, SBR_X_LDT = 36, SBR_X_LDV = 40;
constexpr int SBR_X_A_FLOATS = SBR_X_ROWS * SBR_X_LDT;                  // >= 32 x 136
constexpr int SBR_X_STAGE_FLOATS = SBR_X_A_FLOATS + SBR_B * SBR_X_LDV;   // + the V tile
inline size_t sbr_x_smem_bytes() { return sizeof(float) * SBR_X_STAGES * SBR_X_STAGE_FLOATS; }
// the epilogue's X, T and V tiles reuse the ring
static_assert(SBR_X_STAGES * SBR_X_STAGE_FLOATS >= SBR_X_ROWS * 36 + SBR_B * 40 + SBR_X_ROWS * 40, "sbr_x epilogue");
BKFAC_DEV void sbr_cp4(uint32_t dst, const float* src, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(ok ? 4 : 0) : "memory");
}
BKFAC_DEV void sbr_cp16(uint32_t dst, const float* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0) : "memory");
}
// x = hi + lo, hi = rna_tf32(x) (bit pattern), lo = x - hi (exact; the MMA truncates it to tf32)
BKFAC_DEV void sbr_split(float x, uint32_t& hi, uint32_t& lo) {
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi) : "f"(x));
  lo = __float_as_uint(x - __uint_as_float(hi));
}
BKFAC_DEV void sbr_mma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// one 32-deep k tile of the warp's 32 x 32 block: acc += A(rows, k) V(k, :) in 3xTF32.
// KMAJOR: A(i, k) at a[k * LDK + i], else at a[i * LDT + k]; rb = the warp's first row.
template <bool KMAJOR>
BKFAC_DEV void sbr_x_tile(const float* a, const float* vs, int rb, int g, int t, float (&acc)[2][4][4]) {
  constexpr int LDK = SBR_X_LDK, LDT = SBR_X_LDT, LDV = SBR_X_LDV;
  auto A = [&](int i, int k) { return KMAJOR ? a[k * LDK + i] : a[i * LDT + k]; };
#pragma unroll
  for (int ks = 0; ks < SBR_B / 8; ++ks) {
    const int kb = ks * 8;
    uint32_t ah[2][4], al[2][4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int i = rb + 16 * mt + g;
      sbr_split(A(i, kb + t), ah[mt][0], al[mt][0]);
      sbr_split(A(i + 8, kb + t), ah[mt][1], al[mt][1]);
      sbr_split(A(i, kb + t + 4), ah[mt][2], al[mt][2]);
      sbr_split(A(i + 8, kb + t + 4), ah[mt][3], al[mt][3]);
    }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      uint32_t bh0, bl0, bh1, bl1;
      sbr_split(vs[(kb + t) * LDV + 8 * nt + g], bh0, bl0);
      sbr_split(vs[(kb + t + 4) * LDV + 8 * nt + g], bh1, bl1);
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {   // small terms first
        sbr_mma(acc[mt][nt], al[mt], bh0, bh1);
        sbr_mma(acc[mt][nt], ah[mt], bl0, bl1);
        sbr_mma(acc[mt][nt], ah[mt], bh0, bh1);
      }
    }
  }
}

__global__ void __launch_bounds__(SBR_X_THREADS)
sbr_x_kernel(const __grid_constant__ EigBatch b, int j) {
  const EigProb& p = b.p[blockIdx.y];
  const int m = p.m;
  if (p.sbr == 0 || j >= sbr_panels(m)) return;
  constexpr int B = SBR_B, R = SBR_X_ROWS, NT = SBR_X_THREADS, S = SBR_X_STAGES;
  constexpr int LDK = SBR_X_LDK, LDT = SBR_X_LDT, LDV = SBR_X_LDV;
  const int r0 = (j + 1) * B, L = m - r0;
  const int i0 = blockIdx.x * R;
  if (i0 >= L) return;
  const long ld = p.ldk;
  const float* A = p.K + r0 + (long)r0 * ld;     // stored lower triangle: A22(i, k) = A[i + k ld], i >= k
  const float* Vt = p.Vt + (long)r0 * B;         // V(k, c) = Vt[k B + c]
  extern __shared__ __align__(16) float xsm[];
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(xsm);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // whole 16-byte runs: the leading dimension (and with it L = m - r0) a multiple of 4 floats
  const bool vec = (ld & 3) == 0 && (m & 3) == 0 && (reinterpret_cast<uintptr_t>(p.K) & 15) == 0;
  const bool vvec = (reinterpret_cast<uintptr_t>(p.Vt) & 15) == 0;
  const int nkt = (L + B - 1) / B;
  auto region = [&](int kt) {   // 0 below the diagonal, 1 above, 2 crossing (or unaligned)
    const int k0 = kt * B;
    if (!vec) return 2;
    return (i0 >= k0 + B - 1) ? 0 : (k0 > i0 + R - 1) ? 1 : 2;
  };
  auto issue = [&](int kt) {           // copies of k tile kt into its stage (one commit group)
#ifndef BKFAC_SBRX_NOLOAD
    if (kt < nkt) {
#else
    if (false) {
#endif
      const int k0 = kt * B;
      const uint32_t as = sbase + 4u * (uint32_t)((kt % S) * SBR_X_STAGE_FLOATS);
      const uint32_t vs = as + 4u * (uint32_t)SBR_X_A_FLOATS;
      const int reg = region(kt);
      if (reg == 0) {          // As[k][i]: 4 consecutive rows of stored column k per copy
#pragma unroll
        for (int u = 0; u < B * R / 4 / NT; ++u) {
          const int q = tid + NT * u, k = q / (R / 4), i = (q % (R / 4)) * 4;
          const int gi = i0 + i, gk = k0 + k;
          const bool ok = gi < L && gk < L;
          sbr_cp16(as + 4u * (uint32_t)(k * LDK + i), ok ? A + gi + (long)gk * ld : A, ok);
        }
      } else if (reg == 1) {   // At[i][k]: 4 consecutive k of stored column i per copy
#pragma unroll
        for (int u = 0; u < B * R / 4 / NT; ++u) {
          const int q = tid + NT * u, i = q / (B / 4), k = (q % (B / 4)) * 4;
          const int gi = i0 + i, gk = k0 + k;
          const bool ok = gi < L && gk < L;
          sbr_cp16(as + 4u * (uint32_t)(i * LDT + k), ok ? A + gk + (long)gi * ld : A, ok);
        }
      } else {                 // At[i][k], element by element from the lower triangle
        for (int e = tid; e < B * R; e += NT) {
          const int i = e % R, k = e / R;
          const int gi = i0 + i, gk = k0 + k;
          const bool ok = gi < L && gk < L;
          const float* src = !ok ? A : (gi >= gk ? A + gi + (long)gk * ld : A + gk + (long)gi * ld);
          sbr_cp4(as + 4u * (uint32_t)(i * LDT + k), src, ok);
        }
      }
      // V tile: row k of Vt is 32 contiguous floats (zero-filled beyond L)
#pragma unroll
      for (int u = 0; u < B * B / 4 / NT; ++u) {
        const int q = tid + NT * u, k = q / (B / 4), c = (q % (B / 4)) * 4;
        const bool ok = k0 + k < L;
        const float* src = ok ? Vt + (long)(k0 + k) * B + c : Vt;
        const uint32_t d = vs + 4u * (uint32_t)(k * LDV + c);
        if (vvec) {
          sbr_cp16(d, src, ok);
        } else {
#pragma unroll
          for (int t = 0; t < 4; ++t) sbr_cp4(d + 4u * t, ok ? src + t : Vt, ok);
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");   // (possibly empty) group per tile
  };
  const int g = lane >> 2, t = lane & 3, rb = warp * 32;   // warp w: rows 32w .. 32w+31, all 32 columns
  float sum[2][4][4];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int q = 0; q < 4; ++q) sum[mt][nt][q] = 0.f;
#pragma unroll
  for (int u = 0; u < S - 1; ++u) issue(u);
  for (int kt = 0; kt < nkt; ++kt) {
    asm volatile("cp.async.wait_group %0;" ::"n"(S - 2) : "memory");   // tile kt's copies (own)
    __syncthreads();   // ... everyone's; and every thread is done with tile kt - 1's stage
    issue(kt + S - 1);
    const float* as = xsm + (kt % S) * SBR_X_STAGE_FLOATS;
    const float* vs = as + SBR_X_A_FLOATS;
#ifndef BKFAC_SBRX_NOCOMP
    float acc[2][4][4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[mt][nt][q] = 0.f;
    if (region(kt) == 0) sbr_x_tile<true>(as, vs, rb, g, t, acc);
    else sbr_x_tile<false>(as, vs, rb, g, t, acc);
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int q = 0; q < 4; ++q) sum[mt][nt][q] += acc[mt][nt][q];
#endif
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();   // the ring is free: the epilogue's tiles below reuse it
  // ---- epilogue: X block -> Y = X T (rows of W before its correction, into Wt) and this row
  // block's share of Z = V^T Y (into Zp); sbr_wfin_kernel sums the shares and finishes W
  float* Xs = xsm;                       // X block, [128][36]
  float* Ts = xsm + R * 36;              // T, [32][40]: Ts[a * 40 + c] = T(a, c)
  float* Vs2 = Ts + B * 40;              // V rows of the block, [128][40]
  float* Ys = xsm;                       // Y block, [128][40] (after Xs, Ts are consumed)
  float* Zr = Vs2;                       // per-warp Z shares, [4][32][32] (after Vs2 is consumed)
  float* X = p.Xp + r0;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int li = rb + 16 * mt + g + 8 * h, gi = i0 + li;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int c = 8 * nt + 2 * t;
        Xs[li * 36 + c] = sum[mt][nt][2 * h];
        Xs[li * 36 + c + 1] = sum[mt][nt][2 * h + 1];
        if (gi < L) {
          X[gi + (long)c * m] = sum[mt][nt][2 * h];
          X[gi + (long)(c + 1) * m] = sum[mt][nt][2 * h + 1];
        }
      }
    }
  for (int e = tid; e < B * B; e += NT) Ts[(e % B) * 40 + e / B] = p.Tp[e];   // Tp[a + c B] = T(a, c)
  for (int e = tid; e < R * B; e += NT) {
    const int i = e / B, a = e % B;
    Vs2[i * 40 + a] = (i0 + i < L) ? Vt[(long)(i0 + i) * B + a] : 0.f;
  }
  __syncthreads();
  float y[2][4][4];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int q = 0; q < 4; ++q) y[mt][nt][q] = 0.f;
#pragma unroll
  for (int ks = 0; ks < B / 8; ++ks) {   // Y = X T
    const int kb = ks * 8;
    uint32_t ah[2][4], al[2][4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const float* ar = Xs + (rb + 16 * mt + g) * 36 + kb + t;
      sbr_split(ar[0], ah[mt][0], al[mt][0]);
      sbr_split(ar[8 * 36], ah[mt][1], al[mt][1]);
      sbr_split(ar[4], ah[mt][2], al[mt][2]);
      sbr_split(ar[8 * 36 + 4], ah[mt][3], al[mt][3]);
    }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      uint32_t bh0, bl0, bh1, bl1;
      sbr_split(Ts[(kb + t) * 40 + 8 * nt + g], bh0, bl0);
      sbr_split(Ts[(kb + t + 4) * 40 + 8 * nt + g], bh1, bl1);
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        sbr_mma(y[mt][nt], al[mt], bh0, bh1);
        sbr_mma(y[mt][nt], ah[mt], bl0, bl1);
        sbr_mma(y[mt][nt], ah[mt], bh0, bh1);
      }
    }
  }
  __syncthreads();   // Xs, Ts consumed
  float* Yg = p.Wt + (long)r0 * B;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int li = rb + 16 * mt + g + 8 * h, gi = i0 + li;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int c = 8 * nt + 2 * t;
        Ys[li * 40 + c] = y[mt][nt][2 * h];
        Ys[li * 40 + c + 1] = y[mt][nt][2 * h + 1];
        if (gi < L) *reinterpret_cast<float2*>(Yg + (long)gi * B + c) = make_float2(y[mt][nt][2 * h], y[mt][nt][2 * h + 1]);
      }
    }
  __syncthreads();
  float z[2][4][4];   // this warp's rows' share: Z(a, c) += sum_i V(i, a) Y(i, c)
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int q = 0; q < 4; ++q) z[mt][nt][q] = 0.f;
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const int kb = rb + ks * 8;      // rows of the block = the contraction index
    uint32_t ah[2][4], al[2][4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {  // A(a, i) = V(i, a)
      const float* ar = Vs2 + (kb + t) * 40 + 16 * mt + g;
      sbr_split(ar[0], ah[mt][0], al[mt][0]);
      sbr_split(ar[8], ah[mt][1], al[mt][1]);
      sbr_split(ar[4 * 40], ah[mt][2], al[mt][2]);
      sbr_split(ar[4 * 40 + 8], ah[mt][3], al[mt][3]);
    }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      uint32_t bh0, bl0, bh1, bl1;
      sbr_split(Ys[(kb + t) * 40 + 8 * nt + g], bh0, bl0);
      sbr_split(Ys[(kb + t + 4) * 40 + 8 * nt + g], bh1, bl1);
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        sbr_mma(z[mt][nt], al[mt], bh0, bh1);
        sbr_mma(z[mt][nt], ah[mt], bl0, bl1);
        sbr_mma(z[mt][nt], ah[mt], bh0, bh1);
      }
    }
  }
  __syncthreads();   // Vs2 consumed
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        Zr[warp * B * B + (16 * mt + g + 8 * (q >> 1)) * B + 8 * nt + 2 * t + (q & 1)] = z[mt][nt][q];
  __syncthreads();
  float* Zp = p.Zp + (long)blockIdx.x * B * B;
  for (int e = tid; e < B * B; e += NT) {
    float a = 0.f;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) a += Zr[w * B * B + e];
    Zp[e] = a;
  }
}

// ---------------------------------------------------------------------- stage 1: W (finish)
// grid (row blocks of SBR_X_ROWS, nprob), block SBR_X_ROWS threads (thread = row).  With
// Y = X T in Wt and the row blocks' shares of Z = V^T Y in Zp (sbr_x_kernel's epilogue):
// Z = sum of the shares (fixed order), M2 = 1/2 T^T Z, W = Y - V M2 for this block's rows.
__global__ void __launch_bounds__(SBR_X_ROWS)
sbr_wfin_kernel(const __grid_constant__ EigBatch b, int j) {
  const EigProb& p = b.p[blockIdx.y];
  const int m = p.m;
  if (p.sbr == 0 || j >= sbr_panels(m)) return;
  constexpr int B = SBR_B, R = SBR_X_ROWS, LDT = B + 1;
  const int r0 = (j + 1) * B, L = m - r0;
  const int i0 = blockIdx.x * R, nrb = (L + R - 1) / R;
  if (i0 >= L) return;
  __shared__ float Z[B * LDT], T[B * LDT], M2[B * LDT], Ws[R * LDT];
  const int tid = threadIdx.x;
  for (int e = tid; e < B * B; e += R) {
    // the shares' loads issued together (at most NQ row blocks), then summed in order
    constexpr int NQ = (SBR_MAX_L + SBR_B + SBR_X_ROWS - 1) / SBR_X_ROWS;
    float zq[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) zq[q] = q < nrb ? p.Zp[(long)q * B * B + e] : 0.f;
    float a = 0.f;
#pragma unroll
    for (int q = 0; q < NQ; ++q) if (q < nrb) a += zq[q];
    Z[(e / B) * LDT + e % B] = a;                        // Z(a, c) at Z[a LDT + c]
    T[(e % B) * LDT + e / B] = p.Tp[e];                  // T(a, c) at T[a LDT + c]
  }
  __syncthreads();
  for (int e = tid; e < B * B; e += R) {                 // M2 = 1/2 T^T Z  (T upper: q <= a)
    const int a = e / B, c = e % B;
    float s = 0.f;
    for (int q = 0; q <= a; ++q) s = fmaf(T[q * LDT + a], Z[q * LDT + c], s);
    M2[a * LDT + c] = 0.5f * s;
  }
  __syncthreads();
  const int i = i0 + tid;
  float* Wt = p.Wt + (long)r0 * B;
  const float* Vt = p.Vt + (long)r0 * B;
  if (i < L) {
    float v[B], y[B];   // this row of V and of Y, loaded together
#pragma unroll
    for (int a4 = 0; a4 < B / 4; ++a4) {
      const float4 q = *reinterpret_cast<const float4*>(Vt + (long)i * B + 4 * a4);
      v[4 * a4] = q.x; v[4 * a4 + 1] = q.y; v[4 * a4 + 2] = q.z; v[4 * a4 + 3] = q.w;
      const float4 u = *reinterpret_cast<const float4*>(Wt + (long)i * B + 4 * a4);
      y[4 * a4] = u.x; y[4 * a4 + 1] = u.y; y[4 * a4 + 2] = u.z; y[4 * a4 + 3] = u.w;
    }
#pragma unroll
    for (int c = 0; c < B; ++c) {
      float w = y[c];
#pragma unroll
      for (int a = 0; a < B; ++a) w = fmaf(-v[a], M2[a * LDT + c], w);
      Ws[tid * LDT + c] = w;
    }
  }
  __syncthreads();
  for (int e = tid; e < R * B; e += R) {                 // coalesced write-back of the block's W rows
    const int li = e / B, c = e % B;
    if (i0 + li < L) Wt[(long)(i0 + li) * B + c] = Ws[li * LDT + c];
  }
}

// ---------------------------------------------------------------------- stage 1: block update
// grid (lower tiles of the largest A22, nprob), block SBR_U_THREADS:
//   A22 -= V W^T + W V^T = C0 - [V_I W_I] [W_J V_J]^T      (K = 64)
// on the 128 x 128 tiles (I, J), I >= J, of the lower triangle only -- the upper triangle is
// never read again (X, the panels and the band extraction read the lower one); on a diagonal
// tile the elements above the diagonal are computed and not stored.  Operands: the four
// 128 x 32 row-major blocks V_I, W_I, W_J, V_J (Vt from the panel kernel, Wt from the W
// kernel) by 16-byte cp.async into [128][64] tiles of pitch 68 (conflict-free fragment
// loads); products on mma.sync m16n8k8 tf32 in 3xTF32 (split in registers), warp tile 32 x 64;
// C0 is prefetched into L2 while the operands land and read per fragment after the MMAs.
// Replaces the tcgen05 GEMM with a lower-tile epilogue, whose C0 read + C write streamed at
// 1.2 TB/s (its 8 epilogue warps keep 16 KB in flight per SM).
constexpr int SBR_U_TILE = 128, SBR_U_THREADS = 256, SBR_U_LD = 68;
inline size_t sbr_u_smem_bytes() { return sizeof(float) * 2 * SBR_U_TILE * SBR_U_LD; }
__host__ __device__ inline int sbr_u_tiles(int L) { const int t = (L + SBR_U_TILE - 1) / SBR_U_TILE; return t * (t + 1) / 2; }

__global__ void __launch_bounds__(SBR_U_THREADS, 2)
sbr_update_kernel(const __grid_constant__ EigBatch b, int j) {
  const EigProb& p = b.p[blockIdx.y];
  const int m = p.m;
  if (p.sbr == 0 || j >= sbr_panels(m)) return;
  constexpr int B = SBR_B, T = SBR_U_TILE, NT = SBR_U_THREADS, LD = SBR_U_LD;
  const int r0 = (j + 1) * B, L = m - r0;
  const int tix = blockIdx.x;
  if (tix >= sbr_u_tiles(L)) return;
  int ti = (int)((sqrtf(8.f * tix + 1.f) - 1.f) * 0.5f);   // tix = ti (ti + 1) / 2 + tj, tj <= ti
  while (ti * (ti + 1) / 2 > tix) --ti;
  while ((ti + 1) * (ti + 2) / 2 <= tix) ++ti;
  const int tj = tix - ti * (ti + 1) / 2;
  const int i0 = ti * T, j0 = tj * T;
  const long ld = p.ldk;
  float* C = p.K + r0 + (long)r0 * ld;
  const float* Vt = p.Vt + (long)r0 * B;
  const float* Wt = p.Wt + (long)r0 * B;
  extern __shared__ __align__(16) float usm[];
  const float* As = usm;              // [V_I | W_I]: row i at As + i LD (k 0..63)
  const float* Bs = usm + T * LD;     // [W_J | V_J]: row j at Bs + j LD
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(usm);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool vec = (reinterpret_cast<uintptr_t>(p.Vt) & 15) == 0 && (reinterpret_cast<uintptr_t>(p.Wt) & 15) == 0;
#pragma unroll 4
  for (int u = 0; u < 4 * T * B / 4 / NT; ++u) {
    const int q = tid + NT * u, blk = q / (T * B / 4), r = (q / (B / 4)) % T, c = (q % (B / 4)) * 4;
    const int row = (blk < 2 ? i0 : j0) + r;
    const float* src = ((blk == 0 || blk == 3) ? Vt : Wt) + (long)row * B + c;
    const bool ok = row < L;
    const uint32_t d = sbase + 4u * (uint32_t)((blk >> 1) * T * LD + r * LD + (blk & 1) * B + c);
    if (vec) {
      sbr_cp16(d, ok ? src : Vt, ok);
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) sbr_cp4(d + 4u * e, ok ? src + e : Vt, ok);
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  for (int e = tid; e < T * (T / 32); e += NT) {   // C0 lines (128 bytes) of the tile into L2
    const int col = j0 + e / (T / 32), row = i0 + (e % (T / 32)) * 32;
    if (col < L && row < L) asm volatile("prefetch.global.L2 [%0];" ::"l"(C + row + (long)col * ld));
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  const int g = lane >> 2, t = lane & 3;
  const int rb = (warp & 3) * 32, cb = (warp >> 2) * 64;    // warp tile: 32 rows x 64 columns
  float acc[2][8][4];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[mt][nt][q] = 0.f;
#pragma unroll 2
  for (int ks = 0; ks < 2 * B / 8; ++ks) {
    const int kb = ks * 8;
    uint32_t ah[2][4], al[2][4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const float* ar = As + (rb + 16 * mt + g) * LD + kb + t;
      sbr_split(ar[0], ah[mt][0], al[mt][0]);
      sbr_split(ar[8 * LD], ah[mt][1], al[mt][1]);
      sbr_split(ar[4], ah[mt][2], al[mt][2]);
      sbr_split(ar[8 * LD + 4], ah[mt][3], al[mt][3]);
    }
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const float* br = Bs + (cb + 8 * nt + g) * LD + kb + t;
      uint32_t bh0, bl0, bh1, bl1;
      sbr_split(br[0], bh0, bl0);
      sbr_split(br[4], bh1, bl1);
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {   // small terms first
        sbr_mma(acc[mt][nt], al[mt], bh0, bh1);
        sbr_mma(acc[mt][nt], ah[mt], bl0, bl1);
        sbr_mma(acc[mt][nt], ah[mt], bh0, bh1);
      }
    }
  }
  // C = C0 - acc on the lower triangle; each row tile's 32 C0 loads issued together
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
    float c0[2][8][2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int row = i0 + rb + 16 * mt + g + 8 * h;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = j0 + cb + 8 * nt + 2 * t + e;
          c0[h][nt][e] = (row < L && col <= row) ? C[row + (long)col * ld] : 0.f;
        }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int row = i0 + rb + 16 * mt + g + 8 * h;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = j0 + cb + 8 * nt + 2 * t + e;
          if (row < L && col <= row) C[row + (long)col * ld] = c0[h][nt][e] - acc[mt][nt][2 * h + e];
        }
    }
  }
}

// ---------------------------------------------------------------------- stage 2: chase
#if defined(BKFAC_CHASE_TIMING) || defined(BKFAC_Q2_TIMING)
#define CH_T(v) const unsigned long long v = clock64()
#define CH_ACC(i, a, b) atomicAdd(&g_chase_dbg[i], (b) - (a))
#elif defined(BKFAC_Q2_TIMING)
#define CH_T(v) const unsigned long long v = clock64()
#define CH_ACC(i, a, b)
#else
#define CH_T(v)
#define CH_ACC(i, a, b)
#endif
BKFAC_DEV float sbr_ldcg(const float* a) { return __ldcg(a); }
BKFAC_DEV void sbr_stcg(float* a, float v) { __stcg(a, v); }

// grid (nprob), block SBR_CHASE_WARPS*32.  Band element (r, c), 0 <= r - c < SBR_LDB, at
// AB[c * SBR_LDB + (r - c)].  Outputs d, e (fp32 tridiagonal) and the chase reflectors:
// task (j, k) -> Vq[((j * KT) + k) * B + i], tq[j * KT + k].
__global__ void __launch_bounds__(SBR_CHASE_WARPS * 32, 1)
sbr_chase_kernel(const __grid_constant__ EigBatch b) {
  const EigProb& p = b.p[blockIdx.x];
  if (p.sbr == 0) return;
  const int m = p.m, ld = p.ldk;
  constexpr int B = SBR_B, LDB = SBR_LDB, NW = SBR_CHASE_WARPS, LDT = B + 1;
  const int KT = sbr_tasks(m);
  extern __shared__ __align__(16) float csm[];
  volatile int* prog = reinterpret_cast<volatile int*>(csm);      // 64 ints
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float* Dt = csm + 64 + warp * (2 * B * LDT + 3 * B);
  float* Et = Dt + B * LDT;
  float* vs = Et + B * LDT;
  float* ws = vs + B;
  float* us = ws + B;
  float* AB = p.AB;
  const float* K = p.K;
  // band of the stage-1 result (lower, bandwidth B) + zeroed bulge space
  for (long e = tid; e < (long)m * LDB; e += NW * 32) {
    const int c = (int)(e / LDB), d = (int)(e % LDB);
    AB[e] = (d <= B && c + d < m) ? K[(c + d) + (long)c * ld] : 0.f;
  }
  if (tid < 64) prog[tid] = -1;
  __syncthreads();
#ifdef BKFAC_CHASE_TIMING
  const unsigned long long t_kernel0 = clock64();
#endif
  auto at = [&](int r, int c) -> float* { return AB + (long)c * LDB + (r - c); };
  for (int j = warp; j < m - 2; j += NW) {
    float tau_u = 0.f;
    for (int k = 0;; ++k) {
      const int s = j + 1 + k * B;
      if (s >= m) break;
      const int nk = min(B, m - s);
      const bool row = lane < nk;              // lane = row s + lane of the task's blocks
      CH_T(t0);
      if (j > 0) {
        const int need = ((j - 1) << 8) + (k + 2);
        while (prog[(j - 1) % NW] < need) {
#ifndef BKFAC_CHASE_SPIN
          __nanosleep(20);
#endif
        }
      }
      __syncwarp();
      CH_T(t1);
      // every load of the task in flight at once: the E row (k >= 1; k = 0: column j) and the
      // lower D row (D(lane, l), l <= lane) -- one L2 round trip
      float er[B], dr[B];
#pragma unroll
      for (int l = 0; l < B; ++l) {
        // k >= 1: E(lane, l) = A(s + lane, s - B + l) at AB[(s - B + l) LDB + (B + lane - l)];
        // k = 0: er[0] = A(s + lane, j), the column the sweep annihilates
        if (k == 0) er[l] = (row && l == 0) ? sbr_ldcg(at(s + lane, j)) : 0.f;
        else er[l] = row ? sbr_ldcg(AB + (long)(s - B + l) * LDB + (B + lane - l)) : 0.f;
        dr[l] = (row && l <= lane) ? sbr_ldcg(AB + (long)(s + l) * LDB + (lane - l)) : 0.f;
      }
      float x;
      CH_T(t2);
      if (k == 0) {
        x = er[0];
      } else {
        // E <- E H_{k-1} (u broadcast as float4 loads)
        float ub[B];
#pragma unroll
        for (int l = 0; l < B; l += 4) {
          const float4 f4 = *reinterpret_cast<const float4*>(&us[l]);
          ub[l] = f4.x; ub[l + 1] = f4.y; ub[l + 2] = f4.z; ub[l + 3] = f4.w;
        }
        float tt[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int l = 0; l < B; ++l) tt[l & 3] = fmaf(er[l], ub[l], tt[l & 3]);
        const float t = ((tt[0] + tt[1]) + (tt[2] + tt[3])) * tau_u;
#pragma unroll
        for (int l = 0; l < B; ++l) er[l] = fmaf(-t, ub[l], er[l]);
        x = er[0];
      }
      // reflector from x (length nk): annihilates x[1:nk]
      const float alpha = __shfl_sync(0xffffffffu, x, 0);
      const float xn2 = warp_sum((lane >= 1 && row) ? x * x : 0.f);
      float tau = 0.f, beta = alpha, v = lane == 0 ? 1.f : 0.f;
      if (nk > 1 && xn2 > 0.f) {
        beta = -copysignf(sqrtf(fmaf(alpha, alpha, xn2)), alpha);
        tau = (beta - alpha) / beta;
        v = lane == 0 ? 1.f : (row ? x / (alpha - beta) : 0.f);
      }
      vs[lane] = v;
      if (k == 0) {
        if (row) sbr_stcg(at(s + lane, j), lane == 0 ? beta : 0.f);
      } else {
        // E <- H_k E: s_l = sum_i v_i E(i, l) through a shared-memory transpose
#pragma unroll
        for (int l = 0; l < B; ++l) Et[lane * LDT + l] = er[l];
        __syncwarp();
        float sl[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < B; i += 4) {
          const float4 v4 = *reinterpret_cast<const float4*>(&vs[i]);
          sl[0] = fmaf(v4.x, Et[i * LDT + lane], sl[0]);
          sl[1] = fmaf(v4.y, Et[(i + 1) * LDT + lane], sl[1]);
          sl[2] = fmaf(v4.z, Et[(i + 2) * LDT + lane], sl[2]);
          sl[3] = fmaf(v4.w, Et[(i + 3) * LDT + lane], sl[3]);
        }
        ws[lane] = tau * ((sl[0] + sl[1]) + (sl[2] + sl[3]));
        __syncwarp();
#pragma unroll
        for (int l = 0; l < B; l += 4) {
          const float4 w4 = *reinterpret_cast<const float4*>(&ws[l]);
          if (l > 0) er[l] = fmaf(-v, w4.x, er[l]);
          er[l + 1] = fmaf(-v, w4.y, er[l + 1]);
          er[l + 2] = fmaf(-v, w4.z, er[l + 2]);
          er[l + 3] = fmaf(-v, w4.w, er[l + 3]);
        }
        er[0] = lane == 0 ? beta : 0.f;
        if (row) {
#pragma unroll
          for (int l = 0; l < B; ++l) sbr_stcg(AB + (long)(s - B + l) * LDB + (B + lane - l), er[l]);
        }
      }
      __syncwarp();
      CH_T(t3);
      if (tau != 0.f) {
        // D = A[R_k, R_k] <- H D H:  p = tau D v, w = p - tau/2 (p.v) v, D -= v w^T + w v^T
        // (D v)_i = sum_{l <= i} D(i, l) v_l (this lane's lower row, registers) + sum_{l > i}
        // D(l, i) v_l (column i below the diagonal: lane l's row, through shared memory)
#pragma unroll
        for (int l = 0; l < B; ++l) Dt[lane * LDT + l] = dr[l];   // row lane (zeros above the diagonal)
        float vb[B];
#pragma unroll
        for (int l = 0; l < B; l += 4) {
          const float4 f4 = *reinterpret_cast<const float4*>(&vs[l]);
          vb[l] = f4.x; vb[l + 1] = f4.y; vb[l + 2] = f4.z; vb[l + 3] = f4.w;
        }
        __syncwarp();
        float pp[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int l = 0; l < B; ++l) {
          const float col = (l > lane) ? Dt[l * LDT + lane] : dr[l];
          pp[l & 3] = fmaf(col, vb[l], pp[l & 3]);
        }
        const float pi = tau * ((pp[0] + pp[1]) + (pp[2] + pp[3]));
        const float dot = warp_sum(pi * v);
        const float wi = fmaf(-0.5f * tau * dot, v, pi);
        ws[lane] = wi;
        __syncwarp();
        if (row) {
#pragma unroll
          for (int l = 0; l < B; l += 4) {
            const float4 w4 = *reinterpret_cast<const float4*>(&ws[l]);
            const float wl[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (l + u <= lane)
                sbr_stcg(AB + (long)(s + l + u) * LDB + (lane - l - u), dr[l + u] - v * wl[u] - wi * vb[l + u]);
          }
        }
      }
      CH_T(t4);
      p.Vq[((long)j * KT + k) * B + lane] = v;
      if (lane == 0) p.tq[(long)j * KT + k] = tau;
      us[lane] = v;
      tau_u = tau;
      __syncwarp();
      __threadfence_block();
      if (lane == 0) prog[warp] = (j << 8) + (k + 1);
      CH_T(t5);
#ifdef BKFAC_CHASE_TIMING
      if (lane == 0 && blockIdx.x == 0) {
        CH_ACC(0, t0, t1); CH_ACC(1, t1, t2); CH_ACC(2, t2, t3); CH_ACC(3, t3, t4); CH_ACC(4, t4, t5);
        atomicAdd(&g_chase_dbg[5], 1ull);
      }
#endif
    }
    __syncwarp();
    __threadfence_block();
    if (lane == 0) prog[warp] = (j << 8) + 255;
  }
  __syncthreads();
#ifdef BKFAC_CHASE_TIMING
  if (tid == 0 && blockIdx.x == 0) atomicAdd(&g_chase_dbg[6], clock64() - t_kernel0);
#endif
  for (int i = tid; i < m; i += NW * 32) {
    p.d[i] = sbr_ldcg(AB + (long)i * LDB);
    if (i < m - 1) p.e[i] = sbr_ldcg(AB + (long)i * LDB + 1);
  }
}

// ---------------------------------------------------------------------- Q2 back-transform
// grid (nprob, ceil(r / SBR_Q2_THREADS)), block SBR_Q2_THREADS, thread = eigenvector column c
// (its column of Z is private to it).  Reads the inverse-iteration output Y (fp64,
// Y[i*r + c]) and leaves Q2 Y in Zr (fp32, row-major m x r), which backtr_prep_kernel turns
// into the column-major V.  Per group of SBR_G sweeps the 63-row diamond window slides down
// the column in steps of 32 rows: rows leaving the window are stored, the next 32 rows are
// loaded before the current diamond is applied (they are not touched by it), so each group
// streams the column through registers once.
// NT = 128 columns per CTA; with few factors per launch (an 8-GPU rank's 12) 32-column CTAs
// spread the same per-column work over more SMs (the arithmetic of a column is unchanged)
constexpr int SBR_Q2_THREADS = 128;
template <int NT>
__global__ void __launch_bounds__(NT, (SBR_G > 32 ? 256 : 384) / NT)
sbr_q2_kernel(const __grid_constant__ EigBatch b) {
  const EigProb& p = b.p[blockIdx.x];
  if (p.sbr == 0) return;
  const int m = p.m, r = p.r;
  constexpr int B = SBR_B, G = SBR_G, WIN = B + G - 1;
  static_assert(G % B == 0, "the window slides by one task (B rows) and carries WIN - B = G - 1 rows");
  const int KT = sbr_tasks(m);
  const int c = blockIdx.y * NT + threadIdx.x;
  if (blockIdx.y * NT >= r) return;
  const bool cok = c < r;
  __shared__ __align__(16) float vsm[2][G * B];
  __shared__ float tsm[2][G];
  float* Z = p.Zr + c;
  if (cok)
    for (int i = 0; i < m; ++i) Z[(long)i * r] = (float)p.Y[(long)i * r + c];
  const int nsw = m - 2;
  const int ngroups = (nsw + G - 1) / G;
  // reflectors of diamond (g, k) into buffer q (every thread of the CTA takes a share) by
  // cp.async (zero-filled where a task does not exist): the copies complete while the
  // current diamond is applied, and are waited for before the next diamond's barrier
  auto cp4 = [](float* dst, const float* src, bool ok) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(ok ? 4 : 0) : "memory");
  };
  auto cp16 = [](float* dst, const float* src, bool ok) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(ok ? 16 : 0) : "memory");
  };
  auto stage = [&](int q, int j0, int jn, int k) {
    for (int e = threadIdx.x; e < G * B / 4; e += NT) {   // 16-byte pieces of the reflectors
      const int a = e / (B / 4), i = (e % (B / 4)) * 4;
      const bool ex = a < jn && j0 + a + 1 + k * B < m;
      cp16(&vsm[q][a * B + i], ex ? p.Vq + ((long)(j0 + a) * KT + k) * B + i : p.Vq, ex);
    }
    for (int a = threadIdx.x; a < G; a += NT) {
      const bool ex = a < jn && j0 + a + 1 + k * B < m;
      cp4(&tsm[q][a], ex ? p.tq + (long)(j0 + a) * KT + k : p.tq, ex);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto stage_wait = [] { asm volatile("cp.async.wait_all;" ::: "memory"); };
  int q = 0;
  for (int g = ngroups - 1; g >= 0; --g) {
    const int j0 = g * G, jn = min(G, nsw - j0);
    __syncthreads();
    stage(q, j0, jn, 0);
    stage_wait();
    // window of diamond k: rows j0 + 1 + k B .. + WIN - 1; w[t] <-> row rb + t
    int rb = j0 + 1;
    float w[WIN];
#pragma unroll
    for (int t = 0; t < WIN; ++t) w[t] = (cok && rb + t < m) ? Z[(long)(rb + t) * r] : 0.f;
    for (int k = 0; rb < m; ++k, rb += B) {
      CH_T(q0);
      stage_wait();      // this thread's copies into buffer q have landed
      __syncthreads();   // buffer q staged by every thread; buffer q ^ 1 free
      CH_T(q1);
      if (rb + B < m) stage(q ^ 1, j0, jn, k + 1);
      // next diamond's new rows (rb + WIN .. rb + WIN + B - 1): untouched by this diamond
      // (running pointer laundered through asm: no 64-bit multiply per row)
      float nx[B];
      {
        const float* zp;
        int rl;
        asm volatile("mov.b64 %0, %1;" : "=l"(zp) : "l"(Z + (long)(rb + WIN) * r));
        asm volatile("mov.b32 %0, %1;" : "=r"(rl) : "r"(r));
        const int nn = cok ? m - (rb + WIN) : 0;
#pragma unroll
        for (int t = 0; t < B; ++t) {
          nx[t] = t < nn ? *zp : 0.f;
          zp += rl;
        }
      }
      CH_T(q2);
      // the diamond's block reflector H_{j0} H_{j0+1} ... H_{j0+G-1}: applied last first
      const float* vq = vsm[q];
      // reflector a's vector is loaded while reflector a + 1 is applied (two register sets;
      // the compiler barrier keeps it from hoisting every reflector's loads)
      float vc[B], vn[B];
      float tc = tsm[q][G - 1], tn = 0.f;
#pragma unroll
      for (int i = 0; i < B; i += 4) {
        const float4 f4 = *reinterpret_cast<const float4*>(&vq[(G - 1) * B + i]);
        vc[i] = f4.x; vc[i + 1] = f4.y; vc[i + 2] = f4.z; vc[i + 3] = f4.w;
      }
#pragma unroll
      for (int a = G - 1; a >= 0; --a) {
        asm volatile("" ::: "memory");
        if (a > 0) {
#pragma unroll
          for (int i = 0; i < B; i += 4) {
            const float4 f4 = *reinterpret_cast<const float4*>(&vq[(a - 1) * B + i]);
            vn[i] = f4.x; vn[i + 1] = f4.y; vn[i + 2] = f4.z; vn[i + 3] = f4.w;
          }
          tn = tsm[q][a - 1];
        }
        float dd[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) dd[u] = 0.f;
#pragma unroll
        for (int i = 0; i < B; ++i) dd[i & 7] = fmaf(vc[i], w[a + i], dd[i & 7]);
        const float d = (((dd[0] + dd[1]) + (dd[2] + dd[3])) + ((dd[4] + dd[5]) + (dd[6] + dd[7]))) * tc;
#pragma unroll
        for (int i = 0; i < B; ++i) w[a + i] = fmaf(-d, vc[i], w[a + i]);
#pragma unroll
        for (int i = 0; i < B; ++i) vc[i] = vn[i];
        tc = tn;
      }
      CH_T(q3);
      // rows rb .. rb + B - 1 leave the window; slide by B
      {
        float* zp;
        int rl;
        asm volatile("mov.b64 %0, %1;" : "=l"(zp) : "l"(Z + (long)rb * r));
        asm volatile("mov.b32 %0, %1;" : "=r"(rl) : "r"(r));
        const int nn = cok ? m - rb : 0;
#pragma unroll
        for (int t = 0; t < B; ++t) {
          if (t < nn) *zp = w[t];
          zp += rl;
        }
      }
#ifdef BKFAC_Q2_TIMING
      if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) {
        const unsigned long long q4 = clock64();
        atomicAdd(&g_chase_dbg[0], q1 - q0); atomicAdd(&g_chase_dbg[1], q2 - q1);
        atomicAdd(&g_chase_dbg[2], q3 - q2); atomicAdd(&g_chase_dbg[3], q4 - q3);
        atomicAdd(&g_chase_dbg[5], 1ull);
      }
#endif
#pragma unroll
      for (int t = 0; t < WIN - B; ++t) w[t] = w[t + B];
#pragma unroll
      for (int t = 0; t < B; ++t) w[WIN - B + t] = nx[t];
      q ^= 1;
    }
  }
}

}  // namespace bkfac
