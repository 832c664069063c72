// Householder tridiagonalisation of the Brand core K (Alg 3 line 4 "EVD(M_S)",
// PAPER.md:505) with the lower triangle resident in the distributed shared memory of a
// thread-block cluster, processed in 32 x 32 register tiles.
//
// Storage.  K is padded to m_pad = 32*NB rows/cols (zeros).  The lower tiles (I >= J) are
// enumerated by decreasing block column J (then increasing I): pos(I, J) =
// T(NB-1-J) + I - J, T(n) = n(n+1)/2, and dealt round-robin to the C CTAs of the cluster
// (owner = pos % C, slot = pos / C; each tile 32 x 32 col-major in the owner's shared
// memory).  The tiles still active at step k (J >= k/32) are a prefix of this order, so
// every CTA holds an equal share (+-1) of the active tiles at EVERY step, and each CTA's
// active tiles are a prefix of its slots: warp w takes slots w, w + NW, ...
//
// Step k (reflector H_k = I - tau v v^T zeroing column k below the subdiagonal):
//   (a) EVERY CTA reads column k from its owners' shared memory (ld.shared::cluster; the
//       column is final after step k-1's tiles), applies the pending rank-2 update of step
//       k-1 (A <- A - v w^T - w v^T) and forms v_k, tau_k (dlarfg) locally.  All CTAs
//       compute bitwise-identical v_k (same inputs, same reduction order), so no
//       broadcast and no cluster barrier is needed here; CTA k % C writes d, e, tau and
//       the reflector (rows >= k+2 of column k of K) to global memory;
//   (b) every CTA walks its active tiles with one warp per tile, lane = row: applies the
//       pending update in registers, writes the tile back, and accumulates its partial
//       y = A v_k both ways from the lower triangle -- row sums in a register, column
//       sums by a 31-shuffle transpose-reduce; both go to the CTA's partial y with
//       shared-memory atomics;                                        cluster barrier
//   (c) every CTA sums the C partial y through DSMEM and forms
//       w_k = tau y - (tau^2/2)(y.v) v locally.
// One cluster barrier per step.  Hazards: the partial y are double-buffered by step
// parity (a CTA rewrites a parity only after the next barrier, which every reader of the
// previous use has passed); column k is never written after step k-1's tiles.
// Per element of the trailing matrix and step: one LDS, one STS and five FP32 ops.
// Outputs: d, e, tau and the reflectors (rows >= k+2 of column k) in K's lower triangle
// for the back-transform.
// Instantiations (MODE): 0 = the above, tiles in the cluster's shared memory (m <= ~700);
// 1 = tiles in global memory, one CTA per factor (large m with many factors: HBM-bound);
// 2 = tiles in global memory shared by a cluster of up to 8 CTAs (large m with few factors
// per GPU, e.g. one 8-GPU rank's share: tiles L2-resident, partial y through DSMEM).
#pragma once
#include <cooperative_groups.h>

#include <algorithm>

#include "common.cuh"
#include "eig.cuh"

namespace bkfac {

namespace cgt = cooperative_groups;

constexpr int SYT_THREADS = 512;
constexpr int SYT_SMEM_FLOATS = 55 * 1024;   // per-CTA budget (220 KB)

__host__ __device__ inline int syt_tiles(int NB) { return NB * (NB + 1) / 2; }
// enumeration position of lower tile (I, J): block columns NB-1, NB-2, ..., 0
__host__ __device__ inline int syt_pos(int I, int J, int NB) {
  const int n = NB - 1 - J;
  return n * (n + 1) / 2 + (I - J);
}
// vectors (6 m_pad + 64 scalars) + one m_pad of slack + a 96-float broadcast stage per warp
inline int syt_vec_floats(int m_pad) { return 7 * m_pad + 64 + (SYT_THREADS / 32) * 96; }
inline long syt_own_floats(int NB, int C) { return 1024L * ((syt_tiles(NB) + C - 1) / C); }
// global-tile variant: vectors + a two-tile cp.async ring per warp
inline int syt_gt_smem_floats(int m_pad) { return syt_vec_floats(m_pad) + (SYT_THREADS / 32) * 2048; }
// smallest cluster size whose per-CTA share fits; 0 = does not fit
inline int sytrd_tiled_cluster(int m) {
  const int NB = (m + 31) / 32, m_pad = NB * 32;
  for (int C = 1; C <= 8; C *= 2)
    if (syt_own_floats(NB, C) + syt_vec_floats(m_pad) <= SYT_SMEM_FLOATS) return C;
  return 0;
}
inline size_t sytrd_tiled_smem_bytes(int m, int C) {
  const int NB = (m + 31) / 32, m_pad = NB * 32;
  return sizeof(float) * (size_t)(syt_own_floats(NB, C) + syt_vec_floats(m_pad));
}

// Tile storage of one factor when the tiles do not fit the cluster's shared memory
// (GT = true: one CTA per factor, tiles in global memory / L2).
inline size_t syt_global_tile_floats(int m) {
  const int NB = (m + 31) / 32;
  return (size_t)syt_tiles(NB) * 1024;
}

// Load of float `p` (an address in this CTA's shared memory) from CTA r of the cluster:
// explicit ld.shared::cluster on a mapa'd 32-bit address (no generic-address resolution).
__device__ __forceinline__ float4 syt_dsmem_ld4(const float* p, int r) {   // p 16-byte aligned
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  uint32_t ra;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(r));
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(ra) : "memory");
  return v;
}
__device__ __forceinline__ float syt_dsmem_ld(const float* p, int r) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  uint32_t ra;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(r));
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(ra) : "memory");
  return v;
}

// Block sum with one barrier.  Precondition: every call is separated from the next one
// by at least one __syncthreads (true at both call sites below), so `red` is not
// rewritten while a warp still reads it.
__device__ __forceinline__ float syt_block_sum(float v, float* red) {
  constexpr int NW = SYT_THREADS / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float t = red[lane & (NW - 1)];
#pragma unroll
  for (int o = NW / 2; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  return t;
}

// MODE 0: tiles in the cluster's shared memory; 1: tiles in global memory, one CTA per
// factor; 2: tiles in global memory (L2) shared by a cluster of C CTAs -- for few, large
// factors (an 8-GPU rank's share of configs[4]), where one CTA per factor leaves most SMs idle
template <int MODE>
__global__ void __launch_bounds__(SYT_THREADS, 1)
sytrd_tiled_kernel(const __grid_constant__ EigBatch b, int C) {
  constexpr bool GT = MODE >= 1;    // tiles in global memory
  constexpr bool CL = MODE != 1;    // cluster code compiled (C may exceed 1)
  cgt::cluster_group cluster = cgt::this_cluster();
  const int q = (int)cluster.block_rank();
  const EigProb& p = b.p[blockIdx.x / C];
  const int m = p.m;
  const int ld = p.ldk;
  float* K = p.K;
  const int NB = (m + 31) >> 5, m_pad = NB << 5;
  extern __shared__ __align__(16) float tsm[];
  float* vbuf = tsm;                 // 2 * m_pad  (v_k by parity, formed by every CTA)
  float* ybuf = vbuf + 2 * m_pad;    // 2 * m_pad  (partial y by parity, read remotely)
  float* ys = ybuf + 2 * m_pad;      // m_pad      (summed y)
  float* wp = ys + m_pad;            // m_pad      (w_{k-1})
  float* scal = wp + m_pad;          // 64: [2] bad, [4..35] reduce, [40..41] alpha, d, [44..59] reduce 2, [60] y_k[k+1]
  float* bst = scal + 64 + (threadIdx.x >> 5) * 96;   // this warp's broadcast stage
  float* tiles = GT ? p.gtiles : scal + 64 + (SYT_THREADS / 32) * 96;   // owned tiles, slot s at 1024 s
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = SYT_THREADS / 32;
  float* red = scal + 4;
  const int ntiles = syt_tiles(NB);
  const int nown = (ntiles - q + C - 1) / C;          // tiles owned by this CTA
  // address of `ptr` in CTA r of the cluster (plain local pointer for 1-CTA launches)
  auto rptr = [&](float* ptr, int r) -> float* { return (!CL || C == 1) ? ptr : cluster.map_shared_rank(ptr, r); };
  // this CTA's tile slot sl: shared memory (slot order) or global memory (position order,
  // pos = sl * C + q, so any CTA of the cluster can address any tile)
  auto slot_ptr = [&](int sl) -> float* { return GT ? tiles + 1024L * ((long)sl * C + q) : tiles + 1024L * sl; };
  // (I, J) of the tile at enumeration position pos (inverse of syt_pos)
  auto tile_ij = [&](int pos, int& I, int& J) {
    int n = (int)((sqrtf(8.f * pos + 1.f) - 1.f) * 0.5f);   // largest n: n(n+1)/2 <= pos
    while (n * (n + 1) / 2 > pos) --n;
    while ((n + 1) * (n + 2) / 2 <= pos) ++n;
    J = NB - 1 - n;
    I = J + (pos - n * (n + 1) / 2);
  };

  for (int i = tid; i < 4 * m_pad; i += SYT_THREADS) vbuf[i] = 0.f;   // vbuf + ybuf
  for (int i = tid; i < 2 * m_pad; i += SYT_THREADS) ys[i] = 0.f;     // ys + wp
  // load owned tiles (zero padding) + finiteness check
  int bad = 0;
  for (int sl = warp; sl < nown; sl += NW) {
    int I, J;
    tile_ij(sl * C + q, I, J);
    float* t = slot_ptr(sl);
    const int i = 32 * I + lane;
    for (int jj = 0; jj < 32; ++jj) {
      const int j = 32 * J + jj;
      float a = 0.f;
      if (i < m && j < m && i >= j) { a = K[i + (long)j * ld]; bad |= !isfinite(a); }
      t[jj * 32 + lane] = a;
    }
  }
  bad = __syncthreads_or(bad);
  if (tid == 0) scal[2] = bad ? 1.f : 0.f;
  if (CL && C > 1) cluster.sync(); else __syncthreads();
  float anybad = 0.f;
  for (int r = 0; r < C; ++r) anybad += *rptr(scal + 2, r);
  if (CL && C > 1) cluster.sync(); else __syncthreads();
  if (anybad != 0.f) {
    if (q == 0) {
      if (tid == 0 && p.status) atomicOr(p.status, ST_NONFINITE);
      for (int i = tid; i < m; i += SYT_THREADS) { p.d[i] = 0.f; p.e[i] = 0.f; p.tau[i] = 0.f; }
    }
    return;
  }
  if (m <= 2) {
    if (q == 0 && tid == 0) {
      p.d[0] = K[0];
      p.e[0] = (m == 2) ? K[1] : 0.f;
      p.tau[0] = 0.f;
      if (m == 2) { p.d[1] = K[1 + (long)ld]; p.e[1] = 0.f; p.tau[1] = 0.f; }
    }
    return;
  }

#ifdef BKFAC_SYT_TIMING
  unsigned long long tacc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, tprev = clock64();
#define SYT_T(i) do { if (tid == 0) { unsigned long long tn = clock64(); tacc[i] += tn - tprev; tprev = tn; } } while (0)
#else
#define SYT_T(i) do {} while (0)
#endif
  float* red2 = scal + 44;    // per-warp partial sums of ||x||^2 of the next reflector
  // The reflector v_k is kept UNSCALED in vbuf (x = column k with the pending updates);
  // dlarfg's scaling is applied on read: v_k[i] = 0 (i <= k), 1 (i = k+1), x_i s_k (i >= k+2).
  // Its norm is reduced through the barrier that opens step k, so forming v_k costs no
  // barrier and no pass of its own.
  auto vget = [](const float* buf, int kk, float s, int i) -> float {
    return i >= kk + 2 ? buf[i] * s : (i == kk + 1 ? 1.f : 0.f);
  };
  // (a) for step 0: column 0 (no pending update)
  {
    float ss = 0.f;
    for (int i = tid; i < m; i += SYT_THREADS) {
      const int pos = syt_pos(i >> 5, 0, NB);
      const float x = GT ? tiles[1024L * pos + (i & 31)] : *rptr(tiles + 1024L * (pos / C) + (i & 31), pos % C);
      if (i >= 2) ss = fmaf(x, x, ss);
      else scal[40 + i] = x;
      vbuf[i] = x;
    }
    ss = warp_sum(ss);
    if (lane == 0) red2[warp] = ss;
  }
  float tau = 0.f, sc = 0.f, sc_prev = 0.f;   // tau_k, scale of v_k, scale of v_{k-1}
  SYT_T(0);
  for (int k = 0; k < m - 2; ++k) {
    float* v = vbuf + (k & 1) * m_pad;            // v_k
    const float* vp = vbuf + ((k + 1) & 1) * m_pad;   // v_{k-1} (zero at k = 0)
    float* y = ybuf + (k & 1) * m_pad;
    const bool have_prev = k > 0;
    const int kb = k >> 5;
    __syncthreads();              // raw v_k + its norm partials, w_{k-1}, zeroed y visible
    {
      // dlarfg for v_k, redundantly in every thread (same inputs and order: identical)
      float t = red2[lane & (NW - 1)];
#pragma unroll
      for (int o = NW / 2; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      const float dk = scal[40], alpha = scal[41];
      float tk, beta, scale;
      if (t == 0.f) {
        tk = 0.f; beta = alpha; scale = 0.f;
      } else {
        const float nrm = sqrtf(alpha * alpha + t);
        beta = alpha >= 0.f ? -nrm : nrm;
        tk = (beta - alpha) / beta;
        scale = 1.f / (alpha - beta);
      }
      sc_prev = sc; sc = scale; tau = tk;
      if (q == k % C) {             // the reflector (rows >= k+2) and d, e, tau to global
        float* kcol = K + (long)k * ld;
        for (int i = k + 2 + tid; i < m; i += SYT_THREADS) kcol[i] = v[i] * scale;
        if (tid == 0) { p.d[k] = dk; p.e[k] = beta; p.tau[k] = tk; }
      }
    }
    SYT_T(1);
    // (b) active tiles (J >= kb): this CTA's slots 0 .. nact-1, one per warp
    const int nact = (syt_tiles(NB - kb) - q + C - 1) / C;
    // one tile: pending update (v_{k-1}, w_{k-1}) written back to tcol, partial y = A v_k
    auto tile_work = [&](float (&colv)[32], int I, int J, float* tcol) {
      const int i = 32 * I + lane;
      const float cv = vget(v, k, sc, 32 * J + lane), cvp = vget(vp, k - 1, sc_prev, 32 * J + lane);
      const float cwp = wp[32 * J + lane];
      const float vi = vget(v, k, sc, i), vpi = vget(vp, k - 1, sc_prev, i), wpi = wp[i];
      float racc[4] = {0.f, 0.f, 0.f, 0.f};
      if (I > J) {
        // off-diagonal tile: the column-indexed values go through the warp's shared stage as
        // (cwp, cwp, cvp, cvp) float4 and (cv, cv) float2 pairs read by broadcast, and the
        // arithmetic runs on column pairs (FFMA2): no shuffles in the element loop.  In the
        // current block column (32 J <= k) the finished columns j <= k get zero broadcast
        // values: their elements are written back unchanged and add nothing to y at rows
        // > k (their transposed contributions land in y rows <= k, which are never read).
        const bool live = 32 * J + lane > k;
        bst[(lane >> 1) * 4 + (lane & 1)] = live ? cwp : 0.f;
        bst[(lane >> 1) * 4 + 2 + (lane & 1)] = live ? cvp : 0.f;
        bst[64 + lane] = live ? cv : 0.f;
        __syncwarp();
        const float4* q4 = reinterpret_cast<const float4*>(bst);
        const float2* v2 = reinterpret_cast<const float2*>(bst + 64);
        const float2 nvp2 = make_float2(-vpi, -vpi), nwp2 = make_float2(-wpi, -wpi), vi2 = make_float2(vi, vi);
        float2 r2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int pp = 0; pp < 16; ++pp) {
          float2 x2 = make_float2(colv[2 * pp], colv[2 * pp + 1]);
          if (have_prev) {
            const float4 q = q4[pp];
            x2 = __ffma2_rn(nvp2, make_float2(q.x, q.y), x2);
            x2 = __ffma2_rn(nwp2, make_float2(q.z, q.w), x2);
            tcol[(2 * pp) * 32] = x2.x;
            tcol[(2 * pp + 1) * 32] = x2.y;
          }
          r2[pp & 1] = __ffma2_rn(x2, v2[pp], r2[pp & 1]);
          const float2 c2 = __fmul2_rn(x2, vi2);
          colv[2 * pp] = c2.x;
          colv[2 * pp + 1] = c2.y;
        }
        __syncwarp();                               // the stage is rewritten by the next tile
        racc[0] = r2[0].x; racc[1] = r2[0].y; racc[2] = r2[1].x; racc[3] = r2[1].y;
      } else {
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) {
          const int j = 32 * J + jj;
          const bool valid = (j > k) && (i >= j);
          const float cwpj = __shfl_sync(0xffffffffu, cwp, jj);
          const float cvpj = __shfl_sync(0xffffffffu, cvp, jj);
          const float cvj = __shfl_sync(0xffffffffu, cv, jj);
          float x = colv[jj];
          if (valid && have_prev) {
            x -= vpi * cwpj + wpi * cvpj;
            tcol[jj * 32] = x;
          }
          const float xe = valid ? x : 0.f;
          racc[jj & 3] = fmaf(xe, cvj, racc[jj & 3]);
          colv[jj] = (i > j) ? xe * vi : 0.f;
        }
      }
      // transpose-reduce: lane l ends with sum over lanes of colv[l] (adds on pairs)
#pragma unroll
      for (int s = 16; s >= 2; s >>= 1) {
        const bool upper = (lane & s) != 0;
#pragma unroll
        for (int t = 0; t < s; t += 2) {
          const float2 send = upper ? make_float2(colv[t], colv[t + 1]) : make_float2(colv[t + s], colv[t + s + 1]);
          const float2 keep = upper ? make_float2(colv[t + s], colv[t + s + 1]) : make_float2(colv[t], colv[t + 1]);
          const float2 recv = make_float2(__shfl_xor_sync(0xffffffffu, send.x, s),
                                          __shfl_xor_sync(0xffffffffu, send.y, s));
          const float2 sum = __fadd2_rn(keep, recv);
          colv[t] = sum.x;
          colv[t + 1] = sum.y;
        }
      }
      {
        const bool upper = (lane & 1) != 0;
        const float send = upper ? colv[0] : colv[1];
        const float keep = upper ? colv[1] : colv[0];
        colv[0] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
      }
      atomicAdd(&y[i], (racc[0] + racc[1]) + (racc[2] + racc[3]));
      atomicAdd(&y[32 * J + lane], colv[0]);
    };
    if constexpr (GT) {
      // tiles in global memory (L2 / HBM): each warp streams its tiles through a two-deep
      // shared-memory ring with cp.async, the next tile in flight while this one computes
      float* stg = scal + 64 + NW * 96 + warp * 2048;
      auto issue = [&](int sl2, int bi) {
        const float* src = slot_ptr(sl2);
        const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(stg + bi * 1024));
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8) {
          const int off = (c8 * 32 + lane) * 4;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + off * 4), "l"(src + off) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      };
      if (warp < nact) issue(warp, 0);
      int idx = 0;
      for (int sl = warp; sl < nact; sl += NW, ++idx) {
        if (sl + NW < nact) {
          issue(sl + NW, (idx + 1) & 1);
          asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
          asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncwarp();
        int I, J;
        tile_ij(sl * C + q, I, J);
        const float* sb = stg + (idx & 1) * 1024 + lane;
        float colv[32];
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) colv[jj] = sb[jj * 32];
        __syncwarp();   // the ring slot is refilled two tiles later
        tile_work(colv, I, J, slot_ptr(sl) + lane);
      }
    } else {
      for (int sl = warp; sl < nact; sl += NW) {
        int I, J;
        tile_ij(sl * C + q, I, J);
        float* tcol = tiles + 1024L * sl + lane;   // + jj * 32
        // all 32 loads first: a store to column jj must not order the load of column
        // jj+1 behind it (the compiler cannot prove they differ)
        float colv[32];
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) colv[jj] = tcol[jj * 32];
        tile_work(colv, I, J, tcol);
      }
    }
    SYT_T(2);
    if (CL && C > 1) cluster.sync(); else __syncthreads();   // partial y (and column k+1) ready
    SYT_T(3);
    // (c)+(a) merged: y_k summed through DSMEM -> w_k; in the same pass column k+1 is read
    // from its owners, gets the pending update (v_k, w_k) and yields v_{k+1}, tau_{k+1}
    {
      const int k1 = k + 1;
      const bool next = k1 <= m - 3;
      const int kb1 = k1 >> 5, jk1 = k1 & 31, base1 = syt_pos(kb1, kb1, NB);
      // thread t owns the 4 rows i0 .. i0+3, i0 = (k+1 rounded down to 4) + 4t: 16-byte
      // DSMEM loads of the C partial y and of column k+1 (4 rows never straddle a tile)
      const int i0 = (k1 & ~3) + 4 * tid;
      const bool own = i0 < m;
      float si[4] = {0.f, 0.f, 0.f, 0.f}, xi[4] = {0.f, 0.f, 0.f, 0.f}, vi4[4] = {0.f, 0.f, 0.f, 0.f};
      float pv = 0.f;
      if (own) {
        float4 acc, c4 = make_float4(0.f, 0.f, 0.f, 0.f);
        const int pos1 = base1 + (i0 >> 5) - kb1;   // tile of rows i0.. in column k+1
        if (!CL || C == 1) {                        // one CTA: local partial y
          acc = *reinterpret_cast<const float4*>(y + i0);
        } else {
          // all C remote loads in flight together, then the sums
          float4 t4[8];
#pragma unroll
          for (int r = 0; r < 8; ++r)
            if (r < C) t4[r] = syt_dsmem_ld4(y + i0, r);
          acc = t4[0];
#pragma unroll
          for (int r = 1; r < 8; ++r)
            if (r < C) { acc.x += t4[r].x; acc.y += t4[r].y; acc.z += t4[r].z; acc.w += t4[r].w; }
        }
        if (next) {
          if (GT) c4 = *reinterpret_cast<const float4*>(tiles + 1024L * pos1 + jk1 * 32 + (i0 & 31));
          else if (C == 1) c4 = *reinterpret_cast<const float4*>(tiles + 1024L * pos1 + jk1 * 32 + (i0 & 31));
          else c4 = syt_dsmem_ld4(tiles + 1024L * (pos1 / C) + jk1 * 32 + (i0 & 31), pos1 % C);
        }
        si[0] = acc.x; si[1] = acc.y; si[2] = acc.z; si[3] = acc.w;
        xi[0] = c4.x; xi[1] = c4.y; xi[2] = c4.z; xi[3] = c4.w;
#pragma unroll
        for (int u = 0; u < 4; ++u) vi4[u] = vget(v, k, sc, i0 + u);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (i0 + u >= k1 && i0 + u < m) pv = fmaf(si[u], vi4[u], pv);
          else si[u] = 0.f;
        if (i0 <= k1 && k1 < i0 + 4) {                          // y_k at row k+1
          const int o = k1 - i0;
          scal[60] = o == 0 ? si[0] : o == 1 ? si[1] : o == 2 ? si[2] : si[3];
        }
      }
      SYT_T(5);
      pv = syt_block_sum(pv, red);
      SYT_T(6);
      const float s1 = scal[60];
      const float gamma = 0.5f * tau * tau * pv;
      const float vk1 = 1.f;                       // v_k[k+1]
      const float wk1 = tau * s1 - gamma * vk1;
      float* vn = vbuf + (k1 & 1) * m_pad;         // v_{k+1} (v_{k-1} is no longer needed)
      float ss = 0.f;
      if (own) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + u;
          if (i < k1 || i >= m) continue;
          const float w = tau * si[u] - gamma * vi4[u];
          wp[i] = w;
          if (next) {
            const float x = xi[u] - (vi4[u] * wk1 + w * vk1);
            if (i >= k1 + 2) ss = fmaf(x, x, ss);
            else scal[40 + (i - k1)] = x;         // d_{k+1} (i = k+1), alpha (i = k+2)
            vn[i] = x;                              // raw; scaled on read
          }
        }
      }
      if (tid == 0) wp[k] = 0.f;                  // w_k vanishes at rows <= k
      if (next) {
        float* yn = ybuf + (k1 & 1) * m_pad;       // step k-1's partials: every reader is done
        for (int i = tid; i < m_pad; i += SYT_THREADS) yn[i] = 0.f;
        SYT_T(7);
        ss = warp_sum(ss);                          // reduced after the next step's barrier
        if (lane == 0) red2[warp] = ss;
        SYT_T(8);
      }
    }
    SYT_T(4);
  }
  __syncthreads();
#ifdef BKFAC_SYT_TIMING
  if (tid == 0 && p.status) {   // tuning builds: per-phase cycle sums of CTA q
    unsigned long long* o = reinterpret_cast<unsigned long long*>(p.Y) + 16 * q;
    for (int i = 0; i < 9; ++i) o[i] = tacc[i];
  }
#endif
  // trailing 2x2 block: the pending update of step m-3 (v_{m-3}, w_{m-3}), then d, e;
  // each element by the CTA that owns it
  {
    const float* vq = vbuf + ((m - 1) & 1) * m_pad;   // v_{m-3}
    if (tid < 3) {
      const int i = (tid == 0) ? m - 2 : m - 1, j = (tid == 2) ? m - 1 : m - 2;
      const int pos = syt_pos(i >> 5, j >> 5, NB);
      if (pos % C == q) {
        float* a = (GT ? tiles + 1024L * pos : tiles + 1024L * (pos / C)) + (j & 31) * 32 + (i & 31);
        const float x = *a - (vget(vq, m - 3, sc, i) * wp[j] + wp[i] * vget(vq, m - 3, sc, j));
        *a = x;
        if (tid == 0) { p.d[m - 2] = x; p.tau[m - 2] = 0.f; }
        if (tid == 1) { p.e[m - 2] = x; p.e[m - 1] = 0.f; }
        if (tid == 2) { p.d[m - 1] = x; p.tau[m - 1] = 0.f; }
      }
    }
  }
  if (CL && C > 1) cluster.sync();   // no CTA exits while others may still address its smem
}

}  // namespace bkfac
