// Householder tridiagonalisation with the matrix resident in the distributed shared
// memory of one thread-block cluster per factor (sm_90+/sm_100a DSMEM).
//
// The lower triangle of K (m x m) is split column-cyclically over the C CTAs of a
// cluster: CTA q owns columns j = q, q+C, q+2C, ... (rows j..m-1, packed).  Step k:
//   (a) the owner of column k applies the previous rank-2 update to it, forms the
//       reflector v_k (dlarfg), stores it in place and broadcasts v_k and tau_k into
//       every CTA's shared memory (st.shared::cluster);                  cluster barrier
//   (b) every CTA applies the previous rank-2 update to its own columns j > k and, in
//       the same pass, accumulates its partial y = K22 v_k (lower triangle: column dot
//       for y_j, scatter for y_i, i > j);                                cluster barrier
//   (c) every CTA sums the C partial y vectors through DSMEM and forms
//       w_k = tau y - (tau^2/2)(y.v) v  locally (identical on every CTA).
// v is double-buffered by step parity (an owner may broadcast v_{k+1} while another CTA
// still reads v_k in (c)); y needs one buffer since (b) of step k+1 starts after barrier
// (a) of step k+1, which every CTA reaches only after finishing (c) of step k.
// Outputs as sytrd_kernel: d, e, tau, reflectors in K's lower triangle (rows >= k+2).
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"
#include "eig.cuh"

namespace bkfac {

namespace cg = cooperative_groups;

BKFAC_DEV int own_col_off(int t, int m, int q, int C) {
  return t * m - t * q - C * (t * (t - 1) / 2);
}

constexpr int SYTRD_CLUSTER_SMEM_FLOATS = 53 * 1024;  // 212 KB budget per CTA

// smallest cluster size whose per-CTA share fits; 0 = use the global-memory kernel
inline int sytrd_cluster_size(int m) {
  for (int C = 1; C <= 8; C *= 2) {
    const long own = ((long)m * (m + 1) / 2 + (long)C * m) / C;  // upper bound per CTA
    const long extra = 38L * m + 64;
    if (own + extra <= SYTRD_CLUSTER_SMEM_FLOATS) return C;
  }
  return 0;
}
inline size_t sytrd_cluster_smem_bytes(int m, int C) {
  const long own = ((long)m * (m + 1) / 2 + (long)C * m) / C;
  return sizeof(float) * (size_t)(own + 38L * m + 64);
}

__global__ void __launch_bounds__(1024, 1) sytrd_cluster_kernel(const __grid_constant__ EigBatch b,
                                                               int C) {
  cg::cluster_group cluster = cg::this_cluster();
  const int q = (int)cluster.block_rank();
  const EigProb& p = b.p[blockIdx.x / C];
  const int m = p.m;
  const int ld = p.ldk;
  float* K = p.K;
  extern __shared__ __align__(16) float zsm[];
  float* vb = zsm;            // 2*m  (v double buffer)
  float* wp = vb + 2 * m;     // m    (w of the previous step, local)
  float* y = wp + m;          // m    (partial y; read remotely)
  float* ys = y + m;          // m    (summed y, local)
  float* scal = ys + m;       // 32   [0..1]: tau by parity, [2]: bad flag
  float* red = scal + 32;     // 32
  float* ywarp = red + 32;    // 32 * m  (per-warp partial y)
  float* col = ywarp + 32 * m;  // owned columns, packed
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const int nown = (q < m) ? (m - q + C - 1) / C : 0;

  // load owned columns (lower part) + finiteness check
  int bad = 0;
  for (int t = warp; t < nown; t += nw) {
    const int j = q + t * C;
    float* cj = col + own_col_off(t, m, q, C);
    for (int i = j + lane; i < m; i += 32) {
      const float a = K[i + (long)j * ld];
      bad |= !isfinite(a);
      cj[i - j] = a;
    }
  }
  bad = __syncthreads_or(bad);
  if (tid == 0) scal[2] = bad ? 1.f : 0.f;
  cluster.sync();
  float anybad = 0.f;
  for (int r = 0; r < C; ++r) anybad += *cluster.map_shared_rank(scal + 2, r);
  cluster.sync();
  if (anybad != 0.f) {
    if (q == 0) {
      if (tid == 0 && p.status) atomicOr(p.status, ST_NONFINITE);
      for (int i = tid; i < m; i += nt) { p.d[i] = 0.f; p.e[i] = 0.f; p.tau[i] = 0.f; }
    }
    return;
  }
  if (m <= 2) {  // already tridiagonal
    if (q == 0 && tid == 0) {
      p.d[0] = K[0];
      p.e[0] = (m == 2) ? K[1] : 0.f;
      p.tau[0] = 0.f;
      if (m == 2) { p.d[1] = K[1 + (long)ld]; p.e[1] = 0.f; p.tau[1] = 0.f; }
    }
    return;
  }

  bool have_prev = false;
  for (int k = 0; k < m - 2; ++k) {
    float* v = vb + (k & 1) * m;
    const float* vp = vb + ((k + 1) & 1) * m;   // v_{k-1}
    const int owner = k % C;
    if (q == owner) {
      float* ck = col + own_col_off(k / C, m, q, C);   // rows k..m-1
      if (have_prev)
        for (int i = k + tid; i < m; i += nt) ck[i - k] -= vp[i] * wp[k] + wp[i] * vp[k];
      __syncthreads();
      const float alpha = ck[1];
      float ss = 0.f;
      for (int i = k + 2 + tid; i < m; i += nt) ss += ck[i - k] * ck[i - k];
      ss = block_sum(ss, red);
      float tau, beta, scale;
      if (ss == 0.f) {
        tau = 0.f; beta = alpha; scale = 0.f;
      } else {
        const float nrm = sqrtf(alpha * alpha + ss);
        beta = alpha >= 0.f ? -nrm : nrm;
        tau = (beta - alpha) / beta;
        scale = 1.f / (alpha - beta);
      }
      for (int i = k + 1 + tid; i < m; i += nt) {
        float vi = 1.f;
        if (i >= k + 2) {
          vi = ck[i - k] * scale;
          ck[i - k] = vi;
        }
        for (int r = 0; r < C; ++r) *cluster.map_shared_rank(v + i, r) = vi;
      }
      if (tid == 0) {
        p.d[k] = ck[0];
        p.e[k] = beta;
        p.tau[k] = tau;
        for (int r = 0; r < C; ++r) *cluster.map_shared_rank(scal + (k & 1), r) = tau;
      }
    }
    cluster.sync();                                              // (1) v_k, tau_k everywhere
    const float tau = scal[k & 1];
    float* yw = ywarp + warp * m;     // this warp's private partial of y (no atomics)
    for (int i = k + 1 + lane; i < m; i += 32) yw[i] = 0.f;
    __syncwarp();
    // (b) fused update (v_{k-1}, w_{k-1}) + partial symv with v_k on owned columns j > k
    const int t0 = (k + 1 - q + C - 1) / C > 0 ? (k + 1 - q + C - 1) / C : 0;
    for (int t = t0 + warp; t < nown; t += nw) {
      const int j = q + t * C;
      float* cj = col + own_col_off(t, m, q, C);
      const float vj = v[j];
      const float wpj = have_prev ? wp[j] : 0.f, vpj = have_prev ? vp[j] : 0.f;
      float acc = 0.f;
      for (int i = j + lane; i < m; i += 32) {
        float a = cj[i - j];
        if (have_prev) {
          a -= vp[i] * wpj + wp[i] * vpj;
          cj[i - j] = a;
        }
        acc = fmaf(a, v[i], acc);
        if (i > j) yw[i] = fmaf(a, vj, yw[i]);
      }
      acc = warp_sum(acc);
      __syncwarp();
      if (lane == 0) yw[j] += acc;
      __syncwarp();
    }
    __syncthreads();
    // CTA partial: y[i] = sum over warps
    for (int i = k + 1 + tid; i < m; i += nt) {
      float s = 0.f;
#pragma unroll 8
      for (int w = 0; w < nw; ++w) s += ywarp[w * m + i];
      y[i] = s;
    }
    __syncthreads();
    cluster.sync();                                              // (2) partial y ready
    float pv = 0.f;
    for (int i = k + 1 + tid; i < m; i += nt) {
      float s = 0.f;
      for (int r = 0; r < C; ++r) s += *cluster.map_shared_rank(y + i, r);
      ys[i] = s;
      pv = fmaf(s, v[i], pv);
    }
    pv = block_sum(pv, red);
    const float gamma = 0.5f * tau * tau * pv;
    for (int i = k + 1 + tid; i < m; i += nt) wp[i] = tau * ys[i] - gamma * v[i];
    have_prev = true;
    __syncthreads();
  }
  // trailing 2x2 block: apply the last rank-2 update, read d, e
  {
    const int k = m - 2;
    const float* vp = vb + ((k + 1) & 1) * m;
    if (q == (m - 2) % C && tid < 2) {
      float* c2 = col + own_col_off((m - 2) / C, m, q, C);
      const int i = m - 2 + tid;
      c2[i - (m - 2)] -= vp[i] * wp[m - 2] + wp[i] * vp[m - 2];
    }
    if (q == (m - 1) % C && tid == 32) {
      float* c1 = col + own_col_off((m - 1) / C, m, q, C);
      c1[0] -= 2.f * vp[m - 1] * wp[m - 1];
    }
    __syncthreads();
    if (q == (m - 2) % C && tid == 0) {
      const float* c2 = col + own_col_off((m - 2) / C, m, q, C);
      p.d[m - 2] = c2[0];
      p.e[m - 2] = c2[1];
      p.e[m - 1] = 0.f;
      p.tau[m - 2] = 0.f;
      p.tau[m - 1] = 0.f;
    }
    if (q == (m - 1) % C && tid == 0) p.d[m - 1] = col[own_col_off((m - 1) / C, m, q, C)];
  }
  // write the owned columns (reflectors below the subdiagonal) back for the back-transform
  for (int t = warp; t < nown; t += nw) {
    const int j = q + t * C;
    const float* cj = col + own_col_off(t, m, q, C);
    for (int i = j + lane; i < m; i += 32) K[i + (long)j * ld] = cj[i - j];
  }
  cluster.sync();  // no CTA may exit while others can still address its shared memory
}

}  // namespace bkfac
