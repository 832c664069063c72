// Batched symmetric eigensolver for the Brand core K (m x m, m = r + c) and for the
// dense-path / RSVD projected matrices: "EVD(M_S)" of Alg 3, of which
// only the top-r eigenpairs are kept (truncation, Alg 4 :540-543).
//
//   1. sytrd_tiled_kernel (sytrd_tiled.cuh) Householder tridiagonalisation T = H^T K H.
//   2. bisect_kernel    top-r eigenvalues of T by Sturm-count multisection (fp32, then
//                       fp64; 4 lanes = 4 probes per eigenvalue, 8 eigenvalues per warp).
//   3. invit_kernel     eigenvectors of T by inverse iteration in fp64 (one thread per
//                       eigenvector, tridiagonal LU with partial pivoting).
//   4. cluster_kernel   modified Gram-Schmidt inside clusters of (near-)equal eigenvalues.
//   5. backtr_kernel    V = H Y (apply the m-2 reflectors to the r eigenvectors).
// See DESIGN.md "Eigensolver" for why stage 2/3 replace implicit QL on sm_100a.
#pragma once
#include "common.cuh"

namespace bkfac {

struct EigProb {
  float* K; int ldk;       // m x m symmetric (lower used); overwritten with reflectors
  int m, r;                // order, number of wanted (largest) eigenpairs
  float* d; float* e; float* tau;   // m, m, m (fp32 tridiagonal + reflector scalars)
  double* lam;             // r eigenvalues, descending
  double* Y;               // m x r eigenvectors of T, layout Y[i*r + j]
  double* scr;             // 4*m*r doubles scratch (LU factors)
  unsigned char* piv;      // m*r pivot flags
  float* V; int ldv;       // output eigenvectors of K, m x r col-major
  float* Dout;             // output eigenvalues (r), clamped >= 0
  int* status;
  float* gtiles;           // tridiagonalisation tiles in global memory (large m), else null
  float* Uw;               // blocked back-transform: m x (npanel*BT_PW) panels U_j = W_j T_j
  float* Zw;               // blocked back-transform: BT_PW x r scratch
  float* Sw;               // blocked back-transform: per panel S_j, T_j (BT_PW x BT_PW each)
  int off;                 // reflector offset: reflector of column k has its unit at row k + off
                           // (1: one-stage sytrd; SBR_B: two-stage, sbr.cuh)
  int sbr;                 // two-stage tridiagonalisation (sbr.cuh) for this problem
  float* Vp; float* Xp; float* Wp; float* Tp;   // sbr stage 1: m x B panel V, X, W; B x B T
  float* Vt; float* Wt;    // sbr stage 1: V and W row-major (m x B, row l at + l B)
  float* Zp;               // sbr stage 1: row blocks' shares of Z = V^T Y (ceil(m/128) x B x B)
  float* AB;               // sbr stage 2: band with bulge space, m x SBR_LDB
  float* Vq; float* tq;    // sbr chase reflectors (m x KT x B, m x KT)
  float* Zr;               // sbr: Q2 Y, fp32 row-major m x r (in the inverse-iteration scratch)
};
constexpr int EIG_MAXP = 100;
struct EigBatch { int nprob; EigProb p[EIG_MAXP]; };

// ------------------------------------------------------------------ 2. bisection
// Number of eigenvalues of T strictly below x (Sturm sequence of the LDL^T pivots).
// e2 / q as e2 * rcp(q): hardware reciprocal seed + one Newton step (relative error
// ~1e-14; the count's backward error stays far below the 1e-10 * span stopping width).
// |q| >= pivmin (a normal number), so the flush-to-zero seed is exact in range.
BKFAC_DEV double sturm_div(double e2, double q) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(q));
  y = fma(y, fma(-q, y, 1.0), y);
  return e2 * y;
}

// 1/q for the LU pivots of inverse iteration: reciprocal seed + two Newton steps (relative
// error at the fp64 rounding level; |q| >= tiny, a normal number)
BKFAC_DEV double inv_rcp(double q) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(q));
  y = fma(y, fma(-q, y, 1.0), y);
  return fma(y, fma(-q, y, 1.0), y);
}

BKFAC_DEV int sturm_count(const double* dd, const double* e2, int m, double x, double pivmin) {
  int cnt = 0;
  double q = dd[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  cnt += (q < 0.0);
  for (int i = 1; i < m; ++i) {
    q = (dd[i] - x) - sturm_div(e2[i - 1], q);
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += (q < 0.0);
  }
  return cnt;
}

BKFAC_DEV int sturm_count_f32(const float* dd, const float* e2, int m, float x, float pivmin) {
  int cnt = 0;
  float q = dd[0] - x;
  if (fabsf(q) < pivmin) q = -pivmin;
  cnt += (q < 0.f);
  for (int i = 1; i < m; ++i) {
    q = (dd[i] - x) - __fdividef(e2[i - 1], q);
    if (fabsf(q) < pivmin) q = -pivmin;
    cnt += (q < 0.f);
  }
  return cnt;
}

constexpr int BIS_WARPS = 8;
#ifndef BKFAC_BIS_G
#define BKFAC_BIS_G 4
#endif
constexpr int BIS_G = BKFAC_BIS_G;    // lanes (probes) per eigenvalue
constexpr int BIS_E = 32 / BIS_G;     // eigenvalues per warp

// grid: (nprob, ceil(rmax / (BIS_WARPS * BIS_E))); smem: 2*m doubles + 2*m floats
__global__ void __launch_bounds__(BIS_WARPS * 32) bisect_kernel(const __grid_constant__ EigBatch b) {
  const EigProb& p = b.p[blockIdx.x];
  const int m = p.m;
  extern __shared__ __align__(16) double dsm[];
  double* dd = dsm;
  double* e2 = dd + m;
  float* ddf = reinterpret_cast<float*>(e2 + m);
  float* e2f = ddf + m;
  __shared__ double s_lo, s_hi, s_pivmin;
  const int tid = threadIdx.x;
  for (int i = tid; i < m; i += blockDim.x) {
    dd[i] = (double)p.d[i];
    const double ee = (i < m - 1) ? (double)p.e[i] : 0.0;
    e2[i] = ee * ee;
    ddf[i] = p.d[i];
    e2f[i] = (float)(ee * ee);
  }
  // Gershgorin bounds and max e^2: every thread over its rows, then a block reduction
  // (a single thread walking m rows of global e serialised one load latency per row)
  {
    double lo = 1e300, hi = -1e300, emax = 0.0;
    for (int i = tid; i < m; i += blockDim.x) {
      const double r = (i > 0 ? fabs((double)p.e[i - 1]) : 0.0) + (i < m - 1 ? fabs((double)p.e[i]) : 0.0);
      const double di = (double)p.d[i];
      lo = fmin(lo, di - r);
      hi = fmax(hi, di + r);
      if (i < m - 1) emax = fmax(emax, (double)p.e[i] * (double)p.e[i]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
      emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, o));
    }
    __shared__ double s_red[3][BIS_WARPS];
    if ((tid & 31) == 0) { s_red[0][tid >> 5] = lo; s_red[1][tid >> 5] = hi; s_red[2][tid >> 5] = emax; }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < BIS_WARPS; ++w) {
        lo = fmin(lo, s_red[0][w]); hi = fmax(hi, s_red[1][w]); emax = fmax(emax, s_red[2][w]);
      }
      const double span = fmax(fabs(lo), fabs(hi));
      const double pad = 2.2e-16 * span * 4.0 + 1e-300;
      s_lo = lo - pad;
      s_hi = hi + pad;
      s_pivmin = 2.3e-308 * fmax(1.0, emax);
    }
  }
  __syncthreads();
  // BIS_G lanes per eigenvalue (BIS_G probes per round, the bracket cut into BIS_G + 1
  // parts), BIS_E eigenvalues per warp: far fewer Sturm counts per eigenvalue than one
  // eigenvalue per warp (the fp64 phase was fp64-pipe bound), at ~2x the rounds
  const int lane = tid & 31, warp = tid >> 5;
  const int sub = lane / BIS_G, q = lane % BIS_G;
  const int j = (blockIdx.y * BIS_WARPS + warp) * BIS_E + sub;   // descending index
  if ((blockIdx.y * BIS_WARPS + warp) * BIS_E >= p.r) return;    // whole warp idle
  const bool active = j < p.r;
  const int kasc = m - 1 - (active ? j : p.r - 1);                // ascending index
  const unsigned gmask = ((1u << BIS_G) - 1u) << (sub * BIS_G);
  double lo = s_lo, hi = s_hi;
  const double pivmin = s_pivmin;
  // invariant: count(lo) <= kasc < count(hi).  Phase 1: multisection with fp32 Sturm counts
  // (fast reciprocal) down to ~1e-6 of the spectrum's span; phase 2: the bracket, widened by
  // the fp32 counts' backward error, refined with fp64 counts to 1e-10 of the span (fp32
  // outputs; eigenvalues closer than 1e-7 ||T|| are treated as a cluster by stage 4, so
  // inverse iteration never has to separate them).
  const double span = fmax(fabs(lo), fabs(hi));
  constexpr double NP = BIS_G + 1;
  {
    const float pivf = 1e-30f;
    for (int round = 0; round < 24; ++round) {
      const double w = hi - lo;
      const bool go = w > 1e-6 * span;
      if (!__any_sync(0xffffffffu, go)) break;
      const float xf = (float)(lo + w * (double)(q + 1) / NP);
      const int cnt = sturm_count_f32(ddf, e2f, m, xf, pivf);
      const unsigned above = (__ballot_sync(0xffffffffu, cnt >= kasc + 1) & gmask) >> (sub * BIS_G);
      const int first = above ? __ffs(above) - 1 : BIS_G;
      if (go) {
        const double nlo = (first == 0) ? lo : lo + w * (double)first / NP;
        const double nhi = (first == BIS_G) ? hi : lo + w * (double)(first + 1) / NP;
        lo = nlo;
        hi = nhi;
      }
    }
    const double widen = 4e-7 * span * (1.0 + 0.01 * m);
    lo = fmax(lo - widen, s_lo);
    hi = fmin(hi + widen, s_hi);
  }
  for (int round = 0; round < 24; ++round) {
    const double w = hi - lo;
    const bool go = w > 1e-10 * span + pivmin;
    if (!__any_sync(0xffffffffu, go)) break;
    const double x = lo + w * (double)(q + 1) / NP;
    const int cnt = sturm_count(dd, e2, m, x, pivmin);
    const unsigned above = (__ballot_sync(0xffffffffu, cnt >= kasc + 1) & gmask) >> (sub * BIS_G);
    const int first = above ? __ffs(above) - 1 : BIS_G;
    if (go) {
      const double nlo = (first == 0) ? lo : lo + w * (double)first / NP;
      const double nhi = (first == BIS_G) ? hi : lo + w * (double)(first + 1) / NP;
      lo = nlo;
      hi = nhi;
    }
  }
  if (active && q == 0) p.lam[j] = 0.5 * (lo + hi);
}

// ------------------------------------------------------------------ 3. inverse iteration
BKFAC_DEV double hash_unit(unsigned a, unsigned b) {
  unsigned h = a * 0x9E3779B1u ^ (b + 0x7F4A7C15u) * 0x85EBCA77u;
  h ^= h >> 15; h *= 0x2C1B3C6Du; h ^= h >> 12; h *= 0x297A2D39u; h ^= h >> 15;
  return ((double)h / 4294967296.0) - 0.5;
}

// grid: (nprob, ceil(rmax/INV_THREADS)), block INV_THREADS: thread = eigenvector j.
// smem: 2m doubles.  Small blocks spread the latency-bound chains over every SM.
// Chains (pivot recurrence, forward and back substitution) are carried in registers;
// the per-vector arrays are written once per pass and read back in the next pass
// (interleaved a[i*r + j] so a warp's accesses are coalesced).  U's diagonal is stored
// inverted (one division per LU step, none in the substitutions); each iteration is two
// streaming passes: the 2-norm is accumulated during back substitution and the
// normalisation is folded into the next iteration's forward pass (one final scale pass).
constexpr int INV_THREADS = 32;   // one warp per CTA (the norm reduction below assumes it)
#ifndef BKFAC_INV_ITERS
#define BKFAC_INV_ITERS 2
#endif
constexpr int INV_ITERS = BKFAC_INV_ITERS;   // inverse iterations per eigenvector
__global__ void __launch_bounds__(INV_THREADS) invit_kernel(const __grid_constant__ EigBatch b) {
  const EigProb& p = b.p[blockIdx.x];
  const int m = p.m, r = p.r;
  extern __shared__ __align__(16) double ism[];
  double* dd = ism;        // diagonal
  double* ee = dd + m;     // off-diagonal (ee[m-1] = 0)
  __shared__ double s_tiny;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    dd[i] = (double)p.d[i];
    ee[i] = (i < m - 1) ? (double)p.e[i] : 0.0;
  }
  __syncthreads();
  {   // ||T||_inf over the warp (blockDim = 32) instead of one thread walking m rows
    double tn = 0.0;
    for (int i = threadIdx.x; i < m; i += blockDim.x)
      tn = fmax(tn, fabs(dd[i]) + fabs(ee[i]) + (i > 0 ? fabs(ee[i - 1]) : 0.0));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tn = fmax(tn, __shfl_xor_sync(0xffffffffu, tn, o));
    if (threadIdx.x == 0) s_tiny = fmax(tn, 1e-300) * 2.2e-16;
  }
  __syncthreads();
  const int j = blockIdx.y * blockDim.x + threadIdx.x;
  if (j >= r) return;
  const double tiny = s_tiny;
  double* dUi = p.scr;                 // 1 / (U diagonal), fp64 (tiny pivots: huge reciprocals)
  float* du = reinterpret_cast<float*>(dUi + (long)m * r);   // U first superdiagonal (fp32)
  float* du2 = du + (long)m * r;       // U second superdiagonal (fp32)
  float* dl = du2 + (long)m * r;       // multipliers, |f| <= 1 (fp32)
  unsigned char* pv = p.piv;
  double* x = p.Y;
#define AT(a, i) (a)[(long)(i) * r + j]
  if (m == 1) { AT(x, 0) = 1.0; return; }
  const double lam = p.lam[j];
  // LU with partial pivoting of T - lam I (LAPACK dgttrf recurrence), fused with the first
  // iteration's forward pass (L^{-1} with row interchanges on the start vector, which is
  // generated on the fly: deterministic, distinct per eigenvector)
  double dcur = dd[0] - lam;
  double dufcur = ee[0];
  double carry = hash_unit(0u, (unsigned)j) + 0.5;
  // branch-free (threads = eigenvectors pivot differently; selects instead of divergence)
  for (int i = 0; i < m - 1; ++i) {
    const double sub = ee[i];
    const double dnext = dd[i + 1] - lam;
    const double dunext = ee[i + 1];
    const bool sw = fabs(dcur) < fabs(sub);                 // row interchange
    double piv = sw ? sub : dcur;
    if (!sw && fabs(piv) < tiny) piv = (piv >= 0.0) ? tiny : -tiny;
    const double rp = inv_rcp(piv);
    const double f = (sw ? dcur : sub) * rp;
    AT(dUi, i) = rp;
    AT(du, i) = (float)(sw ? dnext : dufcur);
    AT(du2, i) = (float)(sw ? dunext : 0.0);
    AT(dl, i) = (float)f;
    AT(pv, i) = sw ? 1 : 0;
    {
      const double xs = hash_unit((unsigned)(i + 1), (unsigned)j) + 0.5;
      AT(x, i) = sw ? xs : carry;
      carry = sw ? carry - f * xs : xs - f * carry;
    }
    const double ncur = (sw ? dufcur : dnext) - f * (sw ? dnext : dufcur);
    dufcur = sw ? -f * dunext : dunext;
    dcur = ncur;
  }
  if (fabs(dcur) < tiny) dcur = (dcur >= 0.0) ? tiny : -tiny;
  AT(dUi, m - 1) = 1.0 / dcur;
  // Streaming passes in batches of IB entries: the batch's loads are issued together,
  // unguarded (full batches; the ragged end runs entry by entry), and the recurrences are
  // branch-free selects, so one memory latency is exposed per batch instead of per entry.
  constexpr int IB = 16;
  const long R = r;
  double* xj = x + j;
  const double* dUj = dUi + j;
  const float* duj = du + j;
  const float* du2j = du2 + j;
  const float* dlj = dl + j;
  const unsigned char* pvj = pv + j;
  double s = 1.0;   // pending scale of x (applied as x is read in the next pass)
  double nrm = 0.0, amax = 0.0;
  const double carry_lu = carry;
  for (int it = 0; it < INV_ITERS; ++it) {
    // forward: apply L^{-1} with row interchanges; the running entry is carried (the first
    // iteration's forward pass ran inside the LU loop)
    double carry = it == 0 ? carry_lu : xj[0] * s;
    int i0 = it == 0 ? m - 1 : 0;
    for (; i0 + IB <= m - 1; i0 += IB) {
      double xn[IB], f[IB];
      unsigned char pw[IB];
#pragma unroll
      for (int u = 0; u < IB; ++u) {
        xn[u] = xj[(i0 + u + 1) * R];
        f[u] = dlj[(i0 + u) * R];
        pw[u] = pvj[(i0 + u) * R];
      }
#pragma unroll
      for (int u = 0; u < IB; ++u) {
        const double xs = xn[u] * s;
        const bool sw = pw[u] != 0;
        xj[(i0 + u) * R] = sw ? xs : carry;
        carry = sw ? carry - f[u] * xs : xs - f[u] * carry;
      }
    }
    for (; i0 < m - 1; ++i0) {
      const double xs = xj[(i0 + 1) * R] * s, f = (double)dlj[i0 * R];
      const bool sw = pvj[i0 * R] != 0;
      xj[i0 * R] = sw ? xs : carry;
      carry = sw ? carry - f * xs : xs - f * carry;
    }
    // back substitution with U (bandwidth 2); x1, x2 carried; ||x||_2^2 and max|x| on the fly
    double x1 = carry * dUj[(m - 1) * R];
    double x2 = 0.0;
    nrm = x1 * x1;
    amax = fabs(x1);
    xj[(m - 1) * R] = x1;
    int i1 = m - 2;
    for (; i1 - IB + 1 >= 0; i1 -= IB) {
      double xv[IB], a0[IB];
      float a1[IB], a2[IB];
#pragma unroll
      for (int u = 0; u < IB; ++u) {
        const long o = (i1 - u) * R;
        xv[u] = xj[o]; a0[u] = dUj[o]; a1[u] = duj[o]; a2[u] = du2j[o];
      }
#pragma unroll
      for (int u = 0; u < IB; ++u) {
        const double xi = (xv[u] - a1[u] * x1 - a2[u] * x2) * a0[u];
        xj[(i1 - u) * R] = xi;
        x2 = x1;
        x1 = xi;
        nrm = fma(xi, xi, nrm);
        amax = fmax(amax, fabs(xi));
      }
    }
    for (; i1 >= 0; --i1) {
      const long o = i1 * R;
      const double xi = (xj[o] - duj[o] * x1 - du2j[o] * x2) * dUj[o];
      xj[o] = xi;
      x2 = x1;
      x1 = xi;
      nrm = fma(xi, xi, nrm);
      amax = fmax(amax, fabs(xi));
    }
    if (nrm > 0.0 && isfinite(nrm)) {
      s = 1.0 / sqrt(nrm);
    } else {   // ||x||^2 overflowed (or x = 0): scale by 1/max now, renormalise below
      s = (amax > 0.0 && isfinite(amax)) ? 1.0 / amax : 1.0;
      nrm = 0.0;
    }
  }
  if (nrm == 0.0) {   // the last iteration fell back to 1/max: exact 2-norm of s*x
    double t2 = 0.0;
    for (int i = 0; i < m; ++i) { const double t = xj[i * R] * s; t2 = fma(t, t, t2); }
    s = (t2 > 0.0) ? s / sqrt(t2) : 0.0;
  }
  {
    int i = 0;
    for (; i + IB <= m; i += IB) {
      double t[IB];
#pragma unroll
      for (int u = 0; u < IB; ++u) t[u] = xj[(i + u) * R];
#pragma unroll
      for (int u = 0; u < IB; ++u) xj[(i + u) * R] = t[u] * s;
    }
    for (; i < m; ++i) xj[i * R] *= s;
  }
#undef AT
}

// ------------------------------------------------------------------ 4. clusters
// One CTA (32 warps) per problem; clusters are runs of eigenvalues whose consecutive
// gaps are <= 1e-7 * ||T|| (beyond that, two inverse iterations from shifts accurate to
// 1e-10 * span separate the eigenvectors to ~1e-6).  Each warp orthonormalises one
// cluster by modified Gram-Schmidt.
constexpr int CL_BIG = 32;   // clusters longer than this are orthonormalised by the whole CTA
__global__ void __launch_bounds__(1024) cluster_kernel(const __grid_constant__ EigBatch b) {
  const EigProb& p = b.p[blockIdx.x];
  const int m = p.m, r = p.r;
  __shared__ int s_start[1024], s_len[1024], s_n;
  __shared__ int s_bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    double tn = 0.0;
    for (int j = 0; j < r; ++j) tn = fmax(tn, fabs(p.lam[j]));
    for (int i = 0; i < m; ++i) tn = fmax(tn, fabs((double)p.d[i]));
    const double tol = 1e-7 * fmax(tn, 1e-300);
    int n = 0, st = 0;
    for (int j = 1; j <= r; ++j) {
      if (j == r || p.lam[j - 1] - p.lam[j] > tol) {
        if (j - st > 1 && n < 1024) { s_start[n] = st; s_len[n] = j - st; ++n; }
        st = j;
      }
    }
    s_n = n;
    s_bad = 0;
  }
  __syncthreads();
  double* Y = p.Y;
  // small clusters: one warp each, modified Gram-Schmidt in place
  for (int cl = warp; cl < s_n; cl += 32) {
    const int st = s_start[cl], len = s_len[cl];
    if (len > CL_BIG) continue;
    for (int t = st; t < st + len; ++t) {
      for (int s = st; s < t; ++s) {
        double dot = 0.0;
        for (int i = lane; i < m; i += 32) dot += Y[(long)i * r + s] * Y[(long)i * r + t];
        dot = warp_sum_d(dot);
        for (int i = lane; i < m; i += 32) Y[(long)i * r + t] -= dot * Y[(long)i * r + s];
      }
      double nrm = 0.0;
      for (int i = lane; i < m; i += 32) nrm += Y[(long)i * r + t] * Y[(long)i * r + t];
      nrm = warp_sum_d(nrm);
      const double inv = nrm > 0.0 ? 1.0 / sqrt(nrm) : 0.0;
      for (int i = lane; i < m; i += 32) Y[(long)i * r + t] *= inv;
    }
  }
  __syncthreads();
  // large clusters (near-null spaces of rank-deficient updates: hundreds of equal
  // eigenvalues): the whole CTA, one cluster at a time, classical Gram-Schmidt applied twice
  // per vector (CGS2; the projections onto all previous vectors of the cluster are
  // parallel), on a transposed copy in the free inverse-iteration scratch (vector t
  // contiguous: coalesced)
  __shared__ double s_dot[1024];
  double* Yt = p.scr;
  for (int cl = 0; cl < s_n; ++cl) {
    const int st = s_start[cl], len = s_len[cl];
    if (len <= CL_BIG) continue;
    for (int e = tid; e < len * m; e += blockDim.x) {
      const int t = e / m, i = e % m;
      Yt[e] = Y[(long)i * r + st + t];
    }
    __syncthreads();
    for (int t = 0; t < len; ++t) {
      double* yt = Yt + (long)t * m;
      for (int pass = 0; pass < 2; ++pass) {
        for (int s2 = warp; s2 < t; s2 += 32) {
          const double* ys = Yt + (long)s2 * m;
          double dot = 0.0;
          for (int i = lane; i < m; i += 32) dot = fma(ys[i], yt[i], dot);
          dot = warp_sum_d(dot);
          if (lane == 0) s_dot[s2] = dot;
        }
        __syncthreads();
        for (int i = tid; i < m; i += blockDim.x) {
          double acc = 0.0;
          for (int s2 = 0; s2 < t; ++s2) acc = fma(s_dot[s2], Yt[(long)s2 * m + i], acc);
          yt[i] -= acc;
        }
        __syncthreads();
      }
      double nrm = 0.0;
      for (int i = tid; i < m; i += blockDim.x) nrm = fma(yt[i], yt[i], nrm);
      nrm = block_sum_d(nrm, s_dot);
      const double inv = nrm > 0.0 ? 1.0 / sqrt(nrm) : 0.0;
      for (int i = tid; i < m; i += blockDim.x) yt[i] *= inv;
      __syncthreads();
    }
    for (int e = tid; e < len * m; e += blockDim.x) {
      const int t = e / m, i = e % m;
      Y[(long)i * r + st + t] = Yt[e];
    }
    __syncthreads();
  }
  // eigenvalues out (clamped at 0: the core is PSD) + finiteness check
  for (int j = tid; j < r; j += blockDim.x) {
    const double l = p.lam[j];
    if (!isfinite(l)) s_bad = 1;
    p.Dout[j] = (float)fmax(l, 0.0);
  }
  __syncthreads();
  if (tid == 0 && s_bad && p.status) atomicOr(p.status, ST_EIG_FAIL);
}

// ------------------------------------------------------------------ 5. back-transform
// V(:, cols) = H_0 H_1 ... H_{m-3} Y(:, cols); one CTA per (problem, 32 columns);
// warp w owns column w, kept in shared memory (m floats).  smem: 33*m floats.
__global__ void __launch_bounds__(1024) backtr_kernel(const __grid_constant__ EigBatch b) {
  const EigProb& p = b.p[blockIdx.x];
  const int m = p.m, r = p.r;
  const int col0 = blockIdx.y * 32;
  if (col0 >= r) return;
  extern __shared__ __align__(16) float bsm[];
  float* vs = bsm;              // m
  float* Ys = vs + m;           // 32 * m, column w at Ys + w*m
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int j = col0 + warp;
  const bool act = j < r;
  float* yc = Ys + warp * m;
  int bad = 0;
  for (int i = lane; i < m; i += 32) {
    const float v = act ? (float)p.Y[(long)i * r + j] : 0.f;
    bad |= !isfinite(v);
    yc[i] = v;
  }
  for (int k = m - 3; k >= 0; --k) {
    const float tau = p.tau[k];
    __syncthreads();
    if (tau == 0.f) continue;
    for (int i = k + 1 + tid; i < m; i += blockDim.x)
      vs[i] = (i == k + 1) ? 1.f : p.K[i + (long)k * p.ldk];
    __syncthreads();
    float dot = 0.f;
    for (int i = k + 1 + lane; i < m; i += 32) dot = fmaf(vs[i], yc[i], dot);
    dot = warp_sum(dot) * tau;
    for (int i = k + 1 + lane; i < m; i += 32) yc[i] -= dot * vs[i];
  }
  __syncthreads();
  if (act)
    for (int i = lane; i < m; i += 32) p.V[i + (long)j * p.ldv] = yc[i];
  bad = __syncthreads_or(bad);
  if (bad && tid == 0 && p.status) atomicOr(p.status, ST_EIG_FAIL);
}

// ------------------------------------------------------------------ 5'. blocked back-transform
// V = H_0 H_1 ... H_{m-3} Y applied panel by panel (BT_PW reflectors each, compact WY form
// H_{k0} ... H_{k0+PW-1} = I - W T W^T, T upper triangular, LAPACK dlarft 'F','C'):
//   prep   : K's column k becomes the explicit v_k (0 above row k+1, 1 at row k+1; columns
//            k >= m-2 zero), V = (float) Y;
//   S, U   : S_j = W_j^T W_j and U_j = W_j T_j on the tensor-core GEMM; in between the
//            dlarft recurrence T(0:i, i) = -tau_i T(0:i, 0:i) S(0:i, i), T(i, i) = tau_i
//            (one small CTA per panel);
//   apply  : last panel first, Z = W_j^T V and V -= U_j Z on the tensor-core GEMM
//            (bkfac_api.cu).  2 m^2 r flops become two GEMMs per panel instead of m-2
//            sequential rank-1 reflections.
constexpr int BT_PW = 128;
// panels of BT_PW reflectors; reflectors exist for columns k < m - off - 1
__host__ __device__ inline int bt_panels(int m, int off = 1) {
  return m > off + 1 ? (m - off - 1 + BT_PW - 1) / BT_PW : 0;
}

// grid: (nprob, 64), block 256.  (1) Unit upper-triangular top block of every panel's
// reflector block W_j (the rows of W_j above and on its diagonal hold R / band entries):
// zeros above the diagonal, ones on it -- the back-transform's GEMMs read W_j from its top
// block down, nothing else of K.  (2) V = the eigenvectors of T (Zr, fp32 row-major after
// Q2, or Y, fp64 row-major) as col-major fp32, through 32 x 32 shared-memory transposes
// (coalesced on both sides); non-finite entries flag ST_EIG_FAIL.
__global__ void __launch_bounds__(256) backtr_prep_kernel(const __grid_constant__ EigBatch b) {
  const EigProb& p = b.p[blockIdx.x];
  const int m = p.m, r = p.r, off = p.off;
  constexpr int PW = BT_PW;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long nthr = (long)gridDim.y * blockDim.x;
  const long tot = (long)bt_panels(m, off) * PW * PW;
  for (long e = blockIdx.y * (long)blockDim.x + tid; e < tot; e += nthr) {
    const int jp = (int)(e / (PW * PW)), rem = (int)(e % (PW * PW)), c = rem / PW, rr = rem % PW;
    const int k0 = jp * PW, np = min(PW, m - off - 1 - k0);
    if (c >= np || rr > c) continue;
    p.K[(k0 + off + rr) + (long)(k0 + c) * p.ldk] = rr == c ? 1.f : 0.f;
  }
  __shared__ float tile[8][32 * 33];
  float* ts = tile[warp];
  int bad = 0;
  const int ti = (m + 31) / 32, tj = (r + 31) / 32;
  for (int t = blockIdx.y * 8 + warp; t < ti * tj; t += gridDim.y * 8) {
    const int i0 = (t % ti) * 32, j0 = (t / ti) * 32;
    for (int q = 0; q < 32; ++q) {          // row i0 + q, columns j0 + lane
      const int i = i0 + q, j = j0 + lane;
      float v = 0.f;
      if (i < m && j < r) v = p.sbr ? p.Zr[(long)i * r + j] : (float)p.Y[(long)i * r + j];
      ts[q * 33 + lane] = v;
    }
    __syncwarp();
    for (int q = 0; q < 32; ++q) {          // column j0 + q, rows i0 + lane
      const int i = i0 + lane, j = j0 + q;
      if (i < m && j < r) {
        const float v = ts[lane * 33 + q];
        bad |= !isfinite(v);
        p.V[i + (long)j * p.ldv] = v;
      }
    }
    __syncwarp();
  }
  if (bad && p.status) atomicOr(p.status, ST_EIG_FAIL);
}

// grid: (nprob, max panels), block 128: the dlarft recurrence of one panel from its Gram
// matrix S_j = W_j^T W_j (computed by the tensor-core GEMM), T written next to S.
//   T(0:i, i) = -tau_i T(0:i, 0:i) S(0:i, i),  T(i, i) = tau_i
constexpr int BT_THREADS = 128;
inline size_t bt_smem_bytes() { return sizeof(float) * 2 * BT_PW * (BT_PW + 1); }
__global__ void __launch_bounds__(BT_THREADS) backtr_t_kernel(const __grid_constant__ EigBatch b) {
  const EigProb& p = b.p[blockIdx.x];
  const int m = p.m, j = blockIdx.y;
  if (j >= bt_panels(m, p.off)) return;
  constexpr int PW = BT_PW, LD = BT_PW + 1;
  extern __shared__ __align__(16) float btsm[];
  float* S = btsm;
  float* T = S + PW * LD;
  const int tid = threadIdx.x;
  const int k0 = j * PW, np = min(PW, m - p.off - 1 - k0);
  const float* Sg = p.Sw + (long)j * 2 * PW * PW;         // S_j col-major, ld PW
  float* Tg = p.Sw + (long)j * 2 * PW * PW + PW * PW;     // T_j col-major, ld PW
  for (int e = tid; e < PW * PW; e += BT_THREADS) {
    const int a = e % PW, c = e / PW;
    S[a * LD + c] = (a < np && c < np) ? Sg[a + (long)c * PW] : 0.f;
    T[a * LD + c] = 0.f;
  }
  __syncthreads();
  // T^{-1} = diag(1 / tau) + triu(S, 1) (I - W T W^T = H_1 ... H_np): with every tau != 0 each
  // thread inverts one column by back substitution (no block-wide step per reflector),
  //   T(c, c) = tau_c,  T(i, c) = -tau_i sum_{k=i+1..c} S(i, k) T(k, c)  (i = c-1 .. 0);
  // a zero tau (H_i = I) takes the dlarft recurrence instead, one barrier per reflector.
  const bool allnz = __syncthreads_and(tid >= np || p.tau[k0 + tid] != 0.f);
  if (allnz) {
    const int c = tid;
    if (c < np) {
      T[c * LD + c] = p.tau[k0 + c];
      for (int i = c - 1; i >= 0; --i) {
        float s = 0.f;
        for (int k = i + 1; k <= c; ++k) s = fmaf(S[i * LD + k], T[k * LD + c], s);
        T[i * LD + c] = -p.tau[k0 + i] * s;
      }
    }
  } else {
    for (int i = 0; i < np; ++i) {
      const float taui = p.tau[k0 + i];
      if (tid < i) {
        float s = 0.f;
        for (int c = tid; c < i; ++c) s = fmaf(T[tid * LD + c], S[c * LD + i], s);
        T[tid * LD + i] = -taui * s;
      } else if (tid == i) {
        T[i * LD + i] = taui;
      }
      __syncthreads();
    }
  }
  __syncthreads();
  for (int e = tid; e < PW * PW; e += BT_THREADS) {
    const int a = e % PW, c = e / PW;
    Tg[a + (long)c * PW] = T[a * LD + c];
  }
}

}  // namespace bkfac
