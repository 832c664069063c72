// EXPERIMENT (not built): A operand in TMEM via tcgen05.st.  Correct, but measured slower
// than the SS kernel (47 vs 120 TF/s on 8192^3): tcgen05.st into TMEM is starved while the
// MMA pipe is busy, like st.shared.  Kept as a record of the measurement.
// Grouped 3xTF32 GEMM with the A operand in TENSOR MEMORY (tcgen05.mma ... [a_tmem],
// b_desc: the "TS" form), the production kernel of every contraction on the hot path.
//
// Why A lives in TMEM.  Measured on B200 (tools/microbench.cu): while tcgen05.mma streams
// SS operands at full rate (M=128, N=128, kind::tf32: A 4 KB + B 4 KB per 64-cycle MMA =
// 128 B/cycle, all of shared memory's bandwidth) concurrent st.shared from other warps
// get ~0.2 B/cycle -- the operand reads and the loaders' hi/lo stores time-share one
// 128 B/cycle port.  The SS kernel (gemm_tc.cuh) therefore moves 160 KB of shared memory
// per 32-deep chunk (96 KB of 3-pass operand reads + 64 KB of hi/lo stores) against 768
// MMA cycles.  Here the A tile (hi and lo) is written by its loader threads straight into
// TMEM with tcgen05.st (its own datapath, measured 320 B/cycle), so shared memory carries
// only B: 48 KB of operand reads + 32 KB of stores per chunk, under the MMA time.
//
// Layout and roles (BN = 128, one CTA per SM, persistent over all problems' tiles):
//   TMEM columns  [0,128) [128,256)  two K-block accumulators (promotion, see gemm_tc.cuh)
//                 [256,384)          running sum
//                 [384,448) [448,512) A stages: 32 hi + 32 lo columns of 128 lanes (rows)
//   warps 0-3   epilogue (as gemm_tc.cuh)
//   warp  4     TMEM allocation + single-thread MMA issue
//   warps 5-8   A loaders: thread = tile row (TMEM lane 32*(warp%4) + lane); each chunk
//               it loads its row's 32 k-values, splits hi = rna_tf32(x), lo = x - hi,
//               tcgen05.st both into the stage's columns
//   warps 9-12  B loaders: 128-byte lines -> hi/lo into the swizzled smem B stage
// A from TMEM is always "K-major" (lanes = rows, columns = k) whatever the global layout.
#pragma once
#include "gemm_tc.cuh"

namespace bkfac {

constexpr int TS_A_WARP0 = TC_MMA_WARP + 1;   // warps 5..8
constexpr int TS_A_WARPS = 4;
constexpr int TS_B_WARP0 = TS_A_WARP0 + TS_A_WARPS;
constexpr int TS_B_WARPS = 4;
constexpr int TS_THREADS = (TC_EPI_WARPS + 1 + TS_A_WARPS + TS_B_WARPS) * 32;
constexpr int TS_STAGES = 2;
constexpr int TS_BN = 128;
constexpr int TS_B_BYTES = TS_BN * TC_BK * 4;            // one half (hi or lo)
constexpr int TS_STAGE_BYTES = 2 * TS_B_BYTES;
constexpr int TS_SMEM_BYTES = TS_STAGES * TS_STAGE_BYTES + 1024 + 256;
constexpr int TS_TMEM_COLS = 512;
constexpr int TS_ACOL0 = 384;                            // A stage s at 384 + 64 s

BKFAC_DEV void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  const uint32_t* r = reinterpret_cast<const uint32_t*>(v);
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, "
      "%29, %30, %31, %32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
      "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
      "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
BKFAC_DEV void tc_mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(TS_THREADS, 1) gemm_ts_kernel(const __grid_constant__ GemmBatch b) {
  constexpr int BN = TS_BN;
  extern __shared__ __align__(1024) uint8_t ts_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(ts_smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + TS_STAGES * TS_STAGE_BYTES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * TS_STAGES + 4);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar0 = smem_u32(bars);
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (TS_STAGES + s); };
  auto tfull_bar = [&](int a) { return bar0 + 8u * (2 * TS_STAGES + a); };
  auto tempty_bar = [&](int a) { return bar0 + 8u * (2 * TS_STAGES + 2 + a); };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == TC_MMA_WARP) {
    if (lane == 0) {
      for (int s = 0; s < TS_STAGES; ++s) {
        mbar_init(full_bar(s), TS_A_WARPS + TS_B_WARPS);
        mbar_init(empty_bar(s), 1);
      }
      for (int a = 0; a < 2; ++a) {
        mbar_init(tfull_bar(a), 1);
        mbar_init(tempty_bar(a), TC_EPI_WARPS);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"((uint32_t)TS_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == TC_MMA_WARP) {
    // ------------------------------------------------------------- MMA issuer
    constexpr uint32_t IDESC = umma_idesc_tf32<BN>(false, TB);   // A from TMEM: K-major
    constexpr uint32_t STEP_B = TB ? (2u * (BN / 32 * 512)) >> 4 : 2u;
    const uint64_t dBH = tc_op_desc<TB, BN>(sbase, 0);
    const uint64_t dBL = tc_op_desc<TB, BN>(sbase + TS_B_BYTES, 0);
    if (lane == 0) {
      int stage = 0; uint32_t phase = 0;
      int kb = 0;
      for (int t = blockIdx.x; t < b.total_tiles; t += gridDim.x) {
        const TcTile x = tc_tile<BN>(b, t);
        for (int c0 = x.c_beg; c0 < x.c_end; c0 += TC_PROMO, ++kb) {
          const int buf = kb & 1;
          mbar_wait(tempty_bar(buf), ((kb >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t tmem_d = tmem_base + (uint32_t)(buf * BN);
          const int c1 = min(x.c_end, c0 + TC_PROMO);
          for (int c = c0; c < c1; ++c) {
            mbar_wait(full_bar(stage), phase);
            tc_fence_after();
            const uint64_t so = (uint64_t)((stage * TS_STAGE_BYTES) >> 4);
            const uint32_t acol = tmem_base + (uint32_t)(TS_ACOL0 + 64 * stage);
#pragma unroll
            for (int ks = 0; ks < TC_BK / 8; ++ks) {
              const uint32_t aH = acol + 8u * ks, aL = aH + 32u;
              const uint64_t bH = dBH + so + (uint64_t)(ks * STEP_B);
              const uint64_t bL = dBL + so + (uint64_t)(ks * STEP_B);
              const uint32_t first = (c == c0 && ks == 0) ? 0u : 1u;
              tc_mma_tf32_ts(tmem_d, aL, bH, IDESC, first);   // small terms first
              tc_mma_tf32_ts(tmem_d, aH, bL, IDESC, 1u);
              tc_mma_tf32_ts(tmem_d, aH, bH, IDESC, 1u);
            }
            tc_commit(empty_bar(stage));
            if (++stage == TS_STAGES) { stage = 0; phase ^= 1; }
          }
          tc_commit(tfull_bar(buf));
        }
      }
    }
    __syncwarp();
  } else if (warp > TC_MMA_WARP) {
    // ------------------------------------------------------------- loaders
    const bool isA = warp < TS_B_WARP0;
    int stage = 0; uint32_t phase = 0;
    int t = blockIdx.x, c = 0;
    TcTile x;
    auto seek = [&]() {
      while (t < b.total_tiles) {
        if (c == 0) { x = tc_tile<BN>(b, t); c = x.c_beg; }
        if (c < x.c_end) return true;
        t += gridDim.x; c = 0;
      }
      return false;
    };
    struct Seg { const float* p; long ld; int ks, klen; };
    auto seg_of = [&](const GemmProb& p, bool opA) {
      const int s = c < x.nc1 ? 0 : 1;
      Seg g;
      g.ks = (s ? c - x.nc1 : c) * TC_BK;
      g.klen = s ? p.K - p.k1 : p.k1;
      g.p = opA ? (s ? p.A2 : p.A) : (s ? p.B2 : p.B);
      g.ld = opA ? (s ? p.lda2 : p.lda) : (s ? p.ldb2 : p.ldb);
      return g;
    };
    if (isA) {
      // ---- A: thread = row; 32 k-values -> TMEM (hi, lo)
      const int q = warp & 3;                       // TMEM lane quarter of this warp
      const int row = 32 * q + lane;
      auto loadA = [&](float (&v)[32]) {
        const GemmProb& p = b.p[x.pi];
        const Seg g = seg_of(p, true);
        const int i = x.m0 + row;
        const bool rok = i < p.M;
        if (TA) {   // row contiguous along k
          const float* src = g.p + g.ks + (long)i * g.ld;
          if (rok && (p.vec & 1) && g.ks + 32 <= g.klen) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const float4 w = __ldg(reinterpret_cast<const float4*>(src) + u);
              v[4 * u] = w.x; v[4 * u + 1] = w.y; v[4 * u + 2] = w.z; v[4 * u + 3] = w.w;
            }
          } else {
#pragma unroll
            for (int k = 0; k < 32; ++k) v[k] = (rok && g.ks + k < g.klen) ? __ldg(src + k) : 0.f;
          }
        } else {    // rows contiguous along m: one coalesced load per k
          const float* src = g.p + i + (long)g.ks * g.ld;
#pragma unroll
          for (int k = 0; k < 32; ++k) v[k] = (rok && g.ks + k < g.klen) ? __ldg(src + (long)k * g.ld) : 0.f;
        }
      };
      auto storeA = [&](float (&v)[32]) {
        mbar_wait(empty_bar(stage), phase ^ 1);
        tc_fence_after();
        const uint32_t ta = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(TS_ACOL0 + 64 * stage);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {   // 16 columns at a time: hi, then lo in place
          float h[16], l[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) { h[k] = tf32_round(v[16 * hh + k]); l[k] = v[16 * hh + k] - h[k]; }
          tmem_st16(ta + 16 * hh, h);
          tmem_st16(ta + 32 + 16 * hh, l);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(full_bar(stage));
        if (++stage == TS_STAGES) { stage = 0; phase ^= 1; }
      };
      float va[32], vb[32];
      bool have = seek();
      if (have) { loadA(va); ++c; }
      while (have) {
        const bool more = seek();
        if (more) { loadA(vb); ++c; }
        storeA(va);
        if (!more) break;
        const bool more2 = seek();
        if (more2) { loadA(va); ++c; }
        storeA(vb);
        have = more2;
      }
    } else {
      // ---- B: 128-byte lines in quads (as gemm_tc.cuh), hi/lo into the smem stage
      const int lw = warp - TS_B_WARP0;
      constexpr int NQ = BN / 4 / TS_B_WARPS;        // quads per warp (4)
      auto line_src = [&](const GemmProb& p, const Seg& g, int lb, int e, bool& ok) -> const float* {
        if (!TB) { const int j = x.n0 + lb, k = g.ks + e; ok = j < p.N && k < g.klen; return g.p + k + (long)j * g.ld; }
        const int k = g.ks + (lb & 31), j = x.n0 + ((lb >> 5) << 5) + e;
        ok = j < p.N && k < g.klen;
        return g.p + j + (long)k * g.ld;
      };
      auto loadB = [&](float (&v)[4 * NQ], int& vmode) {
        const GemmProb& p = b.p[x.pi];
        const Seg g = seg_of(p, false);
        vmode = p.vec;
#pragma unroll
        for (int qd = 0; qd < NQ; ++qd) {
          const int gq = lw + qd * TS_B_WARPS;
          if (p.vec & 2) {
            const int lb = 4 * gq + (lane >> 3), e0 = (lane & 7) * 4;
            bool ok0, ok3;
            const float* src = line_src(p, g, lb, e0, ok0);
            line_src(p, g, lb, e0 + 3, ok3);
            if (ok0 && ok3) {
              const float4 w = __ldg(reinterpret_cast<const float4*>(src));
              v[4 * qd + 0] = w.x; v[4 * qd + 1] = w.y; v[4 * qd + 2] = w.z; v[4 * qd + 3] = w.w;
            } else {
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                bool ok;
                const float* s1 = line_src(p, g, lb, e0 + u, ok);
                v[4 * qd + u] = ok ? __ldg(s1) : 0.f;
              }
            }
          } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              bool ok;
              const float* s1 = line_src(p, g, 4 * gq + u, lane, ok);
              v[4 * qd + u] = ok ? __ldg(s1) : 0.f;
            }
          }
        }
      };
      auto storeB = [&](const float (&v)[4 * NQ], int vmode) {
        mbar_wait(empty_bar(stage), phase ^ 1);
        const uint32_t st = sbase + stage * TS_STAGE_BYTES;
#pragma unroll
        for (int qd = 0; qd < NQ; ++qd) {
          const int gq = lw + qd * TS_B_WARPS;
          if (vmode & 2) {
            const int lb = 4 * gq + (lane >> 3), e0 = (lane & 7) * 4;
            const uint32_t dh = st + tc_line_off<TB, BN>(lb, e0), dl = dh + TS_B_BYTES;
            float h[4], lo[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) { h[u] = tf32_round(v[4 * qd + u]); lo[u] = v[4 * qd + u] - h[u]; }
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dh), "f"(h[0]), "f"(h[1]), "f"(h[2]), "f"(h[3]));
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dl), "f"(lo[0]), "f"(lo[1]), "f"(lo[2]), "f"(lo[3]));
          } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int lb = 4 * gq + u;
              const float hi = tf32_round(v[4 * qd + u]);
              const uint32_t dh = st + tc_line_off<TB, BN>(lb, lane);
              sts_f32(dh, hi);
              sts_f32(dh + TS_B_BYTES, v[4 * qd + u] - hi);
            }
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(full_bar(stage));
        if (++stage == TS_STAGES) { stage = 0; phase ^= 1; }
      };
      float va[4 * NQ], vb[4 * NQ];
      int ma = 0, mb = 0;
      bool have = seek();
      if (have) { loadB(va, ma); ++c; }
      while (have) {
        const bool more = seek();
        if (more) { loadB(vb, mb); ++c; }
        storeB(va, ma);
        if (!more) break;
        const bool more2 = seek();
        if (more2) { loadB(va, ma); ++c; }
        storeB(vb, mb);
        have = more2;
      }
    }
  } else {
    // ------------------------------------------------------------- epilogue
    tc_epilogue<BN>(b, tmem_base, warp, lane, tfull_bar(0), tfull_bar(1), tempty_bar(0), tempty_bar(1));
  }
  tc_fence_before();
  __syncthreads();
  if (warp == TC_MMA_WARP) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"((uint32_t)TS_TMEM_COLS));
  }
}

template <bool TA, bool TB>
inline bool ts_set_attr() {
  return cudaFuncSetAttribute(gemm_ts_kernel<TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              TS_SMEM_BYTES) == cudaSuccess;
}
inline bool ts_init_attributes() {
  return ts_set_attr<false, false>() && ts_set_attr<false, true>() && ts_set_attr<true, false>() &&
         ts_set_attr<true, true>();
}
template <bool TA, bool TB>
inline void ts_launch(const GemmBatch& b, int grid, cudaStream_t st) {
  gemm_ts_kernel<TA, TB><<<grid, TS_THREADS, TS_SMEM_BYTES, st>>>(b);
}

}  // namespace bkfac
