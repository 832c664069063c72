// Grouped fp32-accurate GEMM on the 5th-generation tensor cores (tcgen05, sm_100a):
// 3xTF32 splitting, operands staged in swizzled shared memory, accumulators in TMEM.
//
// Same problem description as gemm_simt.cuh (GemmProb / GemmBatch, BLAS col-major,
// optional second K segment, deterministic split-K through the same reduce kernel):
//     C = alpha * op(A) op(B) + beta * C0
//
// Why 3xTF32 (SURVEY §8(c) survey probe; BASELINE north_star): every contraction of the
// Brand update, the RSVD and the preconditioner must meet fp32 tolerances; single-pass
// TF32 fails them.  Each fp32 operand x is split as x = hi + lo with hi = rna_tf32(x),
// lo = x - hi (exact in fp32; the tensor core truncates lo to tf32: |x - hi - tf32(lo)|
// <= 2^-21 |x|; rounding lo explicitly measured no better and costs loader issue slots)
// and the product is accumulated as
//     hi_A hi_B + hi_A lo_B + lo_A hi_B       (the lo_A lo_B term is O(2^-22)).
//
// Accumulator promotion.  The tensor core's fp32 accumulate is not round-to-nearest: a
// measured 3xTF32 product with K = 4609 drifted by 3.2e-5 relative (error linear in K,
// i.e. a bias, 25x the SIMT fp32 kernel).  So the MMA accumulates only TC_PROMO chunks
// (TC_PROMO * 32 of K) into a TMEM buffer; the epilogue warps add each such block into a
// running sum (fp32 FADD, round-to-nearest; the running sum itself lives in a third TMEM
// region, tcgen05.ld/st) while the MMA fills the other buffer.  The bias is then bounded
// by one block's length instead of K.  A problem may ask for other block lengths
// (GemmProb::promo; BKFAC_OPT_PREC_BLOCK for the preconditioner's output GEMM).
//
// Kernel anatomy (one CTA per SM, persistent over the tiles of all problems):
//   warps 0-3  epilogue: thread = tile row = TMEM lane; promotes each K-block into the
//              running sum, then alpha/beta and stores coalesced along M (the contiguous
//              dimension of col-major C)
//   warp  4    TMEM allocator + single-thread tcgen05.mma issuer
//   warps 5-12 loaders: coalesced global loads of 128-byte lines (32 fp32 along the
//              contiguous dimension of the operand), hi/lo split in registers, stores of
//              both halves into the 128B-swizzled canonical UMMA layouts.  A line is a
//              K-run of one row for a K-major operand (A transposed, B not transposed)
//              and an MN-run of one k for an MN-major operand; tcgen05 reads either major
//              order for kind::tf32, so no operand is ever transposed.
//   Loaders keep the next chunk's loads in flight while they split and store the current
//   one.  Loaders and the MMA warp hand shared-memory stages over with mbarriers
//   (full: 8 loader warps arrive after fence.proxy.async; empty: tcgen05.commit);
//   the MMA warp and the epilogue hand the two TMEM block buffers over with a second pair.
//
// Why loaders instead of TMA: the leading dimensions on this path are odd (n = 4609,
// 4097, 16385, d_A = 4097 ...), which cuTensorMapEncodeTiled cannot describe (global
// strides must be multiples of 16 bytes), and the split pass has to touch every element
// in registers anyway.  Loading straight from global into the split registers costs one
// shared-memory write per half instead of TMA write + read + write.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "gemm_simt.cuh"

namespace bkfac {

#define BKFAC_GEMM_PATH "tcgen05 kind::tf32 3xTF32 (TMEM accumulators, mbarrier pipeline)"

constexpr int TC_BM = 128;            // UMMA M (TMEM lanes)
constexpr int TC_BK = 32;             // one 128-byte swizzle line of fp32
// Epilogue warps EPI: 4 (warps 0-3, all columns of their TMEM lane quarter) or 8 (warps 0-3
// plus 4 more after the loaders; quarter = warp % 4, each of a quarter's two warps takes half
// the columns).  8 puts twice the C0/C traffic in flight per SM -- for stages whose K is
// short (<= 8 chunks), where the epilogue, not the MMA, sets the pace (the EA accumulate,
// the residual) -- at the price of 72 instead of 80 registers per thread.
constexpr int TC_MMA_WARP = 4;
#ifndef BKFAC_TC_PROMO
#define BKFAC_TC_PROMO 8     // 256 of K per TMEM block (4: 1.4 % slower at cfg4, same tests)
#endif
#ifndef BKFAC_TC_NLW
#define BKFAC_TC_NLW 16
#endif
#ifndef BKFAC_TC_DEPTH
#define BKFAC_TC_DEPTH 1
#endif
#ifdef BKFAC_TC_DEBUG_NOLOAD          // tuning only: loaders skip global memory
#define TC_LDG(ptr) (1.0f + (float)lane)
#else
#define TC_LDG(ptr) __ldg(ptr)
#endif
constexpr int TC_PROMO = BKFAC_TC_PROMO;   // K chunks accumulated in TMEM before promotion

// NLW loader warps, each keeping DEPTH chunks of loads in flight ahead of its stores.
// PAIR: a CTA pair (cluster of 2, tcgen05 cta_group::2) computes a 256 x BN tile: each CTA
// stages its own 128 rows of A and BN/2 rows of B, the leader issues M = 256 MMAs that read
// both CTAs' shared memory, and each CTA's TMEM holds its 128 rows of the accumulator.
// Per SM per chunk: 1/4 fewer loads and stores, B operand reads halved.
template <int BN, int NLW = 16, int DEPTH = 2, int EPI = 4, bool PAIR = false>
struct TcCfg {
  static constexpr int LOAD_WARPS = NLW;
  static constexpr int EPI_WARPS = EPI;
  static constexpr int THREADS = (EPI + 1 + NLW) * 32;
  static constexpr int BM_T = PAIR ? 2 * TC_BM : TC_BM;     // tile rows (both CTAs)
  static constexpr int B_ROWS = PAIR ? BN / 2 : BN;          // B rows staged by this CTA
  static constexpr int A_BYTES = TC_BM * TC_BK * 4;          // one half (hi or lo)
  static constexpr int B_BYTES = B_ROWS * TC_BK * 4;
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
#ifdef BKFAC_TC_STAGES
  static constexpr int STAGES = BKFAC_TC_STAGES;
#else
  static constexpr int STAGES = PAIR ? ((BN >= 256) ? 3 : 4) : ((BN >= 256) ? 2 : 3);
#endif
  // TMEM: BN <= 128: two K-block buffers + a running-sum region (4 BN columns, a power of
  // two).  BN = 256 ("swap" protocol, see tc_epilogue): two BN-column buffers whose roles
  // alternate per tile -- the running sum of tile t lives in buffer t & 1, its K-blocks after
  // the first accumulate in the other one -- so a 256-wide tile fits the 512 TMEM columns.
  static constexpr bool SWAP = BN >= 256;
  static constexpr int TMEM_COLS = SWAP ? 2 * BN : 4 * BN;
  static constexpr int LINES = TC_BM + B_ROWS;               // 128-byte lines per stage half
  static constexpr int LPW = LINES / NLW;                    // lines per loader warp
  // quads of A lines and of B lines never mix in one loader-warp quad slot
  static_assert(TC_BM % (4 * NLW) == 0 && B_ROWS % (4 * NLW) == 0, "loader quad split");
  // + per-epilogue-warp 16 x 34 staging for the transposed (mirror) stores of symmetric tiles
  static constexpr int EPI_STAGE_FLOATS = 16 * 34;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ +
                                    EPI * EPI_STAGE_FLOATS * 4;
};

// ----------------------------------------------------------------------- PTX helpers
BKFAC_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
BKFAC_DEV void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
BKFAC_DEV void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
BKFAC_DEV void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// Waiter that does not need to react within tens of cycles (the epilogue): the thread is
// suspended until the phase completes or ~the hint (ns) elapses instead of spinning, so
// it does not steal issue slots from the loader warps.
BKFAC_DEV void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAITS_%=;\n\t}" ::"r"(bar),
      "r"(parity), "r"(1000000u)
      : "memory");
}
BKFAC_DEV void sts_f32(uint32_t addr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v));
}
BKFAC_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
BKFAC_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
BKFAC_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
BKFAC_DEV void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
BKFAC_DEV void tc_commit2(uint32_t bar) {   // both CTAs of the pair (same smem offset)
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
      ::"r"(bar), "h"((uint16_t)3) : "memory");
}
BKFAC_DEV void tc_mma2_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on the mbarrier at the same offset in CTA `rank` of the cluster (release.cluster)
BKFAC_DEV void mbar_arrive_remote(uint32_t bar, uint32_t rank) {
  uint32_t rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(bar), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rb) : "memory");
}
BKFAC_DEV void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAITC_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
BKFAC_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
BKFAC_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
BKFAC_DEV void tc_mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Round to the nearest tf32 (ties away from zero) in two integer ops; non-finite values
// stay non-finite (NaN stays NaN, +-inf stays +-inf) so status checks still see them.
BKFAC_DEV float tf32_round(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
BKFAC_DEV float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// 32 consecutive fp32 TMEM columns of this thread's lane
BKFAC_DEV void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
      "%28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// 16 consecutive fp32 TMEM columns of this thread's lane
BKFAC_DEV void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Two 16-column loads (a K-block accumulator and the running sum) in flight together, one wait.
#ifndef BKFAC_TC_LD2
#define BKFAC_TC_LD2 1
#endif
BKFAC_DEV void tmem_ld16x2(uint32_t ta, uint32_t tb, float (&v)[16], float (&w)[16]) {
#if !BKFAC_TC_LD2
  tmem_ld16(ta, v);
  tmem_ld16(tb, w);
  return;
#endif
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  uint32_t* q = reinterpret_cast<uint32_t*>(w);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%32];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, "
      "%26, %27, %28, %29, %30, %31}, [%33];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]),
        "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]),
        "=r"(q[7]), "=r"(q[8]), "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]), "=r"(q[13]),
        "=r"(q[14]), "=r"(q[15])
      : "r"(ta), "r"(tb)
      : "memory");
}

BKFAC_DEV void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  const uint32_t* r = reinterpret_cast<const uint32_t*>(v);
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

// UMMA shared-memory descriptor (SM100 "version 1").  layout: 2 = SWIZZLE_128B (K-major
// operands: 8 rows x 128 B atoms, 16-byte chunks XOR row%8), 1 = SWIZZLE_128B_BASE32B
// (MN-major tf32 operands -- the only MN-major layout kind::tf32 accepts: 4 k-rows x 128 B
// atoms, 32-byte chunks XOR k%4).
BKFAC_DEV uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // version (sm_100)
  d |= (uint64_t)layout << 61;
  return d;
}
// Byte offset of element e (0..31) of 128-byte line l inside one operand buffer of R
// MN-rows.  K-major: line = MN row (32 consecutive k).  MN-major: line = (k-line kk,
// MN atom a) with l = a*32 + kk (32 consecutive MN indices at fixed k).
template <bool MN, int R>
BKFAC_DEV uint32_t tc_line_off(int l, int e) {
  if (!MN) return l * 128u + (((uint32_t)(e >> 2) ^ (uint32_t)(l & 7)) << 4) + ((e & 3) << 2);
  const int kk = l & 31, a = l >> 5;
  return (uint32_t)(kk >> 2) * (uint32_t)(R / 32 * 512) + a * 512u + (kk & 3) * 128u +
         (((uint32_t)(e >> 3) ^ (uint32_t)(kk & 3)) << 5) + ((e & 7) << 2);
}
// Descriptor of k-step ks (8 k = one tf32 MMA) of an operand buffer at saddr.
template <bool MN, int R>
BKFAC_DEV uint64_t tc_op_desc(uint32_t saddr, int ks) {
  if (!MN) return umma_desc(saddr + ks * 32u, 16u, 1024u, 2u);
  return umma_desc(saddr + ks * 2u * (R / 32 * 512), 512u, R / 32 * 512, 1u);
}
// Instruction descriptor: kind::tf32, fp32 accumulate, M = 128, N = BN.
template <int BN, int BMM = TC_BM>
BKFAC_DEV constexpr uint32_t umma_idesc_tf32(bool a_mn_major, bool b_mn_major) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn_major ? 1u : 0u) << 15) |
         ((b_mn_major ? 1u : 0u) << 16) | ((uint32_t)(BN >> 3) << 17) |
         ((uint32_t)(BMM >> 4) << 24);
}

// ----------------------------------------------------------------------- tile walk
struct TcTile {
  int pi, m0, n0, split, c_beg, c_end, nc1;
};

BKFAC_DEV int tc_find_prob(const GemmBatch& b, int t) {
  int lo = 0, hi = b.nprob - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (b.p[mid].tile_start <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}

template <int BN, int BMT = TC_BM>
BKFAC_DEV TcTile tc_tile(const GemmBatch& b, int t) {
  TcTile x;
  x.pi = tc_find_prob(b, t);
  const GemmProb& p = b.p[x.pi];
  const int lt = t - p.tile_start;
  const int per_split = p.sym ? p.tiles_m * (p.tiles_m + 1) / 2 : p.tiles_m * p.tiles_n;
  x.split = lt / per_split;
  const int rem = lt - x.split * per_split;
  if (p.sym) {   // lower-triangular tile (tm >= tn), rem = tm (tm + 1) / 2 + tn
    int tm = (int)((sqrtf(8.f * rem + 1.f) - 1.f) * 0.5f);
    while (tm * (tm + 1) / 2 > rem) --tm;
    while ((tm + 1) * (tm + 2) / 2 <= rem) ++tm;
    x.m0 = tm * BMT;
    x.n0 = (rem - tm * (tm + 1) / 2) * BN;
  } else if (p.nfast) {
    x.n0 = (rem % p.tiles_n) * BN;
    x.m0 = (rem / p.tiles_n) * BMT;
  } else {
    x.m0 = (rem % p.tiles_m) * BMT;
    x.n0 = (rem / p.tiles_m) * BN;
  }
  x.nc1 = (p.k1 + TC_BK - 1) / TC_BK;
  const int nc = x.nc1 + (p.K - p.k1 + TC_BK - 1) / TC_BK;
  x.c_beg = min(nc, x.split * p.kchunk);     // kchunk = chunks per split on this path
  x.c_end = min(nc, x.c_beg + p.kchunk);
  return x;
}

#ifdef BKFAC_TC_TIMING
__device__ unsigned long long g_tc_dbg[148 * 8];   // tuning builds: per-CTA MMA-warp cycle sums
#endif
// Output of one 16-column group of a finished tile (thread = row i): split-K partials
// into w, or C = alpha v + beta C0 (coalesced along M), plus the mirrored tile of a symmetric
// problem through the warp's staging buffer.
BKFAC_DEV void tc_store_group(const GemmProb& p, const TcTile& x, int g, float (&v)[16], int i,
                              int quarter, int lane, float beta, float* w, float* stage,
                              bool& nonfinite) {
  if (w) {
    if (i < p.M) {
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) {
        const int j = x.n0 + g * 16 + jj;
        if (j < p.N) w[i + (long)j * p.M] = v[jj];
      }
    }
    return;
  }
  const bool rowok = i < p.M;
  const int j0 = x.n0 + g * 16;
  // all 16 C0 loads of the group in flight together (each thread reads only the elements
  // it writes, so this is safe when C0 aliases C)
  float c0v[16];
  if (beta != 0.f) {
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) {
      const float* q = p.C0 + i + (long)(j0 + jj) * p.ldc0;
      c0v[jj] = (rowok && j0 + jj < p.N) ? (p.stream_c ? __ldcs(q) : *q) : 0.f;
    }
  }
  // alpha v + beta C0 on pairs (FMUL2 / FFMA2: the same per-element roundings as the scalar
  // o = alpha v; o += beta c0); fused scalings (device alpha, row / column scale, diagonal)
  const float ra = gemm_row_alpha(p, i);
  const float2 be2 = make_float2(beta, beta);
#pragma unroll
  for (int jj = 0; jj < 16; jj += 2) {
    float2 al2 = make_float2(ra, ra);
    if (p.col_scale) {
      al2.x *= (j0 + jj < p.N) ? p.col_scale[j0 + jj] : 0.f;
      al2.y *= (j0 + jj + 1 < p.N) ? p.col_scale[j0 + jj + 1] : 0.f;
    }
    float2 o = __fmul2_rn(al2, make_float2(v[jj], v[jj + 1]));
    if (beta != 0.f) {
      nonfinite |= !isfinite(c0v[jj]) | !isfinite(c0v[jj + 1]);
      o = __ffma2_rn(be2, make_float2(c0v[jj], c0v[jj + 1]), o);
    }
    if (p.diag_vec && i < p.diag_n) {
      if (i == j0 + jj) o.x += p.diag_a * p.diag_vec[i];
      if (i == j0 + jj + 1) o.y += p.diag_a * p.diag_vec[i];
    }
    float* q = p.C + i + (long)(j0 + jj) * p.ldc;
    if (p.stream_c) {
      if (rowok && j0 + jj < p.N) __stcs(q, o.x);
      if (rowok && j0 + jj + 1 < p.N) __stcs(q + p.ldc, o.y);
    } else {
      if (rowok && j0 + jj < p.N) *q = o.x;
      if (rowok && j0 + jj + 1 < p.N) q[p.ldc] = o.y;
    }
    v[jj] = o.x; v[jj + 1] = o.y;
  }
  if (p.sym == 1 && x.m0 != x.n0) {
    // mirror tile C(j, i) = C(i, j): transposed through a warp-private staging buffer so
    // that each store instruction writes two 64-byte column runs instead of 32 scattered words
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) stage[jj * 34 + lane] = v[jj];
    __syncwarp();
#pragma unroll 4
    for (int q = 0; q < 16; ++q) {
      const int jj = lane & 15, rr = 2 * q + (lane >> 4);
      const int ir = x.m0 + quarter * 32 + rr, jc = j0 + jj;
      if (ir < p.M && jc < p.N) p.C[jc + (long)ir * p.ldc] = stage[jj * 34 + rr];
    }
    __syncwarp();
  }
}

// Epilogue, BN <= 128 protocol -- warps 0-3 (thread = tile row = TMEM lane): promote each K-block accumulator
// into the running sum (TMEM), then alpha/beta and coalesced stores of the tile.
template <int BN, int EPI, bool PAIR, int NLW_EPI>
BKFAC_DEV void tc_epilogue(const GemmBatch& b, uint32_t tmem_base, int warp, int lane,
                           uint32_t tfull0, uint32_t tfull1, uint32_t tempty0, uint32_t tempty1,
                           float* stage) {
  constexpr int BMT = PAIR ? 2 * TC_BM : TC_BM;
  const uint32_t crank = PAIR ? cluster_rank() : 0u;
  const int tstride = PAIR ? (int)gridDim.x / 2 : (int)gridDim.x;
  const int tfirst = PAIR ? (int)blockIdx.x / 2 : (int)blockIdx.x;
  auto tfull_bar = [&](int a) { return a ? tfull1 : tfull0; };
  auto tempty_bar = [&](int a) { return a ? tempty1 : tempty0; };
    const int quarter = warp & 3;                             // TMEM lanes this warp may access
    const int row = quarter * 32 + lane;                      // TMEM lane = tile row
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t run = tmem_base + lane_off + 2 * BN;       // running-sum columns
    // column groups of this warp: all, or one half when two warps share the quarter
    // EPI = 4, 8 or 16 warps: warps 0-3 and, after the loaders, groups of 4 consecutive warps
    // (one per TMEM lane quarter); slice = which of the EPI / 4 column slices this warp takes
    constexpr int NG = BN / 16, GPW = NG * 4 / EPI;
    static_assert(EPI == 4 || EPI == 8 || EPI == 16, "epilogue warps");
    const int eidx = warp < 4 ? warp : 4 + (warp - (TC_MMA_WARP + 1 + NLW_EPI));
    const int g_beg = (eidx >> 2) * GPW;
    int kb = 0;
    int tl = 0, jf0 = 0, jf1 = 0;   // swap protocol: local tile count, full waits per buffer
    for (int t = tfirst; t < b.total_tiles; t += tstride) {
      TcTile x = tc_tile<BN, BMT>(b, t);
      x.m0 += (int)crank * TC_BM;                              // this CTA's 128 rows
      const GemmProb& p = b.p[x.pi];
      const int pro = p.promo > 0 ? p.promo : TC_PROMO;
      const int nblk = (x.c_end - x.c_beg + pro - 1) / pro;
      const int i = x.m0 + row;
      bool nonfinite = false;   // inf/NaN in C0 (the operands' tensor-core path cannot report it)
      const float beta = p.beta_dev ? *p.beta_dev : p.beta;
      float* w = p.splits > 1 ? p.ws + (long)x.split * p.M * p.N : nullptr;
      // C0 of this warp's rows x columns into L2 while the tile's K loop runs: the final
      // epilogue then waits for L2, not HBM, on each of its column groups
      if (!w && beta != 0.f && nblk > 0) {
        const int r0 = x.m0 + quarter * 32;
        if (r0 < p.M) {
          const int r1 = min(r0 + 31, p.M - 1);
          for (int c = lane; c < 16 * GPW; c += 32) {
            const int j = x.n0 + g_beg * 16 + c;
            if (j >= p.N) break;
            const float* col = p.C0 + (long)j * p.ldc0;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(col + r0));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(col + r1));
          }
        }
      }
      if constexpr (BN >= 256) {
        // "swap" protocol: the tile's running sum lives in buffer sb = (local tile) & 1 --
        // its first K-block is accumulated there directly -- and every later K-block in
        // buffer ab = sb ^ 1, which is released as soon as it has been read (S += A), so the
        // MMA stalls only for that TMEM pass.  The next tile's sum buffer is this tile's ab;
        // this tile's sb is released after the tile's output, one K-block of slack later.
        const int sb = tl & 1, ab = sb ^ 1;
        ++tl;
        if (nblk > 0) {
          auto waitfull = [&](int bf) {
            int& j = bf ? jf1 : jf0;
            mbar_wait_sleep(tfull_bar(bf), j & 1);
            ++j;
            tc_fence_after();
          };
          auto release = [&](int bf) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              if (PAIR && crank != 0) mbar_arrive_remote(tempty_bar(bf), 0);   // the leader's
              else mbar_arrive(tempty_bar(bf));
            }
          };
          const uint32_t Ssum = tmem_base + lane_off + (uint32_t)(sb * BN);
          const uint32_t Aacc = tmem_base + lane_off + (uint32_t)(ab * BN);
          waitfull(sb);
          for (int blk = 1; blk < nblk; ++blk) {
            waitfull(ab);
#pragma unroll 1
            for (int g = g_beg; g < g_beg + GPW; ++g) {
              float v[16], r[16];
              tmem_ld16x2(Aacc + g * 16, Ssum + g * 16, v, r);
#pragma unroll
              for (int j = 0; j < 16; j += 2) {   // FADD2: same round-to-nearest per element
                const float2 t2 = __fadd2_rn(make_float2(v[j], v[j + 1]), make_float2(r[j], r[j + 1]));
                v[j] = t2.x; v[j + 1] = t2.y;
              }
              tmem_st16(Ssum + g * 16, v);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            release(ab);
          }
#pragma unroll 1
          for (int g = g_beg; g < g_beg + GPW; ++g) {
            if (x.n0 + g * 16 >= p.N) break;      // warp-uniform
            float v[16];
            tmem_ld16(Ssum + g * 16, v);
            tc_store_group(p, x, g, v, i, quarter, lane, beta, w, stage, nonfinite);
          }
          release(sb);
        }
      } else
      for (int blk = 0; blk < nblk; ++blk, ++kb) {
        const int buf = kb & 1;
        const bool last = blk == nblk - 1;
        mbar_wait_sleep(tfull_bar(buf), (kb >> 1) & 1);
        tc_fence_after();
        const uint32_t src = tmem_base + lane_off + (uint32_t)(buf * BN);
#pragma unroll 1
        for (int g = g_beg; g < g_beg + GPW; ++g) {
          if (last && x.n0 + g * 16 >= p.N) break;      // warp-uniform
#ifdef BKFAC_TC_DEBUG_NOEPI
          if (!last) break;                             // tuning only: skip promotion
#endif
          float v[16];
          if (blk > 0) {
            float r[16];
            tmem_ld16x2(src + g * 16, run + g * 16, v, r);
#pragma unroll
            for (int j = 0; j < 16; j += 2) {   // FADD2: same round-to-nearest per element
              const float2 t = __fadd2_rn(make_float2(v[j], v[j + 1]), make_float2(r[j], r[j + 1]));
              v[j] = t.x; v[j + 1] = t.y;
            }
          } else {
            tmem_ld16(src + g * 16, v);
          }
          if (!last) tmem_st16(run + g * 16, v);
          else tc_store_group(p, x, g, v, i, quarter, lane, beta, w, stage, nonfinite);
        }
        if (!last) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (PAIR && crank != 0) mbar_arrive_remote(tempty_bar(buf), 0);   // the leader's
          else mbar_arrive(tempty_bar(buf));
        }
      }
      if (p.status && __any_sync(0xffffffffu, nonfinite) && lane == 0) atomicOr(p.status, ST_NONFINITE);
      if (nblk == 0 && i < p.M) {     // empty K range (split beyond K or K = 0)
        for (int j = x.n0 + 16 * g_beg; j < min(p.N, x.n0 + 16 * (g_beg + GPW)); ++j) {
          if (w) {
            w[i + (long)j * p.M] = 0.f;
          } else {
            p.C[i + (long)j * p.ldc] = gemm_out(p, i, j, 0.f, 0.f, beta);
          }
        }
      }
    }
  }

// ----------------------------------------------------------------------- kernel
template <bool TA, bool TB, int BN, int NLW, int DEPTH, int EPI, bool PAIR>
__global__ void __launch_bounds__(TcCfg<BN, NLW, DEPTH, EPI, PAIR>::THREADS, 1)
gemm_tc_kernel(const __grid_constant__ GemmBatch b) {
  using Cfg = TcCfg<BN, NLW, DEPTH, EPI, PAIR>;
  constexpr int BMT = Cfg::BM_T, B_ROWS = Cfg::B_ROWS;
  const uint32_t crank = PAIR ? cluster_rank() : 0u;
  const int tstride = PAIR ? (int)gridDim.x / 2 : (int)gridDim.x;
  const int tfirst = PAIR ? (int)blockIdx.x / 2 : (int)blockIdx.x;
  constexpr int TC_LOAD_WARPS = NLW;
  extern __shared__ __align__(1024) uint8_t tc_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  // bars: full[S], empty[S], tfull[2], tempty[2], pfull[S] (PAIR peer: its loaders' local
  // barrier, forwarded to the leader by the peer's MMA warp); then the TMEM base address
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * Cfg::STAGES + 4);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar0 = smem_u32(bars);
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (Cfg::STAGES + s); };
  auto tfull_bar = [&](int a) { return bar0 + 8u * (2 * Cfg::STAGES + a); };
  auto tempty_bar = [&](int a) { return bar0 + 8u * (2 * Cfg::STAGES + 2 + a); };
  auto pfull_bar = [&](int s) { return bar0 + 8u * (2 * Cfg::STAGES + 4 + s); };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == TC_MMA_WARP) {
    if (lane == 0) {
      for (int s = 0; s < Cfg::STAGES; ++s) {
        mbar_init(full_bar(s), PAIR ? TC_LOAD_WARPS + 1 : TC_LOAD_WARPS);   // + the peer's forward
        mbar_init(empty_bar(s), 1);
        mbar_init(pfull_bar(s), TC_LOAD_WARPS);
      }
      for (int a = 0; a < 2; ++a) {
        mbar_init(tfull_bar(a), 1);
        mbar_init(tempty_bar(a), PAIR ? 2 * EPI : EPI);                      // + the peer's epilogue
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"((uint32_t)Cfg::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"((uint32_t)Cfg::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  if (PAIR) cluster_sync_all();   // both CTAs' barriers initialised before any remote arrive
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == TC_MMA_WARP) {
    // ------------------------------------------------------------- MMA issuer
    constexpr uint32_t IDESC = umma_idesc_tf32<BN, BMT>(!TA, TB);
    // k-step strides of the start-address field: K-major 32 B, MN-major two 4-row groups
    constexpr uint32_t STEP_A = TA ? 2u : (2u * (TC_BM / 32 * 512)) >> 4;
    constexpr uint32_t STEP_B = TB ? (2u * (B_ROWS / 32 * 512)) >> 4 : 2u;
    const uint64_t dAH = tc_op_desc<!TA, TC_BM>(sbase, 0);
    const uint64_t dAL = tc_op_desc<!TA, TC_BM>(sbase + Cfg::A_BYTES, 0);
    const uint64_t dBH = tc_op_desc<TB, B_ROWS>(sbase + 2 * Cfg::A_BYTES, 0);
    const uint64_t dBL = tc_op_desc<TB, B_ROWS>(sbase + 2 * Cfg::A_BYTES + Cfg::B_BYTES, 0);
    // one thread runs the whole issue loop: the tensor pipe's instruction queue is shallow,
    // so every cycle the issuer spends on warp-wide waits or shuffles is pipe idle time.
    // PAIR: the leader issues for both CTAs; the peer's MMA warp only owns its TMEM
    if (lane == 0 && (!PAIR || crank == 0)) {
      int stage = 0; uint32_t phase = 0;
      int kb = 0;   // K-block counter over all tiles of this CTA (TMEM buffer = kb & 1)
      int tl = 0, u0 = 0, u1 = 0;   // swap protocol (BN = 256): local tile, fills per buffer
      for (int t = tfirst; t < b.total_tiles; t += tstride, ++tl) {
        const TcTile x = tc_tile<BN, BMT>(b, t);
        // single-CTA tiles: the instruction's N shrinks to the tile's valid columns (rounded to
        // 16) -- a narrow problem (N = 32: the band reduction's X = A22 V) costs N / BN of
        // the MMA time.  Pair tiles keep N = BN (each CTA stages half of B's rows).
        uint32_t idesc = IDESC;
        if (!PAIR) {
          const int nv = min(BN, ((b.p[x.pi].N - x.n0 + 15) >> 4) << 4);
          idesc = (IDESC & ~(0x3Fu << 17)) | ((uint32_t)(nv >> 3) << 17);
        }
        const int pro = b.p[x.pi].promo > 0 ? b.p[x.pi].promo : TC_PROMO;
        for (int c0 = x.c_beg; c0 < x.c_end; c0 += pro, ++kb) {
          // swap: first K-block of the tile into its sum buffer (tl & 1), the others into
          // the other buffer (see tc_epilogue)
          const int buf = Cfg::SWAP ? ((c0 == x.c_beg) ? (tl & 1) : ((tl & 1) ^ 1)) : (kb & 1);
          int use = (kb >> 1);
          if (Cfg::SWAP) { int& u = buf ? u1 : u0; use = u; ++u; }
#ifdef BKFAC_TC_TIMING
          unsigned long long t0 = clock64();
#endif
          if (PAIR) mbar_wait_cluster(tempty_bar(buf), (use & 1) ^ 1);
          else mbar_wait(tempty_bar(buf), (use & 1) ^ 1);
#ifdef BKFAC_TC_TIMING
          g_tc_dbg[blockIdx.x * 8 + 0] += clock64() - t0;
#endif
          tc_fence_after();
          const uint32_t tmem_d = tmem_base + (uint32_t)(buf * BN);
          const int c1 = min(x.c_end, c0 + pro);
          for (int c = c0; c < c1; ++c) {
#ifdef BKFAC_TC_TIMING
            unsigned long long t1 = clock64();
#endif
#ifndef BKFAC_TC_DEBUG_NOFULLWAIT
            if (PAIR) mbar_wait_cluster(full_bar(stage), phase);
            else mbar_wait(full_bar(stage), phase);
#endif
#ifdef BKFAC_TC_TIMING
            unsigned long long t2 = clock64();
            g_tc_dbg[blockIdx.x * 8 + 1] += t2 - t1;
#endif
            tc_fence_after();
            // descriptors: precomputed stage-0 bases + (stage, k-step) offsets in 16-byte
            // units (start-address field; smem < 256 KB, so no carry out of the field)
            const uint64_t so = (uint64_t)((stage * Cfg::STAGE_BYTES) >> 4);
#pragma unroll
            for (int ks = 0; ks < TC_BK / 8; ++ks) {
              const uint64_t aH = dAH + so + (uint64_t)(ks * STEP_A);
              const uint64_t aL = dAL + so + (uint64_t)(ks * STEP_A);
              const uint64_t bH = dBH + so + (uint64_t)(ks * STEP_B);
              const uint64_t bL = dBL + so + (uint64_t)(ks * STEP_B);
              const uint32_t first = (c == c0 && ks == 0) ? 0u : 1u;
#ifndef BKFAC_TC_DEBUG_ONEPASS
              if (PAIR) {
                tc_mma2_tf32(tmem_d, aL, bH, IDESC, first);
                tc_mma2_tf32(tmem_d, aH, bL, IDESC, 1u);
                tc_mma2_tf32(tmem_d, aH, bH, IDESC, 1u);
              } else {
                tc_mma_tf32(tmem_d, aL, bH, idesc, first);   // small terms first
                tc_mma_tf32(tmem_d, aH, bL, idesc, 1u);
                tc_mma_tf32(tmem_d, aH, bH, idesc, 1u);
              }
#else                                     // tuning only: 1xTF32 (MMA-rate probe)
              tc_mma_tf32(tmem_d, aH, bH, idesc, first);
#endif
            }
            if (PAIR) tc_commit2(empty_bar(stage)); else tc_commit(empty_bar(stage));
#ifdef BKFAC_TC_TIMING
            g_tc_dbg[blockIdx.x * 8 + 2] += clock64() - t2;
            g_tc_dbg[blockIdx.x * 8 + 3] += 1;
#endif
            if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
          }
          if (PAIR) tc_commit2(tfull_bar(buf)); else tc_commit(tfull_bar(buf));
        }
      }
    } else if (PAIR && lane == 0) {
      // the peer's MMA warp: one cluster-scope arrive per stage on the leader's full barrier
      // once all of this CTA's loader warps have filled it (one release.cluster instead of
      // sixteen)
      int stage = 0; uint32_t phase = 0;
      for (int t = tfirst; t < b.total_tiles; t += tstride) {
        const TcTile x = tc_tile<BN, BMT>(b, t);
        for (int c = x.c_beg; c < x.c_end; ++c) {
          mbar_wait(pfull_bar(stage), phase);
          mbar_arrive_remote(full_bar(stage), 0);
          if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp > TC_MMA_WARP && warp <= TC_MMA_WARP + NLW) {
    // ------------------------------------------------------------- loaders
    const int lw = warp - TC_MMA_WARP - 1;
    int stage = 0; uint32_t phase = 0;
    // the (tile, chunk) sequence of this CTA, walked one step ahead of the stores
    int t = tfirst, c = 0;
    TcTile x;
    auto seek = [&]() {   // advance (t, c) to the next existing chunk; false when done
      while (t < b.total_tiles) {
        if (c == 0) {
          x = tc_tile<BN, BMT>(b, t);
          x.m0 += (int)crank * TC_BM;      // PAIR: this CTA's 128 rows of A ...
          x.n0 += (int)crank * B_ROWS;     // ... and its half of B
          c = x.c_beg;
        }
        if (c < x.c_end) return true;
        t += tstride; c = 0;
      }
      return false;
    };
    // Lines are handled in quads (4 consecutive lines; quad g = lw + qd * NLW).  A quad
    // whose operand is 16-byte aligned (base and leading dimension) is loaded with one
    // LDG.128 per lane (lane: line 4g + lane/8, elements 4*(lane%8) .. +3) and stored with
    // STS.128; otherwise with four coalesced LDG.32 (lane = element of each of the 4
    // lines) and scalar stores.  Both keep 4 values per lane per quad.
    constexpr int NQ = Cfg::LPW / 4;
    auto line_src = [&](const GemmProb& p, const float* Ap, const float* Bp, long lda, long ldb,
                        int ks, int klen, int l, int e, bool& ok, bool isA) -> const float* {
      if (isA) {                                   // l < TC_BM (compile-time per quad)
        if (TA) { const int i = x.m0 + l, k = ks + e; ok = i < p.M && k < klen; return Ap + k + (long)i * lda; }
        const int k = ks + (l & 31), i = x.m0 + ((l >> 5) << 5) + e;
        ok = i < p.M && k < klen;
        return Ap + i + (long)k * lda;
      }
      const int lb = l - TC_BM;
      if (!TB) { const int j = x.n0 + lb, k = ks + e; ok = j < p.N && k < klen; return Bp + k + (long)j * ldb; }
      const int k = ks + (lb & 31), j = x.n0 + ((lb >> 5) << 5) + e;
      ok = j < p.N && k < klen;
      return Bp + j + (long)k * ldb;
    };
    int* st_b = nullptr;   // status pointer of the chunk just loaded
    auto load = [&](float (&v)[Cfg::LPW], int& vmode) {
      const GemmProb& p = b.p[x.pi];
      const int seg = c < x.nc1 ? 0 : 1;
      const int ks = (seg ? c - x.nc1 : c) * TC_BK;
      const int klen = seg ? p.K - p.k1 : p.k1;
      const float* Ap = seg ? p.A2 : p.A;
      const float* Bp = seg ? p.B2 : p.B;
      const long lda = seg ? p.lda2 : p.lda;
      const long ldb = seg ? p.ldb2 : p.ldb;
      vmode = p.vec;
      st_b = p.status;
#pragma unroll
      for (int qd = 0; qd < NQ; ++qd) {
        const int g = lw + qd * TC_LOAD_WARPS;
        const bool isA = qd < TC_BM / (4 * TC_LOAD_WARPS);   // compile-time: g = lw + qd * NLW, lw < NLW
        const bool vec = isA ? (p.vec & 1) : (p.vec & 2);
        if (vec) {
          const int l = 4 * g + (lane >> 3), e0 = (lane & 7) * 4;
          bool ok0, ok3;
          const float* src = line_src(p, Ap, Bp, lda, ldb, ks, klen, l, e0, ok0, isA);
          line_src(p, Ap, Bp, lda, ldb, ks, klen, l, e0 + 3, ok3, isA);
          if (ok0 && ok3) {
            const float4 w = __ldg(reinterpret_cast<const float4*>(src));
            v[4 * qd + 0] = w.x; v[4 * qd + 1] = w.y; v[4 * qd + 2] = w.z; v[4 * qd + 3] = w.w;
          } else {
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              bool ok;
              const float* s1 = line_src(p, Ap, Bp, lda, ldb, ks, klen, l, e0 + t, ok, isA);
              v[4 * qd + t] = ok ? __ldg(s1) : 0.f;
            }
          }
        } else {
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            bool ok;
            const float* s1 = line_src(p, Ap, Bp, lda, ldb, ks, klen, 4 * g + t, lane, ok, isA);
            v[4 * qd + t] = ok ? __ldg(s1) : 0.f;
          }
        }
      }
    };
    auto store = [&](const float (&v)[Cfg::LPW], int vmode, int*) {
      mbar_wait_sleep(empty_bar(stage), phase ^ 1);
      const uint32_t st = sbase + stage * Cfg::STAGE_BYTES;
#ifndef BKFAC_TC_DEBUG_NOSTORE
#pragma unroll
      for (int qd = 0; qd < NQ; ++qd) {
        const int g = lw + qd * TC_LOAD_WARPS;
        const bool isA = qd < TC_BM / (4 * TC_LOAD_WARPS);   // compile-time: g = lw + qd * NLW, lw < NLW
        const bool vec = isA ? (vmode & 1) : (vmode & 2);
        if (vec) {
          const int l = 4 * g + (lane >> 3), e0 = (lane & 7) * 4;
          uint32_t dh, dl;
          if (isA) { dh = st + tc_line_off<!TA, TC_BM>(l, e0); dl = dh + Cfg::A_BYTES; }
          else { dh = st + 2 * Cfg::A_BYTES + tc_line_off<TB, B_ROWS>(l - TC_BM, e0); dl = dh + Cfg::B_BYTES; }
          float h[4], lo[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) { h[t] = tf32_round(v[4 * qd + t]); lo[t] = v[4 * qd + t] - h[t]; }
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dh), "f"(h[0]), "f"(h[1]), "f"(h[2]), "f"(h[3]));
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dl), "f"(lo[0]), "f"(lo[1]), "f"(lo[2]), "f"(lo[3]));
        } else {
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int l = 4 * g + t;
            const float hi = tf32_round(v[4 * qd + t]);
            const float lo = v[4 * qd + t] - hi;
            uint32_t dh, dl;
            if (isA) { dh = st + tc_line_off<!TA, TC_BM>(l, lane); dl = dh + Cfg::A_BYTES; }
            else { dh = st + 2 * Cfg::A_BYTES + tc_line_off<TB, B_ROWS>(l - TC_BM, lane); dl = dh + Cfg::B_BYTES; }
            sts_f32(dh, hi);
            sts_f32(dl, lo);
          }
        }
      }
#endif
#ifndef BKFAC_TC_DEBUG_NOFENCE
      fence_proxy_async_smem();
#endif
      __syncwarp();
      if (lane == 0) {
        if (PAIR && crank != 0) mbar_arrive(pfull_bar(stage));   // forwarded to the leader
        else mbar_arrive(full_bar(stage));
      }
      if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
    };
    float va[Cfg::LPW], vb[Cfg::LPW];
    int ma = 0, mb = 0;
    int* sa_ = nullptr;
    int* sb_ = nullptr;
    bool have = seek();
    if (have) { load(va, ma); sa_ = st_b; ++c; }
    while (have) {
      const bool more = seek();
      if (more) { load(vb, mb); sb_ = st_b; ++c; }
      store(va, ma, sa_);
      if (!more) break;
      const bool more2 = seek();
      if (more2) { load(va, ma); sa_ = st_b; ++c; }
      store(vb, mb, sb_);
      have = more2;
    }
  } else {
    // ------------------------------------------------------------- epilogue
    const int e = warp < 4 ? warp : 4 + (warp - (TC_MMA_WARP + 1 + NLW));   // epilogue warp index
    float* stage = reinterpret_cast<float*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES + 256) +
                   e * Cfg::EPI_STAGE_FLOATS;
    tc_epilogue<BN, EPI, PAIR, NLW>(b, tmem_base, warp, lane, tfull_bar(0), tfull_bar(1), tempty_bar(0), tempty_bar(1),
                    stage);
  }
  tc_fence_before();
  if (PAIR) cluster_sync_all();   // neither CTA frees TMEM / exits while the pair still works
  else __syncthreads();
  if (warp == TC_MMA_WARP) {
    tc_fence_after();
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"((uint32_t)Cfg::TMEM_COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"((uint32_t)Cfg::TMEM_COLS));
  }
}

// Launch configuration of the hot-path GEMM (BN = 128 tiles, 16 loader warps, two
// chunks of loads in flight per loader).
#ifndef BKFAC_TC_BN_PAIR
#define BKFAC_TC_BN_PAIR 256
#endif
// CTA pairs compute 256 x TC_BN_PAIR tiles: with N = 256 every MMA (M = 256, N = 256, K = 8,
// 128 cycles) reads 4 KB of A and 4 KB of B from each CTA's shared memory (64 B/cycle), and
// the loaders store 64 KB (hi/lo of 128 A rows + 128 B rows) per 32-deep chunk of 12 MMAs
// (42 B/cycle): both fit the ~128 B/cycle of shared memory together.  With N = 128 the same
// chunk needed 96 + 64 B/cycle, which capped the pipe near 80 % of its rate.
constexpr int TC_BN = 128, TC_BN_PAIR = BKFAC_TC_BN_PAIR, TC_NLW = BKFAC_TC_NLW, TC_DEPTH = BKFAC_TC_DEPTH;
using TcMain = TcCfg<TC_BN, TC_NLW, TC_DEPTH, 4>;
// short-K stages (every K <= 8 chunks): the epilogue, not the MMA, sets the pace (C0 read
// + C write of whole output tiles): more epilogue warps, fewer loaders
#ifndef BKFAC_TC_SHORT_EPI
#define BKFAC_TC_SHORT_EPI 8
#endif
#ifndef BKFAC_TC_SHORT_NLW
#define BKFAC_TC_SHORT_NLW TC_NLW
#endif
constexpr int TC_SHORT_EPI = BKFAC_TC_SHORT_EPI, TC_SHORT_NLW = BKFAC_TC_SHORT_NLW;
using TcShortK = TcCfg<TC_BN, TC_SHORT_NLW, TC_DEPTH, TC_SHORT_EPI>;
// Pair kernels come with 4 epilogue warps (long K: the mainloop sets the pace, registers go
// to the loaders) and with 8 (K <= TC_PAIR_EPI8_CHUNKS chunks: a 256 x 256 tile's output --
// C0 read + C write, 512 KB per pair -- must drain within about one K-block of the next
// tile's MMAs; measured at configs[4]: prec_out 57.8 -> 46.3 ms, resid 10.8 -> 7.6 ms)
constexpr int TC_PAIR_EPI8_CHUNKS = 48;
using TcPair = TcCfg<TC_BN_PAIR, TC_NLW, TC_DEPTH, 4, true>;
using TcPair8 = TcCfg<TC_BN_PAIR, TC_NLW, TC_DEPTH, 8, true>;
constexpr int TC_SHORT_K_CHUNKS = 8;   // stages with every K <= 8 chunks use 8 epilogue warps

template <bool TA, bool TB, int EPI, bool PAIR>
inline bool tc_set_attr() {
  constexpr int BN = PAIR ? TC_BN_PAIR : TC_BN;
  using Cfg = TcCfg<BN, TC_NLW, TC_DEPTH, EPI, PAIR>;
  return cudaFuncSetAttribute(gemm_tc_kernel<TA, TB, BN, TC_NLW, TC_DEPTH, EPI, PAIR>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES) == cudaSuccess;
}

inline bool tc_init_attributes() {
  bool ok = true;
  ok &= tc_set_attr<false, false, 4, false>();
  ok &= tc_set_attr<false, true, 4, false>();
  ok &= tc_set_attr<true, false, 4, false>();
  ok &= tc_set_attr<true, true, 4, false>();
  ok &= cudaFuncSetAttribute(gemm_tc_kernel<false, false, TC_BN, TC_SHORT_NLW, TC_DEPTH, TC_SHORT_EPI, false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, TcShortK::SMEM_BYTES) == cudaSuccess;
  ok &= cudaFuncSetAttribute(gemm_tc_kernel<false, true, TC_BN, TC_SHORT_NLW, TC_DEPTH, TC_SHORT_EPI, false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, TcShortK::SMEM_BYTES) == cudaSuccess;
  ok &= cudaFuncSetAttribute(gemm_tc_kernel<true, false, TC_BN, TC_SHORT_NLW, TC_DEPTH, TC_SHORT_EPI, false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, TcShortK::SMEM_BYTES) == cudaSuccess;
  ok &= cudaFuncSetAttribute(gemm_tc_kernel<true, true, TC_BN, TC_SHORT_NLW, TC_DEPTH, TC_SHORT_EPI, false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, TcShortK::SMEM_BYTES) == cudaSuccess;
  ok &= tc_set_attr<false, false, 4, true>();
  ok &= tc_set_attr<false, true, 4, true>();
  ok &= tc_set_attr<true, false, 4, true>();
  ok &= tc_set_attr<true, true, 4, true>();
  ok &= tc_set_attr<false, false, 8, true>();
  ok &= tc_set_attr<false, true, 8, true>();
  ok &= tc_set_attr<true, false, 8, true>();
  ok &= tc_set_attr<true, true, 8, true>();
  return ok;
}

// grid: persistent CTAs (pair mode: CTA pairs, 2 x grid CTAs in clusters of 2)
template <bool TA, bool TB>
inline cudaError_t tc_launch(const GemmBatch& b, int grid, cudaStream_t st, int max_chunks, bool pair) {
  const bool short_k = max_chunks <= TC_SHORT_K_CHUNKS;
  if (pair) {
    const bool e8 = max_chunks <= TC_PAIR_EPI8_CHUNKS;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * grid), 1, 1);
    cfg.blockDim = dim3(e8 ? TcPair8::THREADS : TcPair::THREADS, 1, 1);
    cfg.dynamicSmemBytes = e8 ? TcPair8::SMEM_BYTES : TcPair::SMEM_BYTES;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (e8) return cudaLaunchKernelEx(&cfg, gemm_tc_kernel<TA, TB, TC_BN_PAIR, TC_NLW, TC_DEPTH, 8, true>, b);
    return cudaLaunchKernelEx(&cfg, gemm_tc_kernel<TA, TB, TC_BN_PAIR, TC_NLW, TC_DEPTH, 4, true>, b);
  }
  if (short_k)
    gemm_tc_kernel<TA, TB, TC_BN, TC_SHORT_NLW, TC_DEPTH, TC_SHORT_EPI, false><<<grid, TcShortK::THREADS, TcShortK::SMEM_BYTES, st>>>(b);
  else
    gemm_tc_kernel<TA, TB, TC_BN, TC_NLW, TC_DEPTH, 4, false><<<grid, TcMain::THREADS, TcMain::SMEM_BYTES, st>>>(b);
  return cudaGetLastError();
}

}  // namespace bkfac
