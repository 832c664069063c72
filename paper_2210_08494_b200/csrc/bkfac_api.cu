// C ABI of the B-KFAC hot path (include/bkfac.h): workspace planning, validation and
// the stream-ordered stage sequence of each call.  All arithmetic runs in the kernels
// of gemm_*.cuh, chol.cuh, eig.cuh and misc.cuh.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <map>
#include <string>
#include <functional>
#include <vector>

#include "bkfac.h"
#include "chol.cuh"
#include "chol_tiled.cuh"
#include "common.cuh"
#include "eig.cuh"
#include "gemm_simt.cuh"
#include "gemm_tc.cuh"
#include "misc.cuh"
#include "sbr.cuh"
#include "sytrd_tiled.cuh"

using namespace bkfac;

namespace {

constexpr int kSplitMax = 16;
constexpr int kNumSM = 148;
constexpr int kRsvdOversampleMax = 32;

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// caller leading dimensions (bkfac.h "Leading dimensions"): 0 = packed
inline int ldx(int ld, int rows) { return ld > 0 ? ld : rows; }
inline bool ld_ok(int ld, int rows) { return ld == 0 || ld >= rows; }
// the GEMM loaders' 16-byte path: aligned base, leading dimension a multiple of 4
inline bool al16(const void* q, int ld) {
  return (reinterpret_cast<uintptr_t>(q) & 15) == 0 && (ld & 3) == 0;
}
inline int pad32(int x) { return (x + 31) / 32 * 32; }

struct Arena {
  size_t cur = 0;
  size_t take(size_t bytes) {
    size_t o = cur;
    cur += align256(bytes ? bytes : 1);
    return o;
  }
};

struct EigWs {  // workspace of one eigen problem of order <= m with <= r outputs
  size_t K, d, e, tau, lam, Y, scr, piv, V, gt, U, Z, S;
  size_t Vp = 0, Vt = 0, Wt = 0, Zp = 0, Xp = 0, Wp = 0, Tp = 0, AB = 0, Vq = 0, tq = 0;   // two-stage (sbr.cuh)
  bool sbr = false;   // two-stage workspace planned (sbr_supported(m))
  int m, r;
};

void plan_eig(Arena& a, EigWs& w, int m, int r) {
  w.m = m; w.r = r;
  w.K = a.take(sizeof(float) * (size_t)m * m);
  w.gt = sytrd_tiled_cluster(m) == 0 ? a.take(sizeof(float) * syt_global_tile_floats(m)) : 0;
  w.sbr = sbr_supported(m);
  if (w.sbr) {
    const size_t mb = sizeof(float) * (size_t)m * SBR_B;
    w.Vp = a.take(mb); w.Vt = a.take(mb); w.Wt = a.take(mb); w.Xp = a.take(mb); w.Wp = a.take(mb);
    w.Zp = a.take(sizeof(float) * (size_t)ceil_div(m, SBR_X_ROWS) * SBR_B * SBR_B);
    w.Tp = a.take(sizeof(float) * SBR_B * SBR_B);
    w.AB = a.take(sizeof(float) * (size_t)m * SBR_LDB);
    w.Vq = a.take(sizeof(float) * (size_t)m * sbr_tasks(m) * SBR_B);
    w.tq = a.take(sizeof(float) * (size_t)m * sbr_tasks(m));
  }
  w.d = a.take(sizeof(float) * m);
  w.e = a.take(sizeof(float) * m);
  w.tau = a.take(sizeof(float) * m);
  w.lam = a.take(sizeof(double) * r);
  w.Y = a.take(sizeof(double) * (size_t)m * r);
  w.scr = a.take(sizeof(double) * 4 * (size_t)m * r);
  w.piv = a.take((size_t)m * r);
  w.V = a.take(sizeof(float) * (size_t)m * r);
  w.U = a.take(sizeof(float) * (size_t)m * std::max(bt_panels(m), 1) * BT_PW);
  w.Z = a.take(sizeof(float) * (size_t)BT_PW * r);
  w.S = a.take(sizeof(float) * (size_t)std::max(bt_panels(m), 1) * 2 * BT_PW * BT_PW);
}

struct FactorPlan {
  bkfac_factor_desc d;
  bool dense = false;  // r + c_max >= n: form the n x n sum densely (a6')
  int m = 0;           // core order (r + c_max, or n on the dense path)
  int rout = 0;        // output columns: r, or min(n, r + c_max) with BKFAC_FACTOR_FULL_RANK
  int nld = 0;         // leading dimension of the internal n-row buffers (R, Qb, Urot): n
                       // rounded up to 32, so their GEMM loads take the 16-byte vector path
  // Brand path
  size_t W, P2, R, Qb, G, L1, L1i, L2, L2i, cscr, ws, Vf = 0;
  size_t Ms = 0, Us = 0;   // aligned copies (ld nld) of the caller's M and U_in (odd n only)
  size_t ws_elems = 0;
  // dense path
  size_t T;
  // orthonormality refresh of the output basis (both paths): U' before, U'^T U', split-K
  size_t Urot, Gref, wsr;
  size_t wsr_elems = 0;
  EigWs eig;
  // RSVD
  bool rsvd = false;
  int lmax = 0;
  size_t Yr, Qr, Q2r, Tr, Gr, L1r, L1ir, L2r, L2ir, Br, cscr_r, ws_r;
  size_t ws_r_elems = 0;
  EigWs eig_r;
};

struct LayerPlan {
  bkfac_layer_desc d;
  size_t Y, Xt, Z, sA, sG, lam, ws;  // lam: [lamA, lamG, coef, 1/lamA, 1/lamG]
  int ldY = 0, ldXt = 0;             // Y (d_G x r_A), Xt (d_A x r_G): padded to 32
  size_t ws_elems = 0;
  // Algorithm 8 (n_max > 0): P_G = G^T U_G, P_A = A^T U_A (n x r), G_b, A_b (d x n)
  size_t fPG = 0, fPA = 0, fGb = 0, fAb = 0, fws = 0, fws2 = 0;
  size_t fws_elems = 0;
};

}  // namespace

struct bkfac_ctx_s {
  int device = 0;
  std::vector<FactorPlan> f;
  std::vector<LayerPlan> l;
  size_t ws_bytes = 0;
  size_t status_off = 0;
  char* ws = nullptr;
  size_t ws_cap = 0;
  uint64_t launches = 0;
  int* host_status = nullptr;
  bool use_tc = true;
  // side streams for independent launch groups inside one call (fork/join with events)
  cudaStream_t side[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t ev_fork = nullptr, ev_join[4] = {nullptr, nullptr, nullptr, nullptr};
  // bkfac_brand_ea_update: the EA accumulate, launched on ea_stream by the eigensolver
  // (pending_ea(busy SMs)) so that it runs on the SMs the tridiagonalisation leaves idle
  cudaStream_t ea_stream = nullptr;
  cudaEvent_t ev_ea_fork = nullptr, ev_ea_done = nullptr;
  std::function<bkfac_status(int)> pending_ea;
  int nvtx = 0;       // BKFAC_OPT_NVTX: every stage inside an NVTX range named by its tag
  int sbr_x = 1;      // BKFAC_OPT_SBR_X: band reduction's X and update kernels (mma.sync, lower triangle)
  int grid_cap = 0;   // > 0: persistent GEMM grids capped at this many CTAs; < 0: one CTA per tile
  int prec_block = 0;  // BKFAC_OPT_PREC_BLOCK: K chunks per TMEM accumulation block of gemm_prec_out (0: TC_PROMO)
  int user_cap = 0;   // BKFAC_OPT_GEMM_CAP: > 0 caps every persistent GEMM grid of this context's
                      // calls (two calls sharing the GPU on two streams, each on its own SMs)
  bool ea_join_early = false;   // join the side-stream EA right after the tridiagonalisation
  int pair_mode = 1;  // CTA-pair GEMM tiles: 0 never, 1 large long-K stages, 2 always (tests)
  // run-time options (bkfac_set_option; defaults are the tuned configuration)
  int two_stage = 0;    // eigensolver reduction: 0 auto (two-stage when the one-stage tiles do
                        // not fit a cluster's shared memory), 1 one-stage only, 2 two-stage
                        // wherever supported
  int gt_cluster = 8;   // largest cluster of the global-tile tridiagonalisation / Cholesky
  int syt_cluster = 0;  // > 0: wider clusters for the shared-memory tridiagonalisation (tuning)
  int bt_simt = 0;      // back-transform Gram / T products on the fp32 SIMT GEMM
  int ea_mode = 0;      // EA accumulate: 0 beside the eigensolver (capped grid), 1 serial
                        // first, 2 beside uncapped, 3/4 one CTA per tile (4: early join)
  int ea_cap = 0;       // > 0: EA grid cap (CTAs) instead of the idle-SM count
  int chol_blocked = 1; // Cholesky of orders > 256 blocked on the tcgen05 GEMM (0: one tiled
                        // CTA / cluster per factor, chol_tiled_kernel)
  // optional per-stage CUDA-event profiling (bkfac_profile_enable)
  bool prof = false;
  struct Rec { std::string tag; cudaEvent_t a, b; double flops, bytes; uint64_t launches; };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  size_t pool_used = 0;
  int open_rec = -1;
};

namespace {

template <typename T>
T* at(bkfac_ctx c, size_t off) { return reinterpret_cast<T*>(c->ws + off); }

int* status_ptr(bkfac_ctx c, int factor) { return at<int>(c, c->status_off) + factor; }

bool cuda_ok(cudaError_t e) {
  if (e != cudaSuccess) {
    fprintf(stderr, "bkfac: CUDA error %s\n", cudaGetErrorString(e));
    return false;
  }
  return true;
}

cudaEvent_t prof_event(bkfac_ctx c) {
  if (c->pool_used == c->pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->pool.push_back(e);
  }
  return c->pool[c->pool_used++];
}

// Records a profiling event on `st`.  Under stream capture a plain cudaEventRecord only
// becomes a dependency edge; cudaEventRecordExternal makes it an event-record node, which
// every replay of the graph re-records (so per-stage times can be read after a replay).
void prof_record(cudaEvent_t e, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
  else
    cudaEventRecord(e, st);
}

// Brackets one stage (one or more kernel launches on `st`) with CUDA events.
void prof_begin(bkfac_ctx c, const char* tag, cudaStream_t st, double flops, double bytes) {
  if (c->nvtx) nvtxRangePushA(tag);   // host ranges: ncu --nvtx --nvtx-include "<stage>/"
  if (!c->prof) return;
  bkfac_ctx_s::Rec r;
  r.tag = tag; r.flops = flops; r.bytes = bytes; r.launches = c->launches;
  r.a = prof_event(c); r.b = prof_event(c);
  prof_record(r.a, st);
  c->recs.push_back(r);
  c->open_rec = (int)c->recs.size() - 1;
}
void prof_end(bkfac_ctx c, cudaStream_t st) {
  if (c->nvtx) nvtxRangePop();
  if (!c->prof || c->open_rec < 0) return;
  auto& r = c->recs[c->open_rec];
  prof_record(r.b, st);
  r.launches = c->launches - r.launches;
  c->open_rec = -1;
}

// largest cluster for the global-tile tridiagonalisation and Cholesky (few factors per GPU);
// option BKFAC_OPT_GT_CLUSTER = 1 forces one CTA per factor (tests cover the cluster sizes)
int gt_cluster_max(bkfac_ctx c) { return std::max(1, std::min(8, c->gt_cluster)); }

// two-stage reduction (sbr.cuh) for an eigenproblem of order m?
bool use_sbr(bkfac_ctx c, const EigWs& w, int m) {
  if (!w.sbr || !sbr_supported(m) || c->two_stage == 1) return false;
  return c->two_stage == 2 || sytrd_tiled_cluster(m) == 0;
}

#define LAUNCH_CHECK(ctx)                                   \
  do {                                                      \
    (ctx)->launches++;                                      \
    if (!cuda_ok(cudaGetLastError())) return BKFAC_ERR_CUDA; \
  } while (0)

// ------------------------------------------------------------------ GEMM stage
struct GemmStage {
  bool fp32_simt = false;   // this stage on the fp32 CUDA-core kernel (accuracy-critical, small)
  std::vector<GemmProb> probs[4];
  std::vector<long> caps[4];
  void add(bool ta, bool tb, const GemmProb& p, long ws_cap_elems) {
    const int v = (ta ? 2 : 0) + (tb ? 1 : 0);
    probs[v].push_back(p);
    caps[v].push_back(ws_cap_elems);
  }
  bool empty() const {
    return probs[0].empty() && probs[1].empty() && probs[2].empty() && probs[3].empty();
  }
};

GemmProb gp(const float* A, int lda, const float* B, int ldb, float* C, int ldc, int M, int N,
            int K, float alpha, const float* C0 = nullptr, int ldc0 = 0, float beta = 0.f) {
  GemmProb p;
  memset(&p, 0, sizeof(p));
  p.A = A; p.lda = lda; p.A2 = A; p.lda2 = lda;
  p.B = B; p.ldb = ldb; p.B2 = B; p.ldb2 = ldb;
  p.C = C; p.ldc = ldc; p.C0 = C0 ? C0 : C; p.ldc0 = C0 ? ldc0 : ldc;
  p.M = M; p.N = N; p.K = K; p.k1 = K;
  p.alpha = alpha; p.beta = beta;
  return p;
}

template <bool TA, bool TB>
bkfac_status launch_variant(bkfac_ctx ctx, std::vector<GemmProb>& v, cudaStream_t st, bool tc,
                            bool pair) {
  size_t i0 = 0;
  while (i0 < v.size()) {
    const size_t n = std::min(v.size() - i0, (size_t)GEMM_MAXP);
    static thread_local GemmBatch b;  // host staging (large); kernel params are copied at launch
    b.nprob = (int)n;
    int tiles = 0;
    bool any_split = false;
    int max_chunks = 0;   // K chunks of the longest work item (short K: epilogue-bound)
    for (size_t i = 0; i < n; ++i) {
      GemmProb p = v[i0 + i];
      max_chunks = std::max(max_chunks, p.splits > 1 ? p.kchunk
                                                     : ceil_div(std::max(p.k1, 0), TC_BK) +
                                                           ceil_div(std::max(p.K - p.k1, 0), TC_BK));
      p.tile_start = tiles;
      tiles += (p.sym ? p.tiles_m * (p.tiles_m + 1) / 2 : p.tiles_m * p.tiles_n) * p.splits;
      any_split |= p.splits > 1;
      b.p[i] = p;
    }
    b.total_tiles = tiles;
    if (tiles > 0) {
      if (tc) {
        const int nsm = ctx->grid_cap > 0 ? ctx->grid_cap
                      : ctx->user_cap > 0 ? std::max(2, ctx->user_cap) : kNumSM;
        // grid_cap < 0: one CTA per tile (a background job whose CTAs retire quickly)
        const int grid = ctx->grid_cap < 0 ? tiles : std::min(tiles, pair ? nsm / 2 : nsm);
        if (!cuda_ok(tc_launch<TA, TB>(b, grid, st, max_chunks, pair)))
          return BKFAC_ERR_CUDA;
      } else {
        gemm_simt_kernel<TA, TB><<<tiles, 256, 0, st>>>(b);
      }
      LAUNCH_CHECK(ctx);
      if (any_split) {
        long items = 0;   // largest reduce of the batch, in 4-row groups (about 2 per thread)
        for (size_t i = 0; i < n; ++i)
          if (b.p[i].splits > 1) items = std::max(items, (long)b.p[i].M * b.p[i].N / 4);
        const unsigned gx = (unsigned)std::max(64L, std::min(2048L, (items + 511) / 512));
        gemm_splitk_reduce_kernel<<<dim3(gx, (unsigned)n), 256, 0, st>>>(b);
        LAUNCH_CHECK(ctx);
      }
    }
    i0 += n;
  }
  return BKFAC_OK;
}

bkfac_status run_gemms_impl(bkfac_ctx ctx, GemmStage& s, cudaStream_t st);
bkfac_status run_gemms(bkfac_ctx ctx, GemmStage& s, cudaStream_t st, const char* tag) {
  double flops = 0.0, bytes = 0.0;
  for (int v = 0; v < 4; ++v)
    for (auto& p : s.probs[v]) {
      // a symmetric product's algorithmic work is its lower triangle
      flops += (p.sym && p.M == p.N ? (double)p.M * (p.N + 1) : 2.0 * p.M * (double)p.N) * p.K;
      bytes += 4.0 * ((double)p.M * p.K + (double)p.K * p.N + (double)p.M * p.N *
                      ((p.beta != 0.f || p.beta_dev) ? 2.0 : 1.0));
    }
  prof_begin(ctx, tag, st, flops, bytes);
  bkfac_status rr = run_gemms_impl(ctx, s, st);
  prof_end(ctx, st);
  return rr;
}

// Tile-shape and split-K planning.  SIMT: K units, 64 x 64 tiles, splits while the stage
// has fewer tiles than twice the SM count.  tcgen05 (the hot path): every decision depends on
// the problem alone, never on the rest of the batch, so a factor's arithmetic (and its bits)
// is the same whichever rank computes it and whatever else shares the launch:
//   * CTA-pair 256 x 256 tiles for non-symmetric problems with long K (> 8 chunks) and
//     M >= 512, N >= 256; 128 x 128 tiles otherwise (a stage launches each group separately);
//   * split-K (deterministic fixed-order reduction) into work items of at most
//     TC_SPLIT_CHUNKS chunks of 32, for problems with fewer tiles than SMs, when the caller
//     supplied a workspace.
constexpr int TC_SPLIT_CHUNKS = 128;
bool tc_pair_tiles(const bkfac_ctx ctx, const GemmProb& p) {
  if (p.sym == 2 || ctx->pair_mode == 0) return false;
  const int nc = ceil_div(std::max(p.k1, 0), TC_BK) + ceil_div(std::max(p.K - p.k1, 0), TC_BK);
  // a symmetric problem takes pair tiles only where it will be split (the split-K reduce
  // writes its mirrored upper tiles; the pair epilogue has no mirrored store)
  if (p.sym) {
    const long t2 = (long)ceil_div(p.M, 2 * TC_BM) * ceil_div(p.N, TC_BN_PAIR);
    if (p.M != p.N || TC_BN_PAIR != 2 * TC_BM || p.ws == nullptr || nc <= TC_SPLIT_CHUNKS ||
        t2 >= kNumSM)
      return false;
  }
  if (ctx->pair_mode == 2) return true;
  return nc > TC_SHORT_K_CHUNKS && p.M >= 512 && p.N >= 256;
}

bkfac_status run_gemms_impl(bkfac_ctx ctx, GemmStage& s, cudaStream_t st) {
  const bool tc = ctx->use_tc && !s.fp32_simt;
  if (tc) {
    GemmStage ps;   // the pair-tile problems of the stage
    for (int v = 0; v < 4; ++v) {
      std::vector<GemmProb> keep;
      std::vector<long> keepc;
      for (size_t i = 0; i < s.probs[v].size(); ++i) {
        GemmProb p = s.probs[v][i];
        const bool pair = tc_pair_tiles(ctx, p);
        const int bm = pair ? 2 * TC_BM : TC_BM, bn = pair ? TC_BN_PAIR : TC_BN;
        p.tiles_m = ceil_div(std::max(p.M, 1), bm);
        p.tiles_n = ceil_div(std::max(p.N, 1), bn);
        if (p.M <= 0 || p.N <= 0) p.tiles_m = p.tiles_n = 0;
        if (p.M != p.N || bm != bn) p.sym = 0;   // lower tiles of square tiles only
        p.tbm = bm;
        // walk the tiles along the smaller operand: A (M x K) re-read per column block when
        // M is walked first, B (K x N) per row block otherwise
        p.nfast = (!p.sym && p.M > p.N) ? 1 : 0;
        auto al = [](const float* q, int ld) {
          return q == nullptr || ((reinterpret_cast<uintptr_t>(q) & 15) == 0 && (ld & 3) == 0);
        };
        p.vec = ((al(p.A, p.lda) && al(p.A2, p.lda2)) ? 1 : 0) | ((al(p.B, p.ldb) && al(p.B2, p.ldb2)) ? 2 : 0);
        const long mn = (long)p.M * p.N;
        const long cap = (p.ws != nullptr && mn > 0) ? s.caps[v][i] / mn : 1;
        const int nc = ceil_div(std::max(p.k1, 0), TC_BK) + ceil_div(std::max(p.K - p.k1, 0), TC_BK);
        int splits = 1;
        const long own_tiles = (long)p.tiles_m * p.tiles_n;   // the problem alone fills the GPU?
        if (nc > TC_SPLIT_CHUNKS && own_tiles < kNumSM && p.ws != nullptr) {
          splits = std::min(kSplitMax, ceil_div(nc, TC_SPLIT_CHUNKS));
          splits = (int)std::min<long>(splits, cap);
          splits = std::max(splits, 1);
        }
        const int cps = std::max(ceil_div(nc, splits), 1);
        p.splits = std::max(ceil_div(nc, cps), 1);
        p.kchunk = cps;
        // symmetric problems: the split-K reduce mirrors (or skips) the upper tiles; without
        // split-K only the 128 x 128 epilogue has the mirrored store
        if (pair && p.splits == 1) p.sym = 0;
        if (pair) { ps.probs[v].push_back(p); ps.caps[v].push_back(s.caps[v][i]); }
        else { keep.push_back(p); keepc.push_back(s.caps[v][i]); }
      }
      s.probs[v].swap(keep);
      s.caps[v].swap(keepc);
    }
    bkfac_status r;
    for (int pass = 0; pass < 2; ++pass) {
      GemmStage& g = pass == 0 ? ps : s;
      const bool pair = pass == 0;
      if ((r = launch_variant<false, false>(ctx, g.probs[0], st, true, pair)) != BKFAC_OK) return r;
      if ((r = launch_variant<false, true>(ctx, g.probs[1], st, true, pair)) != BKFAC_OK) return r;
      if ((r = launch_variant<true, false>(ctx, g.probs[2], st, true, pair)) != BKFAC_OK) return r;
      if ((r = launch_variant<true, true>(ctx, g.probs[3], st, true, pair)) != BKFAC_OK) return r;
    }
    for (int v = 0; v < 4; ++v) { s.probs[v].clear(); s.caps[v].clear(); }
    s.fp32_simt = false;
    return BKFAC_OK;
  }
  const int bm = SG_BM, bn = SG_BN;
  long base_tiles = 0;
  for (int v = 0; v < 4; ++v)
    for (auto& p : s.probs[v]) {
      p.tiles_m = ceil_div(std::max(p.M, 1), bm);
      p.tiles_n = ceil_div(std::max(p.N, 1), bn);
      if (p.M <= 0 || p.N <= 0) p.tiles_m = p.tiles_n = 0;
      p.sym = 0;
      base_tiles += (long)p.tiles_m * p.tiles_n;
    }
  const long target = 2L * kNumSM;
  for (int v = 0; v < 4; ++v)
    for (size_t i = 0; i < s.probs[v].size(); ++i) {
      GemmProb& p = s.probs[v][i];
      const long mn = (long)p.M * p.N;
      const long cap = (p.ws != nullptr && mn > 0) ? s.caps[v][i] / mn : 1;
      int splits = 1;
      if (p.K >= 1024 && base_tiles > 0 && base_tiles < target && p.ws != nullptr) {
        splits = (int)std::min<long>(kSplitMax, (target + base_tiles - 1) / base_tiles);
        splits = std::min(splits, p.K / 256);
        splits = (int)std::min<long>(splits, cap);
        splits = std::max(splits, 1);
      }
      int kchunk = p.K;
      if (splits > 1) {
        kchunk = ceil_div(p.K, splits);
        kchunk = (kchunk + SG_BK - 1) / SG_BK * SG_BK;
        splits = ceil_div(p.K, kchunk);
      }
      p.splits = splits;
      p.kchunk = std::max(kchunk, 1);
    }
  bkfac_status r;
  if ((r = launch_variant<false, false>(ctx, s.probs[0], st, false, false)) != BKFAC_OK) return r;
  if ((r = launch_variant<false, true>(ctx, s.probs[1], st, false, false)) != BKFAC_OK) return r;
  if ((r = launch_variant<true, false>(ctx, s.probs[2], st, false, false)) != BKFAC_OK) return r;
  if ((r = launch_variant<true, true>(ctx, s.probs[3], st, false, false)) != BKFAC_OK) return r;
  for (int v = 0; v < 4; ++v) { s.probs[v].clear(); s.caps[v].clear(); }
  s.fp32_simt = false;
  return BKFAC_OK;
}

// ------------------------------------------------------------------ small stages
bkfac_status run_ew(bkfac_ctx ctx, std::vector<EwProb>& v, cudaStream_t st, const char* tag) {
  double bytes = 0.0;
  for (auto& p : v) bytes += (p.op == EW_ADD_DIAG) ? 8.0 * p.rows : 12.0 * p.rows * (double)p.cols;
  prof_begin(ctx, tag, st, 0.0, bytes);
  size_t i0 = 0;
  while (i0 < v.size()) {
    const size_t n = std::min(v.size() - i0, (size_t)EW_MAXP);
    static thread_local EwBatch b;
    b.nprob = (int)n;
    for (size_t i = 0; i < n; ++i) b.p[i] = v[i0 + i];
    ew_kernel<<<dim3(128, (unsigned)n), 256, 0, st>>>(b);
    LAUNCH_CHECK(ctx);
    i0 += n;
  }
  v.clear();
  prof_end(ctx, st);
  return BKFAC_OK;
}

bkfac_status run_gemms(bkfac_ctx ctx, GemmStage& s, cudaStream_t st, const char* tag);
bkfac_status run_ew(bkfac_ctx ctx, std::vector<EwProb>& v, cudaStream_t st, const char* tag);

// Blocked Cholesky + triangular inverse for orders c > 256 (chol_tiled.cuh,
// chol_blocked_prep_kernel): 256 x 256 diagonal blocks on chol_smem_kernel (L_kk and
// L_kk^{-1}), the panel L21 = A21 L11^{-T} and the trailing SYRK A22 -= L21 L21^T on the
// tcgen05 GEMM; then X = L^{-1} by block rows, X(i, 0:i) = -X_ii (L(i, 0:i) X(0:i, 0:i)),
// two GEMMs per block row.  Scratch per problem: the tolerance reference (first float) and a
// c x 256 panel (from float 64 on).
bkfac_status run_chol_blocked(bkfac_ctx ctx, std::vector<CholProb>& v, cudaStream_t st) {
  constexpr int BS = 32 * CS_MAXNB;
  const int n = (int)v.size();
  static thread_local CholTiledBatch pb;   // host staging (the kernels copy their parameters)
  bkfac_status rs;
  for (int i0 = 0; i0 < n; i0 += CT_MAXP) {
    pb.nprob = std::min(n - i0, CT_MAXP);
    for (int i = 0; i < pb.nprob; ++i) {
      const CholProb& q = v[i0 + i];
      pb.p[i] = CholTiledProb{q.G, q.ldg, q.L, q.Linv, q.scratch, q.status, q.c, q.shift, 0, q.scratch};
    }
    prof_begin(ctx, "chol_diag", st, 0.0, 0.0);
    chol_blocked_prep_kernel<<<dim3((unsigned)pb.nprob, 32), 256, 0, st>>>(pb);
    LAUNCH_CHECK(ctx);
    prof_end(ctx, st);
  }
  int nbmax = 0;
  for (auto& q : v) nbmax = std::max(nbmax, ceil_div(q.c, BS));
  GemmStage gs;
  std::vector<EwProb> ew;
  for (int kb = 0; kb < nbmax; ++kb) {
    int nd = 0;
    for (int i = 0; i < n; ++i) {
      const CholProb& q = v[i];
      const int o = kb * BS;
      if (o >= q.c) continue;
      const int w = std::min(BS, q.c - o);
      float* Lk = q.L + o + (long)o * q.c;
      pb.p[nd++] = CholTiledProb{Lk, q.c, Lk, q.Linv + o + (long)o * q.c, nullptr, q.status, w, 0.f, q.c, q.scratch};
      if (nd == CT_MAXP) {
        pb.nprob = nd;
        prof_begin(ctx, "chol_diag", st, 2.0 / 3.0 * BS * BS * (double)BS * nd, 0.0);
        chol_smem_kernel<<<(unsigned)nd, CT_THREADS, chol_smem_bytes(BS), st>>>(pb);
        LAUNCH_CHECK(ctx);
        prof_end(ctx, st);
        nd = 0;
      }
    }
    if (nd) {
      pb.nprob = nd;
      prof_begin(ctx, "chol_diag", st, 2.0 / 3.0 * BS * BS * (double)BS * nd, 0.0);
      chol_smem_kernel<<<(unsigned)nd, CT_THREADS, chol_smem_bytes(BS), st>>>(pb);
      LAUNCH_CHECK(ctx);
      prof_end(ctx, st);
    }
    bool more = false;
    for (auto& q : v) {
      const int o = kb * BS, w = std::min(BS, q.c - o), o2 = o + w, rem = q.c - o2;
      if (o >= q.c || rem <= 0) continue;
      more = true;
      float* T21 = q.scratch + 64;
      // T21 = A21 L11^{-T}
      gs.add(false, true, gp(q.L + o2 + (long)o * q.c, q.c, q.Linv + o + (long)o * q.c, q.c, T21, q.c,
                             rem, w, w, 1.f), 0);
    }
    if (!more) continue;
    if ((rs = run_gemms(ctx, gs, st, "chol_panel")) != BKFAC_OK) return rs;
    for (auto& q : v) {
      const int o = kb * BS, w = std::min(BS, q.c - o), o2 = o + w, rem = q.c - o2;
      if (o >= q.c || rem <= 0) continue;
      float* T21 = q.scratch + 64;
      EwProb e{};
      e.Y = q.L + o2 + (long)o * q.c; e.ldy = q.c; e.X = T21; e.ldx = q.c; e.rows = rem; e.cols = w;
      e.op = EW_COPY;
      ew.push_back(e);
      float* A22 = q.L + o2 + (long)o2 * q.c;
      GemmProb pu = gp(T21, q.c, T21, q.c, A22, q.c, rem, rem, w, -1.f, A22, q.c, 1.f);
      pu.sym = 2;   // lower tiles only: the upper triangle of L stays zero
      gs.add(false, true, pu, 0);
    }
    if ((rs = run_ew(ctx, ew, st, "chol_copy")) != BKFAC_OK) return rs;
    if ((rs = run_gemms(ctx, gs, st, "chol_syrk")) != BKFAC_OK) return rs;
  }
  if (!ctx->use_tc) {   // the SIMT GEMM computes whole squares: clear what the SYRK left above
    for (auto& q : v) {
      EwProb e{};
      e.Y = q.L; e.ldy = q.c; e.rows = q.c; e.cols = q.c; e.op = EW_ZERO_UPPER;
      ew.push_back(e);
    }
    if ((rs = run_ew(ctx, ew, st, "chol_copy")) != BKFAC_OK) return rs;
  }
  // X = L^{-1}: block row i (offset oi, width wi): T = L(i, 0:i) X(0:i, 0:i); X(i, 0:i) = -X_ii T
  for (int i = 1; i < nbmax; ++i) {
    bool any = false;
    for (auto& q : v) {
      const int oi = i * BS;
      if (oi >= q.c) continue;
      any = true;
      const int wi = std::min(BS, q.c - oi);
      gs.add(false, false, gp(q.L + oi, q.c, q.Linv, q.c, q.scratch + 64, wi, wi, oi, oi, 1.f), 0);
    }
    if (!any) break;
    if ((rs = run_gemms(ctx, gs, st, "chol_inv_t")) != BKFAC_OK) return rs;
    for (auto& q : v) {
      const int oi = i * BS;
      if (oi >= q.c) continue;
      const int wi = std::min(BS, q.c - oi);
      gs.add(false, false, gp(q.Linv + oi + (long)oi * q.c, q.c, q.scratch + 64, wi, q.Linv + oi, q.c,
                              wi, oi, wi, -1.f), 0);
    }
    if ((rs = run_gemms(ctx, gs, st, "chol_inv_x")) != BKFAC_OK) return rs;
  }
  return BKFAC_OK;
}

bkfac_status run_chol(bkfac_ctx ctx, std::vector<CholProb>& v, cudaStream_t st) {
  double flops = 0.0, bytes = 0.0;
  for (auto& p : v) { flops += 2.0 * p.c * (double)p.c * p.c / 3.0; bytes += 12.0 * p.c * (double)p.c; }
  // orders above the shared-memory kernel's 256: blocked on the tensor-core GEMM
  if (ctx->chol_blocked) {
    std::vector<CholProb> big, small;
    for (auto& p : v) (p.c > 32 * CS_MAXNB ? big : small).push_back(p);
    if (!big.empty()) {
      const bkfac_status rb = run_chol_blocked(ctx, big, st);
      if (rb != BKFAC_OK) return rb;
      v.swap(small);
      if (v.empty()) return BKFAC_OK;
      flops = bytes = 0.0;
      for (auto& p : v) { flops += 2.0 * p.c * (double)p.c * p.c / 3.0; bytes += 12.0 * p.c * (double)p.c; }
    }
  }
  prof_begin(ctx, "chol_inv", st, flops, bytes);
  static thread_local CholTiledBatch b;
  size_t i0 = 0;
  while (i0 < v.size()) {
    const size_t n = std::min(v.size() - i0, (size_t)CT_MAXP);
    b.nprob = (int)n;
    for (size_t i = 0; i < n; ++i) {
      const CholProb& q = v[i0 + i];
      b.p[i] = CholTiledProb{q.G, q.ldg, q.L, q.Linv, q.scratch, q.status, q.c, q.shift, 0, nullptr};
    }
    int cmax = 0;
    for (size_t i = 0; i < n; ++i) cmax = std::max(cmax, b.p[i].c);
    if (cmax <= 32 * CS_MAXNB)   // every tile resident in shared memory
      chol_smem_kernel<<<(unsigned)n, CT_THREADS, chol_smem_bytes(cmax), st>>>(b);
    else {
      // tiles in global memory; clusters of up to 8 CTAs per factor when the factors alone
      // would leave most SMs idle
      const int cc = std::max(1, std::min(gt_cluster_max(ctx), kNumSM / std::max(1, (int)n)));
      if (cc == 1) {
        chol_tiled_kernel<<<(unsigned)n, CT_THREADS, CT_SMEM_BYTES, st>>>(b, 1);
      } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(cc * n), 1, 1);
        cfg.blockDim = dim3(CT_THREADS, 1, 1);
        cfg.dynamicSmemBytes = CT_SMEM_BYTES;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)cc;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (!cuda_ok(cudaLaunchKernelEx(&cfg, chol_tiled_kernel, b, cc))) return BKFAC_ERR_CUDA;
      }
    }
    LAUNCH_CHECK(ctx);
    i0 += n;
  }
  v.clear();
  prof_end(ctx, st);
  return BKFAC_OK;
}

// Two-stage reduction (sbr.cuh) of the batch's problems with p.sbr set: stage 1 panel by
// panel (panel QR, X = A22 V, W, A22 -= V W^T + W V^T), then the bulge chase to d, e.
bkfac_status run_sbr(bkfac_ctx ctx, const EigBatch& b, cudaStream_t st) {
  const int n = b.nprob;
  int pmax = 0, mmax = 0;
  for (int i = 0; i < n; ++i)
    if (b.p[i].sbr) { pmax = std::max(pmax, sbr_panels(b.p[i].m)); mmax = std::max(mmax, b.p[i].m); }
  constexpr int B = SBR_B;
  GemmStage gs;
  bkfac_status rs;
  for (int j = 0; j < pmax; ++j) {
    int lmax_j = 0;
    for (int i = 0; i < n; ++i)
      if (b.p[i].sbr && j < sbr_panels(b.p[i].m)) lmax_j = std::max(lmax_j, b.p[i].m - (j + 1) * B);
    double pf = 0.0;
    for (int i = 0; i < n; ++i)
      if (b.p[i].sbr && j < sbr_panels(b.p[i].m)) pf += 4.0 * (double)(b.p[i].m - (j + 1) * B) * B * B;
    prof_begin(ctx, "eig_sbr_panel", st, pf, 0.0);
    sbr_panel_kernel<<<(unsigned)n, SBR_PANEL_THREADS, sbr_panel_smem_bytes(mmax), st>>>(b, j);
    LAUNCH_CHECK(ctx);
    prof_end(ctx, st);
    if (ctx->sbr_x) {   // X = A22 V from the lower triangle (sbr_x_kernel)
      double xf = 0.0, xb = 0.0;
      int lmax = 0;
      for (int i = 0; i < n; ++i) {
        if (!b.p[i].sbr || j >= sbr_panels(b.p[i].m)) continue;
        const double L = b.p[i].m - (j + 1) * B;
        xf += 2.0 * L * L * B;
        xb += 4.0 * L * L;
        lmax = std::max(lmax, (int)L);
      }
      prof_begin(ctx, "eig_sbr_x", st, xf, xb);
      sbr_x_kernel<<<dim3((unsigned)ceil_div(lmax, SBR_X_ROWS), (unsigned)n), SBR_X_THREADS, sbr_x_smem_bytes(), st>>>(b, j);
      LAUNCH_CHECK(ctx);
      prof_end(ctx, st);
    } else {
      for (int i = 0; i < n; ++i) {     // X = A22 V
        const EigProb& q = b.p[i];
        if (!q.sbr || j >= sbr_panels(q.m)) continue;
        const int r0 = (j + 1) * B, L = q.m - r0;
        float* A22 = q.K + r0 + (long)r0 * q.ldk;
        gs.add(false, false, gp(A22, q.ldk, q.Vp + r0, q.m, q.Xp + r0, q.m, L, B, L, 1.f), 0);
      }
      if ((rs = run_gemms(ctx, gs, st, "gemm_sbr_x")) != BKFAC_OK) return rs;
    }
    prof_begin(ctx, "eig_sbr_w", st, pf, 0.0);
    if (ctx->sbr_x)   // Y = X T and the shares of V^T Y came out of sbr_x_kernel
      sbr_wfin_kernel<<<dim3((unsigned)ceil_div(lmax_j, SBR_X_ROWS), (unsigned)n), SBR_X_ROWS, 0, st>>>(b, j);
    else
      sbr_w_kernel<<<(unsigned)n, SBR_W_WARPS * 32, sbr_w_smem_bytes(), st>>>(b, j);
    LAUNCH_CHECK(ctx);
    prof_end(ctx, st);
    if (ctx->sbr_x) {   // A22 -= V W^T + W V^T on the lower 128 x 128 tiles (sbr_update_kernel)
      double uf = 0.0, ub = 0.0;
      int tmax = 0;
      for (int i = 0; i < n; ++i) {
        if (!b.p[i].sbr || j >= sbr_panels(b.p[i].m)) continue;
        const int L = b.p[i].m - (j + 1) * B;
        uf += 2.0 * (double)L * (L + 1) * 2 * B;          // lower triangle, K = 2B
        ub += 4.0 * (double)L * (L + 1);                  // its C0 read + C write
        tmax = std::max(tmax, sbr_u_tiles(L));
      }
      prof_begin(ctx, "eig_sbr_update", st, uf, ub);
      sbr_update_kernel<<<dim3((unsigned)tmax, (unsigned)n), SBR_U_THREADS, sbr_u_smem_bytes(), st>>>(b, j);
      LAUNCH_CHECK(ctx);
      prof_end(ctx, st);
      continue;
    }
    // A22 -= V W^T + W V^T  (symmetric: lower tiles computed, mirrored: X reads full storage)
    for (int i = 0; i < n; ++i) {
      const EigProb& q = b.p[i];
      if (!q.sbr || j >= sbr_panels(q.m)) continue;
      const int r0 = (j + 1) * B, L = q.m - r0;
      float* A22 = q.K + r0 + (long)r0 * q.ldk;
      GemmProb pu = gp(q.Vp + r0, q.m, q.Wp + r0, q.m, A22, q.ldk, L, L, 2 * B, -1.f, A22, q.ldk, 1.f);
      pu.A2 = q.Wp + r0; pu.lda2 = q.m;
      pu.B2 = q.Vp + r0; pu.ldb2 = q.m;
      pu.k1 = B;
      pu.sym = 1;
      gs.add(false, true, pu, 0);
    }
    if ((rs = run_gemms(ctx, gs, st, "gemm_sbr_update")) != BKFAC_OK) return rs;
  }
  double cf = 0.0;
  for (int i = 0; i < n; ++i)
    if (b.p[i].sbr) cf += 6.0 * (double)b.p[i].m * b.p[i].m * B;
  prof_begin(ctx, "eig_sbr_chase", st, cf, 0.0);
  sbr_chase_kernel<<<(unsigned)n, SBR_CHASE_WARPS * 32, sbr_chase_smem_bytes(), st>>>(b);
  LAUNCH_CHECK(ctx);
  prof_end(ctx, st);
  return BKFAC_OK;
}

// Auto mode (BKFAC_OPT_TWO_STAGE = 0): the two-stage reduction pays off when many large
// cores share the launch (its chase and back-transform are per-factor latency chains, the
// one-stage global-tile kernel is HBM-bound with one CTA per factor); with few (an 8-GPU
// rank's share) the one-stage kernel on clusters of up to 8 CTAs per factor is faster.
// Measured on one B200, ms per step of one rank's share of configs[4] (two-stage / one-stage),
// round 2 session 4 (band reduction on mma.sync): 96 factors 217.6 / >300, 48: 121.1 / 155.5,
// 24: 76.1 / 84.2, 12: 55.7 / 42.7 -- crossover near 20 (session 3: 24: 91.4 / 91.3).
constexpr int SBR_AUTO_MIN_FACTORS = 20;

bkfac_status run_eig(bkfac_ctx ctx, std::vector<EigProb>& v, cudaStream_t st) {
  if (ctx->two_stage == 0) {
    int nbig = 0;
    for (auto& q : v) nbig += q.sbr != 0;
    if (nbig > 0 && nbig < SBR_AUTO_MIN_FACTORS)
      for (auto& q : v) { q.sbr = 0; q.off = 1; }
  }
  size_t i0 = 0;
  static thread_local EigBatch b;
  while (i0 < v.size()) {
    const size_t n = std::min(v.size() - i0, (size_t)EIG_MAXP);
    b.nprob = (int)n;
    int mmax = 0, rmax = 0;
    for (size_t i = 0; i < n; ++i) {
      b.p[i] = v[i0 + i];
      mmax = std::max(mmax, b.p[i].m);
      rmax = std::max(rmax, b.p[i].r);
    }
    double m3 = 0.0, m2 = 0.0, m2r = 0.0, mr = 0.0;
    for (size_t i = 0; i < n; ++i) {
      const double m = b.p[i].m, r = b.p[i].r;
      m3 += m * m * m; m2 += m * m; m2r += m * m * r; mr += m * r;
    }
    // bkfac_brand_ea_update: the EA GEMM runs beside the tridiagonalisation on the SMs its
    // clusters leave idle.  It depends only on the work before this point (fork event here)
    // but is SUBMITTED after the tridiagonalisation, so the clusters are placed first.
    int ea_busy = 0;
    if (ctx->pending_ea) {
      int ngt = 0;
      for (size_t i = 0; i < n; ++i) ngt += !b.p[i].sbr && sytrd_tiled_cluster(b.p[i].m) == 0;
      const int cgt = std::max(1, std::min(gt_cluster_max(ctx), kNumSM / std::max(1, ngt)));
      for (size_t i = 0; i < n; ++i) {
        const int C = sytrd_tiled_cluster(b.p[i].m);
        ea_busy += b.p[i].sbr ? 1 : (C == 0 ? cgt : C);   // CTAs its reduction occupies
      }
      if (!cuda_ok(cudaEventRecord(ctx->ev_ea_fork, st))) return BKFAC_ERR_CUDA;
    }
    // sytrd: 4/3 m^3 flops; algorithmic bytes: read K (lower), write reflectors + T.  When
    // every factor's tiles live in global memory ("eig_sytrd_gt"), the one-stage reduction
    // streams the trailing lower triangle every column (symv + rank-2 update: read + write
    // of (m-k)^2/2 floats at step k, 4/3 m^3 bytes in all) -- that is its algorithmic traffic
    bool any_sbr = false, all_sbr = n > 0;
    for (size_t i = 0; i < n; ++i) { any_sbr |= b.p[i].sbr != 0; all_sbr &= b.p[i].sbr != 0; }
    if (any_sbr) {
      const bkfac_status rs0 = run_sbr(ctx, b, st);
      if (rs0 != BKFAC_OK) return rs0;
    }
    bool all_gt = n > 0;
    for (size_t i = 0; i < n; ++i) all_gt &= b.p[i].sbr || sytrd_tiled_cluster(b.p[i].m) == 0;
    if (all_sbr) {
      // every problem was reduced in two stages above
    } else {
    if (all_gt) prof_begin(ctx, "eig_sytrd_gt", st, 4.0 / 3.0 * m3, 4.0 / 3.0 * m3);
    else prof_begin(ctx, "eig_sytrd", st, 4.0 / 3.0 * m3, 4.0 * m2);
    {
      // one launch per cluster size; the launches are independent problems, so all but
      // the first run on side streams (fork/join) and overlap on the GPU
      static thread_local EigBatch sub[5];
      int ngroups = 0;
      const int Cs[5] = {0, 1, 2, 4, 8};
      int gC[5], gm[5];
      for (int ci = 0; ci < 5; ++ci) {
        EigBatch& sb = sub[ngroups];
        sb.nprob = 0;
        int msub = 0;
        for (size_t i = 0; i < n; ++i)
          if (!b.p[i].sbr && sytrd_tiled_cluster(b.p[i].m) == Cs[ci]) {
            sb.p[sb.nprob++] = b.p[i];
            msub = std::max(msub, b.p[i].m);
          }
        if (sb.nprob == 0) continue;
        int Cg = Cs[ci];
        if (ctx->syt_cluster > Cg && Cg >= 2) Cg = std::min(ctx->syt_cluster, 8);   // tuning: wider clusters
        gC[ngroups] = Cg; gm[ngroups] = msub; ++ngroups;
      }
      const bool fork = ngroups > 1 && ctx->ev_fork != nullptr;
      if (fork && !cuda_ok(cudaEventRecord(ctx->ev_fork, st))) return BKFAC_ERR_CUDA;
      for (int g = 0; g < ngroups; ++g) {
        cudaStream_t sg = (fork && g > 0) ? ctx->side[g - 1] : st;
        if (sg != st && !cuda_ok(cudaStreamWaitEvent(sg, ctx->ev_fork, 0))) return BKFAC_ERR_CUDA;
        const int C = gC[g], msub = gm[g];
        // tiles in global memory: one CTA per factor when the factors fill the GPU, else a
        // cluster of up to 8 CTAs per factor sharing its tiles through L2 (an 8-GPU rank's
        // share of configs[4]: 12 factors of m = 1536)
        const int cgt = std::max(1, std::min(gt_cluster_max(ctx), kNumSM / std::max(1, sub[g].nprob)));
        if (C == 0 && cgt == 1) {
          const int mp = (msub + 31) / 32 * 32;
          sytrd_tiled_kernel<1><<<(unsigned)sub[g].nprob, SYT_THREADS,
                                  sizeof(float) * (size_t)syt_gt_smem_floats(mp), sg>>>(sub[g], 1);
        } else if (C == 0) {
          const int mp = (msub + 31) / 32 * 32;
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3((unsigned)(cgt * sub[g].nprob), 1, 1);
          cfg.blockDim = dim3(SYT_THREADS, 1, 1);
          cfg.dynamicSmemBytes = sizeof(float) * (size_t)syt_gt_smem_floats(mp);
          cfg.stream = sg;
          cudaLaunchAttribute attr[1];
          attr[0].id = cudaLaunchAttributeClusterDimension;
          attr[0].val.clusterDim.x = (unsigned)cgt;
          attr[0].val.clusterDim.y = 1;
          attr[0].val.clusterDim.z = 1;
          cfg.attrs = attr;
          cfg.numAttrs = 1;
          if (!cuda_ok(cudaLaunchKernelEx(&cfg, sytrd_tiled_kernel<2>, sub[g], cgt))) return BKFAC_ERR_CUDA;
        } else {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3((unsigned)(C * sub[g].nprob), 1, 1);
          cfg.blockDim = dim3(SYT_THREADS, 1, 1);
          cfg.dynamicSmemBytes = sytrd_tiled_smem_bytes(msub, C);
          cfg.stream = sg;
          cudaLaunchAttribute attr[2];
          attr[0].id = cudaLaunchAttributeClusterDimension;
          attr[0].val.clusterDim.x = (unsigned)C;
          attr[0].val.clusterDim.y = 1;
          attr[0].val.clusterDim.z = 1;
          // highest scheduling priority: when the EA GEMM runs beside (bkfac_brand_ea_update),
          // pending clusters are placed before its pending CTAs
          static const int prio = [] { int lo = 0, hi = 0; cudaDeviceGetStreamPriorityRange(&lo, &hi); return hi; }();
          attr[1].id = cudaLaunchAttributePriority;
          attr[1].val.priority = prio;
          cfg.attrs = attr;
          cfg.numAttrs = 2;
          if (!cuda_ok(cudaLaunchKernelEx(&cfg, sytrd_tiled_kernel<0>, sub[g], C))) return BKFAC_ERR_CUDA;
        }
        LAUNCH_CHECK(ctx);
        if (sg != st && !cuda_ok(cudaEventRecord(ctx->ev_join[g - 1], sg))) return BKFAC_ERR_CUDA;
      }
      if (fork)
        for (int g = 1; g < ngroups; ++g)
          if (!cuda_ok(cudaStreamWaitEvent(st, ctx->ev_join[g - 1], 0))) return BKFAC_ERR_CUDA;
    }
    prof_end(ctx, st);
    }   // one-stage problems
    if (ctx->pending_ea) {
      auto f = std::move(ctx->pending_ea);
      ctx->pending_ea = nullptr;
      const bkfac_status re = f(ea_busy);
      if (re != BKFAC_OK) return re;
      // mode 4: the rest of the eigensolver waits for the EA (which then only shares the GPU
      // with the tridiagonalisation)
      if (ctx->ea_join_early && !cuda_ok(cudaStreamWaitEvent(st, ctx->ev_ea_done, 0))) return BKFAC_ERR_CUDA;
    }
#ifdef BKFAC_SYT_TIMING
    i0 += n;
    continue;   // tuning builds: keep the sytrd timing sums in Y
#endif
    prof_begin(ctx, "eig_bisect", st, 0.0, 0.0);
    bisect_kernel<<<dim3((unsigned)n, (unsigned)ceil_div(rmax, BIS_WARPS * BIS_E)), BIS_WARPS * 32,
                    sizeof(double) * 3 * (size_t)mmax, st>>>(b);
    LAUNCH_CHECK(ctx);
    prof_end(ctx, st);
    prof_begin(ctx, "eig_invit", st, 0.0, 8.0 * mr);
    invit_kernel<<<dim3((unsigned)n, (unsigned)ceil_div(rmax, INV_THREADS)), INV_THREADS,
                   sizeof(double) * 2 * (size_t)mmax, st>>>(b);
    LAUNCH_CHECK(ctx);
    prof_end(ctx, st);
    prof_begin(ctx, "eig_cluster", st, 0.0, 0.0);
    cluster_kernel<<<(unsigned)n, 1024, 0, st>>>(b);
    LAUNCH_CHECK(ctx);
    prof_end(ctx, st);
    // back-transform V = H Y, blocked (eig.cuh 5'): 2 m^2 r flops in two GEMMs per panel
    // of BT_PW reflectors, applied last panel first
    {
      if (any_sbr) {   // Q2 (chase reflectors) first: Zr = Q2 Y
        double q2f = 0.0;
        for (size_t i = 0; i < n; ++i)
          if (b.p[i].sbr) q2f += 2.0 * (double)b.p[i].m * b.p[i].m * b.p[i].r;
        prof_begin(ctx, "eig_sbr_q2", st, q2f, 0.0);
        int nsbr = 0;
        for (size_t i = 0; i < n; ++i) nsbr += b.p[i].sbr != 0;
        if ((long)nsbr * ceil_div(rmax, SBR_Q2_THREADS) >= kNumSM)
          sbr_q2_kernel<SBR_Q2_THREADS><<<dim3((unsigned)n, (unsigned)ceil_div(rmax, SBR_Q2_THREADS)), SBR_Q2_THREADS, 0, st>>>(b);
        else
          sbr_q2_kernel<32><<<dim3((unsigned)n, (unsigned)ceil_div(rmax, 32)), 32, 0, st>>>(b);
        LAUNCH_CHECK(ctx);
        prof_end(ctx, st);
      }
      int pmax = 0;
      for (size_t i = 0; i < n; ++i) pmax = std::max(pmax, bt_panels(b.p[i].m, b.p[i].off));
      prof_begin(ctx, "eig_backtr", st, 0.0, 4.0 * m2 + 12.0 * mr);
      backtr_prep_kernel<<<dim3((unsigned)n, 64), 256, 0, st>>>(b);
      LAUNCH_CHECK(ctx);
      prof_end(ctx, st);
      GemmStage gs;
      bkfac_status rs2;
      if (pmax > 0) {
        for (size_t i = 0; i < n; ++i) {      // S_j = W_j^T W_j
          const EigProb& q = b.p[i];
          for (int j = 0; j < bt_panels(q.m, q.off); ++j) {
            const int r0 = j * BT_PW + q.off, np = std::min(BT_PW, q.m - q.off - 1 - j * BT_PW);
            const float* Wj = q.K + r0 + (long)(j * BT_PW) * q.ldk;
            gs.add(true, false, gp(Wj, q.ldk, Wj, q.ldk, q.Sw + (long)j * 2 * BT_PW * BT_PW, BT_PW, np, np,
                                   q.m - r0, 1.f), 0);
          }
        }
        // S and U define the compact-WY operator I - W T W^T: their errors become departures
        // from orthogonality of V.  On the 3xTF32 tensor-core path (~1e-6) those departures
        // are removed by the per-step Newton-Schulz refresh of U_out (R8; the 50-step config-2
        // chain is unchanged: 5.2e-6 vs 5.0e-6 with fp32 SIMT).  BKFAC_BT_SIMT selects the
        // fp32 SIMT kernel for them instead.
        gs.fp32_simt = ctx->bt_simt != 0;
        if ((rs2 = run_gemms(ctx, gs, st, "gemm_backtr_s")) != BKFAC_OK) return rs2;
        prof_begin(ctx, "eig_backtr", st, 0.0, 0.0);
        backtr_t_kernel<<<dim3((unsigned)n, (unsigned)pmax), BT_THREADS, bt_smem_bytes(), st>>>(b);
        LAUNCH_CHECK(ctx);
        prof_end(ctx, st);
        for (size_t i = 0; i < n; ++i) {      // U_j = W_j T_j
          const EigProb& q = b.p[i];
          for (int j = 0; j < bt_panels(q.m, q.off); ++j) {
            const int r0 = j * BT_PW + q.off, np = std::min(BT_PW, q.m - q.off - 1 - j * BT_PW);
            gs.add(false, false, gp(q.K + r0 + (long)(j * BT_PW) * q.ldk, q.ldk,
                                    q.Sw + (long)j * 2 * BT_PW * BT_PW + BT_PW * BT_PW, BT_PW,
                                    q.Uw + (long)(j * BT_PW) * q.m + r0, q.m, q.m - r0, np, np, 1.f), 0);
          }
        }
        gs.fp32_simt = ctx->bt_simt != 0;
        if ((rs2 = run_gemms(ctx, gs, st, "gemm_backtr_wt")) != BKFAC_OK) return rs2;
      }
      for (int j = pmax - 1; j >= 0; --j) {
        for (size_t i = 0; i < n; ++i) {
          const EigProb& q = b.p[i];
          if (j >= bt_panels(q.m, q.off)) continue;
          const int r0 = j * BT_PW + q.off, mr0 = q.m - r0;
          const int np = std::min(BT_PW, q.m - q.off - 1 - j * BT_PW);   // reflectors in this panel
          // Z = W_j^T V(r0:, :)   (np x r)
          gs.add(true, false, gp(q.K + r0 + (long)(j * BT_PW) * q.ldk, q.ldk, q.V + r0, q.ldv, q.Zw, BT_PW,
                                 np, q.r, mr0, 1.f), 0);
        }
        if ((rs2 = run_gemms(ctx, gs, st, "gemm_backtr_z")) != BKFAC_OK) return rs2;
        for (size_t i = 0; i < n; ++i) {
          const EigProb& q = b.p[i];
          if (j >= bt_panels(q.m, q.off)) continue;
          const int r0 = j * BT_PW + q.off, mr0 = q.m - r0;
          const int np = std::min(BT_PW, q.m - q.off - 1 - j * BT_PW);
          // V(r0:, :) -= U_j(r0:, 0:np) Z
          gs.add(false, false, gp(q.Uw + (long)(j * BT_PW) * q.m + r0, q.m, q.Zw, BT_PW, q.V + r0, q.ldv,
                                  mr0, q.r, np, -1.f, q.V + r0, q.ldv, 1.f), 0);
        }
        if ((rs2 = run_gemms(ctx, gs, st, "gemm_backtr_u")) != BKFAC_OK) return rs2;
      }
    }
    i0 += n;
  }
  v.clear();
  return BKFAC_OK;
}

EigProb eig_prob(bkfac_ctx ctx, const EigWs& w, int m, int r, float* V, int ldv, float* Dout,
                 int* status) {
  EigProb p;
  p.K = at<float>(ctx, w.K); p.ldk = m;
  p.m = m; p.r = r;
  p.d = at<float>(ctx, w.d); p.e = at<float>(ctx, w.e); p.tau = at<float>(ctx, w.tau);
  p.lam = at<double>(ctx, w.lam);
  p.Y = at<double>(ctx, w.Y);
  p.scr = at<double>(ctx, w.scr);
  p.piv = at<unsigned char>(ctx, w.piv);
  p.V = V; p.ldv = ldv;
  p.Dout = Dout;
  p.status = status;
  p.gtiles = w.gt ? at<float>(ctx, w.gt) : nullptr;
  p.Uw = at<float>(ctx, w.U);
  p.Zw = at<float>(ctx, w.Z);
  p.Sw = at<float>(ctx, w.S);
  p.sbr = use_sbr(ctx, w, m) ? 1 : 0;
  p.off = p.sbr ? SBR_B : 1;
  p.Vp = w.sbr ? at<float>(ctx, w.Vp) : nullptr;
  p.Vt = w.sbr ? at<float>(ctx, w.Vt) : nullptr;
  p.Wt = w.sbr ? at<float>(ctx, w.Wt) : nullptr;
  p.Zp = w.sbr ? at<float>(ctx, w.Zp) : nullptr;
  p.Xp = w.sbr ? at<float>(ctx, w.Xp) : nullptr;
  p.Wp = w.sbr ? at<float>(ctx, w.Wp) : nullptr;
  p.Tp = w.sbr ? at<float>(ctx, w.Tp) : nullptr;
  p.AB = w.sbr ? at<float>(ctx, w.AB) : nullptr;
  p.Vq = w.sbr ? at<float>(ctx, w.Vq) : nullptr;
  p.tq = w.sbr ? at<float>(ctx, w.tq) : nullptr;
  p.Zr = reinterpret_cast<float*>(p.scr);   // free once inverse iteration has finished
  return p;
}

CholProb chol_prob(bkfac_ctx ctx, const float* G, int c, size_t L, size_t Li, size_t scr,
                   int* status, float shift = 0.f) {
  CholProb p;
  p.G = G; p.ldg = c;
  p.L = at<float>(ctx, L); p.Linv = at<float>(ctx, Li);
  p.scratch = at<float>(ctx, scr);
  p.status = status;
  p.c = c;
  p.shift = shift;
  return p;
}

void gemm_ws(GemmProb& p, float* ws) { p.ws = ws; }

}  // namespace

// =====================================================================================
extern "C" {

const char* bkfac_status_string(bkfac_status s) {
  switch (s) {
    case BKFAC_OK: return "ok";
    case BKFAC_ERR_INVALID_ARG: return "invalid argument";
    case BKFAC_ERR_DIM: return "dimension error";
    case BKFAC_ERR_RANK: return "rank too large";
    case BKFAC_ERR_ALIAS: return "output aliases input";
    case BKFAC_ERR_WORKSPACE: return "workspace missing or too small";
    case BKFAC_ERR_CUDA: return "CUDA error";
    case BKFAC_ERR_NUMERIC: return "numeric failure on device";
    case BKFAC_ERR_UNSUPPORTED: return "unsupported shape";
  }
  return "unknown status";
}

const char* bkfac_build_info(void) {
  return "bkfac sm_100a; GEMM: " BKFAC_GEMM_PATH "; CholeskyQR2; Householder "
         "tridiagonalisation + fp64 multisection/inverse iteration";
}

bkfac_status bkfac_init(bkfac_ctx* out, const bkfac_factor_desc* factors, int nfactors,
                        const bkfac_layer_desc* layers, int nlayers, int device) {
  if (!out || nfactors < 0 || nlayers < 0 || (nfactors > 0 && !factors) ||
      (nlayers > 0 && !layers))
    return BKFAC_ERR_INVALID_ARG;
  *out = nullptr;
  bkfac_ctx c = new (std::nothrow) bkfac_ctx_s();
  if (!c) return BKFAC_ERR_INVALID_ARG;
  c->device = device;
  Arena a;
  c->status_off = a.take(sizeof(int) * (size_t)(nfactors + nlayers + 1));
  for (int i = 0; i < nfactors; ++i) {
    FactorPlan fp;
    fp.d = factors[i];
    const int n = fp.d.n, r = fp.d.r, cm = fp.d.c_max;
    if (n <= 0 || r <= 0 || r > n || cm <= 0) { delete c; return BKFAC_ERR_DIM; }
    fp.dense = (r + cm >= n);
    const bool full = (fp.d.flags & BKFAC_FACTOR_FULL_RANK) != 0;
    fp.nld = (n + 31) / 32 * 32;
    fp.rout = full ? std::min(n, r + cm) : r;
    const int ro = fp.rout;
    if (fp.dense) {
      fp.m = n;
      fp.T = a.take(sizeof(float) * (size_t)n * r);
      plan_eig(a, fp.eig, n, ro);
    } else {
      const int m = r + cm;
      fp.m = m;
      fp.W = a.take(sizeof(float) * (size_t)m * cm);
      fp.P2 = a.take(sizeof(float) * (size_t)r * cm);
      fp.R = a.take(sizeof(float) * (size_t)fp.nld * cm);
      fp.Qb = a.take(sizeof(float) * (size_t)fp.nld * cm);
      if (n % 4 != 0) {   // caller buffers with a leading dimension the vector loads cannot use
        fp.Ms = a.take(sizeof(float) * (size_t)fp.nld * cm);
        fp.Us = a.take(sizeof(float) * (size_t)fp.nld * r);
      }
      const size_t cc = sizeof(float) * (size_t)cm * cm;
      fp.G = a.take(cc); fp.L1 = a.take(cc); fp.L1i = a.take(cc); fp.L2 = a.take(cc); fp.L2i = a.take(cc);
      fp.cscr = a.take(sizeof(float) * chol_tiled_scratch_floats(cm));
      fp.Vf = a.take(sizeof(float) * (size_t)cm * ro);
      fp.ws_elems = (long)kSplitMax * std::max(r, cm) * (long)cm;
      fp.ws = a.take(sizeof(float) * fp.ws_elems);
      plan_eig(a, fp.eig, m, ro);
    }
    fp.Urot = a.take(sizeof(float) * (size_t)fp.nld * ro);
    fp.Gref = a.take(sizeof(float) * (size_t)ro * ro);
    fp.wsr_elems = (long)kSplitMax * ro * (long)ro;
    fp.wsr = a.take(sizeof(float) * fp.wsr_elems);
    if (fp.d.flags & BKFAC_FACTOR_DENSE_EA) {
      fp.rsvd = true;
      const int l = std::min(n, r + kRsvdOversampleMax);
      fp.lmax = l;
      const size_t nl = sizeof(float) * (size_t)n * l;
      fp.Yr = a.take(nl); fp.Qr = a.take(nl); fp.Q2r = a.take(nl); fp.Tr = a.take(nl);
      const size_t ll = sizeof(float) * (size_t)l * l;
      fp.Gr = a.take(ll); fp.L1r = a.take(ll); fp.L1ir = a.take(ll); fp.L2r = a.take(ll);
      fp.L2ir = a.take(ll); fp.Br = a.take(ll);
      fp.cscr_r = a.take(sizeof(float) * chol_tiled_scratch_floats(l));
      fp.ws_r_elems = (long)kSplitMax * l * (long)l;
      fp.ws_r = a.take(sizeof(float) * fp.ws_r_elems);
      plan_eig(a, fp.eig_r, l, r);
    }
    c->f.push_back(fp);
  }
  for (int i = 0; i < nlayers; ++i) {
    LayerPlan lp;
    lp.d = layers[i];
    const auto& d = lp.d;
    if (d.d_G <= 0 || d.d_A <= 0 || d.r_G < 0 || d.r_A < 0 || d.r_G > d.d_G || d.r_A > d.d_A ||
        d.n_max < 0) {
      delete c;
      return BKFAC_ERR_DIM;
    }
    lp.ldY = pad32(d.d_G);
    lp.ldXt = pad32(d.d_A);
    lp.Y = a.take(sizeof(float) * (size_t)lp.ldY * std::max(d.r_A, 1));
    lp.Xt = a.take(sizeof(float) * (size_t)lp.ldXt * std::max(d.r_G, 1));
    lp.Z = a.take(sizeof(float) * (size_t)std::max(d.r_G, 1) * std::max(d.r_A, 1));
    lp.sA = a.take(sizeof(float) * std::max(d.r_A, 1));
    lp.sG = a.take(sizeof(float) * std::max(d.r_G, 1));
    lp.lam = a.take(sizeof(float) * 8);
    if (d.n_max > 0) {
      const size_t nm = (size_t)d.n_max;
      lp.fPG = a.take(sizeof(float) * nm * std::max(d.r_G, 1));
      lp.fPA = a.take(sizeof(float) * nm * std::max(d.r_A, 1));
      lp.fGb = a.take(sizeof(float) * nm * d.d_G);
      lp.fAb = a.take(sizeof(float) * nm * d.d_A);
      lp.fws_elems = (long)kSplitMax * (long)nm * std::max(std::max(d.r_G, d.r_A), 1);
      lp.fws = a.take(sizeof(float) * lp.fws_elems);
      lp.fws2 = a.take(sizeof(float) * lp.fws_elems);
    }
    lp.ws_elems = (long)kSplitMax * std::max((long)d.d_G * d.r_A, (long)d.d_A * d.r_G);
    lp.ws = a.take(sizeof(float) * std::max<long>(lp.ws_elems, 1));
    c->l.push_back(lp);
  }
  // every eigenproblem order must fit one of the tridiagonalisation paths: shared-memory
  // cluster tiles (m <= 864), two-stage (m <= 1632), or global tiles whose per-CTA vectors and
  // staging fit the shared-memory opt-in (m up to ~3100)
  auto eig_ok = [](int m) {
    const int m_pad = (m + 31) / 32 * 32;
    return sytrd_tiled_cluster(m) != 0 || sbr_supported(m) || syt_gt_smem_floats(m_pad) <= SYT_SMEM_FLOATS;
  };
  for (const auto& fp : c->f) {
    if (!eig_ok(fp.m) || (fp.rsvd && !eig_ok(fp.lmax))) { delete c; return BKFAC_ERR_UNSUPPORTED; }
  }
  c->ws_bytes = a.cur;
  cudaError_t e = cudaMallocHost(&c->host_status, sizeof(int) * (size_t)(nfactors + nlayers + 1));
  if (e != cudaSuccess) { delete c; return BKFAC_ERR_CUDA; }
  // opt-in shared memory sizes
  int dev_prev = 0;
  cudaGetDevice(&dev_prev);
  cudaSetDevice(device);
  const int big = 220 * 1024;  // below the 227 KB opt-in limit minus static smem
  bool attr_ok = true;
  attr_ok &= cudaFuncSetAttribute(sytrd_tiled_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, SYT_SMEM_FLOATS * 4) == cudaSuccess;
  attr_ok &= cudaFuncSetAttribute(sytrd_tiled_kernel<0>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
  attr_ok &= cudaFuncSetAttribute(sytrd_tiled_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, SYT_SMEM_FLOATS * 4) == cudaSuccess;
  attr_ok &= cudaFuncSetAttribute(sytrd_tiled_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SYT_SMEM_FLOATS * 4) == cudaSuccess;
  attr_ok &= cudaFuncSetAttribute(backtr_t_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bt_smem_bytes()) == cudaSuccess;
  attr_ok &= cudaFuncSetAttribute(invit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, big) == cudaSuccess;
  attr_ok &= cudaFuncSetAttribute(bisect_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, big) == cudaSuccess;
  attr_ok &= cudaFuncSetAttribute(chol_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CT_SMEM_BYTES) == cudaSuccess;
  attr_ok &= cudaFuncSetAttribute(chol_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)chol_smem_bytes(32 * CS_MAXNB)) == cudaSuccess;
  attr_ok &= cudaFuncSetAttribute(sbr_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sbr_panel_smem_bytes(SBR_MAX_L + SBR_B)) == cudaSuccess;
  attr_ok &= cudaFuncSetAttribute(sbr_x_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sbr_x_smem_bytes()) == cudaSuccess;
  attr_ok &= cudaFuncSetAttribute(sbr_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sbr_u_smem_bytes()) == cudaSuccess;
  attr_ok &= cudaFuncSetAttribute(sbr_w_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sbr_w_smem_bytes()) == cudaSuccess;
  attr_ok &= cudaFuncSetAttribute(sbr_chase_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sbr_chase_smem_bytes()) == cudaSuccess;
  attr_ok &= tc_init_attributes();
  if (!attr_ok) fprintf(stderr, "bkfac: cudaFuncSetAttribute failed: %s\n", cudaGetErrorString(cudaGetLastError()));
  cudaGetLastError();  // never leave a sticky error behind
  cudaSetDevice(dev_prev);
  cudaSetDevice(device);
  for (int i = 0; i < 4; ++i) {
    if (cudaStreamCreateWithFlags(&c->side[i], cudaStreamNonBlocking) != cudaSuccess) c->side[i] = nullptr;
    if (cudaEventCreateWithFlags(&c->ev_join[i], cudaEventDisableTiming) != cudaSuccess) c->ev_join[i] = nullptr;
  }
  if (cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess) c->ev_fork = nullptr;
  if (cudaStreamCreateWithFlags(&c->ea_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_ea_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_ea_done, cudaEventDisableTiming) != cudaSuccess) {
    fprintf(stderr, "bkfac: side stream creation failed\n");
    return BKFAC_ERR_CUDA;
  }
  for (int i = 0; i < 4; ++i)
    if (!c->side[i] || !c->ev_join[i]) { if (c->ev_fork) cudaEventDestroy(c->ev_fork); c->ev_fork = nullptr; }
  cudaGetLastError();
  cudaSetDevice(dev_prev);
  *out = c;
  return BKFAC_OK;
}

bkfac_status bkfac_set_option(bkfac_ctx c, int option, int value) {
  if (!c) return BKFAC_ERR_INVALID_ARG;
  switch (option) {
    case BKFAC_OPT_TWO_STAGE: if (value < 0 || value > 2) return BKFAC_ERR_INVALID_ARG; c->two_stage = value; break;
    case BKFAC_OPT_NVTX: c->nvtx = value != 0; break;
    case BKFAC_OPT_SBR_X: c->sbr_x = value != 0; break;
    case BKFAC_OPT_GT_CLUSTER: if (value < 1 || value > 8) return BKFAC_ERR_INVALID_ARG; c->gt_cluster = value; break;
    case BKFAC_OPT_GEMM_PAIR: if (value < 0 || value > 2) return BKFAC_ERR_INVALID_ARG; c->pair_mode = value; break;
    case BKFAC_OPT_GEMM_SIMT: c->use_tc = value == 0; break;
    case BKFAC_OPT_EA_MODE: if (value < 0 || value > 4) return BKFAC_ERR_INVALID_ARG; c->ea_mode = value; break;
    case BKFAC_OPT_EA_CAP: if (value < 0) return BKFAC_ERR_INVALID_ARG; c->ea_cap = value; break;
    case BKFAC_OPT_SYT_CLUSTER: if (value < 0 || value > 8) return BKFAC_ERR_INVALID_ARG; c->syt_cluster = value; break;
    case BKFAC_OPT_BT_SIMT: c->bt_simt = value != 0; break;
    case BKFAC_OPT_CHOL_BLOCKED: c->chol_blocked = value != 0; break;
    case BKFAC_OPT_PREC_BLOCK: if (value < 0 || value > 4096) return BKFAC_ERR_INVALID_ARG; c->prec_block = value; break;
    case BKFAC_OPT_GEMM_CAP: if (value < 0 || value > kNumSM) return BKFAC_ERR_INVALID_ARG; c->user_cap = value; break;
    default: return BKFAC_ERR_INVALID_ARG;
  }
  return BKFAC_OK;
}

size_t bkfac_workspace_bytes(bkfac_ctx c) { return c ? c->ws_bytes : 0; }

bkfac_status bkfac_set_workspace(bkfac_ctx c, void* p, size_t bytes) {
  if (!c || !p) return BKFAC_ERR_INVALID_ARG;
  if (bytes < c->ws_bytes || (reinterpret_cast<uintptr_t>(p) & 255)) return BKFAC_ERR_WORKSPACE;
  c->ws = static_cast<char*>(p);
  c->ws_cap = bytes;
  if (!cuda_ok(cudaMemset(c->ws + c->status_off, 0, sizeof(int) * (c->f.size() + c->l.size() + 1))))
    return BKFAC_ERR_CUDA;
  return BKFAC_OK;
}

bkfac_status bkfac_destroy(bkfac_ctx c) {
  if (!c) return BKFAC_ERR_INVALID_ARG;
  if (c->host_status) cudaFreeHost(c->host_status);
  for (auto e : c->pool) cudaEventDestroy(e);
  for (int i = 0; i < 4; ++i) {
    if (c->side[i]) cudaStreamDestroy(c->side[i]);
    if (c->ev_join[i]) cudaEventDestroy(c->ev_join[i]);
  }
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ea_stream) cudaStreamDestroy(c->ea_stream);
  if (c->ev_ea_fork) cudaEventDestroy(c->ev_ea_fork);
  if (c->ev_ea_done) cudaEventDestroy(c->ev_ea_done);
  delete c;
  return BKFAC_OK;
}

uint64_t bkfac_launch_count(bkfac_ctx c) { return c ? c->launches : 0; }

bkfac_status bkfac_profile_enable(bkfac_ctx c, int enable) {
  if (!c) return BKFAC_ERR_INVALID_ARG;
  c->prof = enable != 0;
  c->recs.clear();
  c->pool_used = 0;
  c->open_rec = -1;
  return BKFAC_OK;
}

namespace {
int profile_aggregate(bkfac_ctx c, bkfac_stage_stat* out, int max_out, bool clear, size_t begin,
                      size_t end) {
  if (!c) return -1;
  std::map<std::string, bkfac_stage_stat> agg;
  std::vector<std::string> order;
  end = std::min(end, c->recs.size());
  for (size_t ri = begin; ri < end; ++ri) {
    const auto& r = c->recs[ri];
    if (!cuda_ok(cudaEventSynchronize(r.b))) return -1;
    float ms = 0.f;
    if (!cuda_ok(cudaEventElapsedTime(&ms, r.a, r.b))) return -1;
    auto it = agg.find(r.tag);
    if (it == agg.end()) {
      bkfac_stage_stat z;
      memset(&z, 0, sizeof(z));
      strncpy(z.name, r.tag.c_str(), sizeof(z.name) - 1);
      it = agg.emplace(r.tag, z).first;
      order.push_back(r.tag);
    }
    it->second.calls += 1;
    it->second.launches += (long long)r.launches;
    it->second.ms += ms;
    it->second.flops += r.flops;
    it->second.bytes += r.bytes;
  }
  int n = 0;
  for (auto& t : order) {
    if (out && n < max_out) out[n] = agg[t];
    ++n;
  }
  if (clear) {
    c->recs.clear();
    c->pool_used = 0;
  }
  return n;
}
}  // namespace

int bkfac_profile_read(bkfac_ctx c, bkfac_stage_stat* out, int max_out) {
  return profile_aggregate(c, out, max_out, true, 0, ~size_t(0));
}

int bkfac_profile_count(bkfac_ctx c) { return c ? (int)c->recs.size() : -1; }

int bkfac_profile_read_range(bkfac_ctx c, int begin, int end, bkfac_stage_stat* out, int max_out) {
  if (!c || begin < 0 || end < begin) return -1;
  return profile_aggregate(c, out, max_out, false, (size_t)begin, (size_t)end);
}

// ------------------------------------------------------------------------- Brand
bkfac_status bkfac_brand_update(bkfac_ctx ctx, const bkfac_brand_args* args, int count,
                                void* stream) {
  if (!ctx || (count > 0 && !args) || count < 0) return BKFAC_ERR_INVALID_ARG;
  if (!ctx->ws) return BKFAC_ERR_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (int i = 0; i < count; ++i) {
    const auto& a = args[i];
    if (a.factor < 0 || a.factor >= (int)ctx->f.size()) return BKFAC_ERR_INVALID_ARG;
    const auto& fp = ctx->f[a.factor];
    if (!a.U_in || !a.D_in || !a.M || !a.U_out || !a.D_out) return BKFAC_ERR_INVALID_ARG;
    if (!(a.alpha >= 0.f) || !(a.beta > 0.f) || !std::isfinite(a.alpha) || !std::isfinite(a.beta))
      return BKFAC_ERR_INVALID_ARG;
    if (a.c <= 0 || a.c > fp.d.c_max) return BKFAC_ERR_DIM;
    if (!ld_ok(a.ld_U, fp.d.n) || !ld_ok(a.ld_M, fp.d.n)) return BKFAC_ERR_DIM;
    if (a.U_out == a.U_in || a.D_out == a.D_in) return BKFAC_ERR_ALIAS;
    for (int j = 0; j < i; ++j)
      if (args[j].factor == a.factor) return BKFAC_ERR_INVALID_ARG;  // one update per factor per batch
  }
  if (count == 0) return BKFAC_OK;
  int dev_prev = 0;
  cudaGetDevice(&dev_prev);
  if (dev_prev != ctx->device) cudaSetDevice(ctx->device);

  bkfac_status rs = BKFAC_OK;
  GemmStage gs;
  std::vector<EwProb> ew;
  std::vector<CholProb> ch;
  std::vector<EigProb> eg;
  std::vector<int> brand, dense;
  for (int i = 0; i < count; ++i) (ctx->f[args[i].factor].dense ? dense : brand).push_back(i);

  auto run = [&](const char* tag) -> bkfac_status { return run_gemms(ctx, gs, st, tag); };
  // output eigenpairs of this call: r, or (BKFAC_FACTOR_FULL_RANK) all min(n, r + c)
  auto rout_of = [&](const bkfac_brand_args& a) {
    const auto& fp = ctx->f[a.factor];
    return (fp.d.flags & BKFAC_FACTOR_FULL_RANK) ? std::min(fp.d.n, fp.d.r + a.c) : fp.d.r;
  };
  auto ldU = [&](const bkfac_brand_args& a) { return ldx(a.ld_U, ctx->f[a.factor].d.n); };
  auto ldM = [&](const bkfac_brand_args& a) { return ldx(a.ld_M, ctx->f[a.factor].d.n); };
  // internal 16-byte-aligned copies (ld nld) of M / U_in: odd n and a caller layout the
  // vector loads cannot use
  auto useMs = [&](const bkfac_brand_args& a) { return ctx->f[a.factor].Ms && !al16(a.M, ldM(a)); };
  auto useUs = [&](const bkfac_brand_args& a) { return ctx->f[a.factor].Us && !al16(a.U_in, ldU(a)); };
#define STAGE(x) do { if ((rs = (x)) != BKFAC_OK) goto done; } while (0)

  // full-rank factors with c < c_max: zero the output columns / entries beyond r + c
  for (int i = 0; i < count; ++i) {
    const auto& a = args[i];
    const auto& fp = ctx->f[a.factor];
    const int ro = rout_of(a);
    if (ro < fp.rout) {
      if (!cuda_ok(cudaMemsetAsync(a.U_out + (size_t)ldU(a) * ro, 0,
                                   sizeof(float) * ((size_t)ldU(a) * (fp.rout - ro - 1) + fp.d.n), st)) ||
          !cuda_ok(cudaMemsetAsync(a.D_out + ro, 0, sizeof(float) * (fp.rout - ro), st))) {
        rs = BKFAC_ERR_CUDA;
        goto done;
      }
    }
  }

  // ---------------- dense path (r + c >= n): K = alpha U diag(D) U^T + beta M M^T
  if (!dense.empty()) {
    for (int i : dense) {
      const auto& a = args[i];
      const auto& fp = ctx->f[a.factor];
      if (a.alpha != 0.f) {
        EwProb e{};
        e.Y = at<float>(ctx, fp.T); e.ldy = fp.d.n; e.X = a.U_in; e.ldx = ldU(a);
        e.vec = a.D_in; e.rows = fp.d.n; e.cols = fp.d.r; e.op = EW_SCALE_COLS;
        ew.push_back(e);
      }
    }
    STAGE(run_ew(ctx, ew, st, "ew_dense_scale"));
    {   // M reaches the tensor cores only as an MMA operand on this path: guard it (every
        // dense factor, in launches of up to NF_MAXP)
      static thread_local NfBatch nb;
      for (size_t i0 = 0; i0 < dense.size(); i0 += NF_MAXP) {
        nb.nprob = 0;
        for (size_t q = i0; q < std::min(dense.size(), i0 + NF_MAXP); ++q) {
          const auto& a = args[dense[q]];
          nb.p[nb.nprob++] = NfProb{a.M, ctx->f[a.factor].d.n, a.c, ldM(a), status_ptr(ctx, a.factor)};
        }
        nonfinite_kernel<<<dim3(16, (unsigned)nb.nprob), 256, 0, st>>>(nb);
        LAUNCH_CHECK(ctx);
      }
    }
    for (int i : dense) {
      const auto& a = args[i];
      const auto& fp = ctx->f[a.factor];
      if (a.alpha != 0.f) {
        const int n = fp.d.n;
        gs.add(false, true, gp(at<float>(ctx, fp.T), n, a.U_in, ldU(a), at<float>(ctx, fp.eig.K), n, n, n,
                               fp.d.r, a.alpha), 0);
      }
    }
    STAGE(run("gemm_dense_core"));
    for (int i : dense) {
      const auto& a = args[i];
      const auto& fp = ctx->f[a.factor];
      const int n = fp.d.n;
      float* K = at<float>(ctx, fp.eig.K);
      gs.add(false, true, gp(a.M, ldM(a), a.M, ldM(a), K, n, n, n, a.c, a.beta, K, n, a.alpha != 0.f ? 1.f : 0.f), 0);
    }
    STAGE(run("gemm_dense_core"));
    for (int i : dense) {
      const auto& a = args[i];
      const auto& fp = ctx->f[a.factor];
      eg.push_back(eig_prob(ctx, fp.eig, fp.d.n, rout_of(a), at<float>(ctx, fp.Urot), fp.nld, a.D_out,
                            status_ptr(ctx, a.factor)));
    }
  }

  // ---------------- Brand path
  if (!brand.empty()) {
    // M and U_in of factors with n % 4 != 0 are first copied to ld = nld (one streaming
    // pass, ~2 (c + r) n floats), so every GEMM that reads them takes the 16-byte loads
    for (int i : brand) {
      const auto& a = args[i];
      const auto& fp = ctx->f[a.factor];
      const int n = fp.d.n;
      if (useMs(a)) {
        EwProb e{};
        e.Y = at<float>(ctx, fp.Ms); e.ldy = fp.nld; e.X = a.M; e.ldx = ldM(a); e.rows = n; e.cols = a.c;
        e.op = EW_COPY;
        ew.push_back(e);
      }
      if (useUs(a)) {
        EwProb u{};
        u.Y = at<float>(ctx, fp.Us); u.ldy = fp.nld; u.X = a.U_in; u.ldx = ldU(a); u.rows = n; u.cols = fp.d.r;
        u.op = EW_COPY;
        ew.push_back(u);
      }
    }
    if (!ew.empty()) STAGE(run_ew(ctx, ew, st, "ew_align"));
    // operand views: the aligned copies where they exist
    auto Uin = [&](const bkfac_brand_args& a) -> const float* {
      return useUs(a) ? at<float>(ctx, ctx->f[a.factor].Us) : a.U_in;
    };
    auto Min = [&](const bkfac_brand_args& a) -> const float* {
      return useMs(a) ? at<float>(ctx, ctx->f[a.factor].Ms) : a.M;
    };
    auto ldUin = [&](const bkfac_brand_args& a) -> int {
      return useUs(a) ? ctx->f[a.factor].nld : ldU(a);
    };
    auto ldMin = [&](const bkfac_brand_args& a) -> int {
      return useMs(a) ? ctx->f[a.factor].nld : ldM(a);
    };
    // A: P = U^T M  -> W rows [0, r)
    for (int i : brand) {
      const auto& a = args[i];
      const auto& fp = ctx->f[a.factor];
      const int n = fp.d.n, r = fp.d.r;
      GemmProb p = gp(Uin(a), ldUin(a), Min(a), ldMin(a), at<float>(ctx, fp.W), fp.m, r, a.c, n, 1.f);
      gemm_ws(p, at<float>(ctx, fp.ws));
      gs.add(true, false, p, fp.ws_elems);
    }
    STAGE(run("gemm_proj"));
    // B: R = M - U P
    for (int i : brand) {
      const auto& a = args[i];
      const auto& fp = ctx->f[a.factor];
      const int n = fp.d.n, r = fp.d.r;
      GemmProb pr = gp(Uin(a), ldUin(a), at<float>(ctx, fp.W), fp.m, at<float>(ctx, fp.R), fp.nld, n, a.c,
                       r, -1.f, Min(a), ldMin(a), 1.f);
      pr.status = status_ptr(ctx, a.factor);   // every element of M passes this epilogue
      gs.add(false, false, pr, 0);
    }
    STAGE(run("gemm_resid"));
    // CGS2 re-projection: P2 = U^T R; R -= U P2; P += P2
    bool any_reorth = false;
    for (int i : brand) {
      const auto& a = args[i];
      if (a.flags & BKFAC_BRAND_NO_REORTH) continue;
      any_reorth = true;
      const auto& fp = ctx->f[a.factor];
      const int n = fp.d.n, r = fp.d.r;
      GemmProb p = gp(Uin(a), ldUin(a), at<float>(ctx, fp.R), fp.nld, at<float>(ctx, fp.P2), r, r, a.c, n, 1.f);
      gemm_ws(p, at<float>(ctx, fp.ws));
      gs.add(true, false, p, fp.ws_elems);
    }
    if (any_reorth) {
      STAGE(run("gemm_cgs2_proj"));
      for (int i : brand) {
        const auto& a = args[i];
        if (a.flags & BKFAC_BRAND_NO_REORTH) continue;
        const auto& fp = ctx->f[a.factor];
        const int n = fp.d.n, r = fp.d.r;
        float* R = at<float>(ctx, fp.R);
        gs.add(false, false, gp(Uin(a), ldUin(a), at<float>(ctx, fp.P2), r, R, fp.nld, n, a.c, r, -1.f, R, fp.nld, 1.f), 0);
        EwProb e{};
        e.Y = at<float>(ctx, fp.W); e.ldy = fp.m; e.X = at<float>(ctx, fp.P2); e.ldx = r;
        e.rows = r; e.cols = a.c; e.a = 1.f; e.op = EW_ADD;
        ew.push_back(e);
      }
      STAGE(run("gemm_cgs2_resid"));
      STAGE(run_ew(ctx, ew, st, "ew_cgs2"));
    }
    // CholeskyQR2 of R:  G = R^T R; L1; Q1 = R L1^{-T}; G = Q1^T Q1; L2; Q = Q1 L2^{-T}
    for (int pass = 0; pass < 2; ++pass) {
      for (int i : brand) {
        const auto& a = args[i];
        const auto& fp = ctx->f[a.factor];
        const int n = fp.d.n, c = a.c;
        const float* X = at<float>(ctx, pass == 0 ? fp.R : fp.Qb);
        GemmProb p = gp(X, fp.nld, X, fp.nld, at<float>(ctx, fp.G), c, c, c, n, 1.f);
        p.sym = 1;   // Gram: lower tiles computed, the upper mirrored
        gemm_ws(p, at<float>(ctx, fp.ws));
        gs.add(true, false, p, fp.ws_elems);
      }
      STAGE(run("gemm_gram"));
      for (int i : brand) {
        const auto& a = args[i];
        const auto& fp = ctx->f[a.factor];
        // pass 0 is shifted (shift = c u tr(G)): shifted CholeskyQR2 (see chol.cuh)
        ch.push_back(chol_prob(ctx, at<float>(ctx, fp.G), a.c, pass == 0 ? fp.L1 : fp.L2,
                               pass == 0 ? fp.L1i : fp.L2i, fp.cscr, status_ptr(ctx, a.factor),
                               pass == 0 ? (float)a.c * 1.1920929e-7f : 0.f));
      }
      STAGE(run_chol(ctx, ch, st));
      // pass 1's product Q = Q1 L2^{-T} is never formed: the rotation takes Q1 with the
      // eigenvector rows folded by L2^{-T} (gemm_qfold below), one c x c x r_out product
      // instead of n x c x c
      if (pass == 1) break;
      for (int i : brand) {
        const auto& a = args[i];
        const auto& fp = ctx->f[a.factor];
        const int n = fp.d.n, c = a.c;
        const float* X = at<float>(ctx, pass == 0 ? fp.R : fp.Qb);
        float* Y = at<float>(ctx, pass == 0 ? fp.Qb : fp.R);
        const float* Li = at<float>(ctx, pass == 0 ? fp.L1i : fp.L2i);
        gs.add(false, true, gp(X, fp.nld, Li, c, Y, fp.nld, n, c, c, 1.f), 0);
      }
      STAGE(run("gemm_qmul"));
    }
    // R_Q = L2^T L1^T -> W rows [r, r+c); then core K = beta W W^T (+ alpha D on the diagonal)
    for (int i : brand) {
      const auto& a = args[i];
      const auto& fp = ctx->f[a.factor];
      const int c = a.c, r = fp.d.r;
      gs.add(true, true, gp(at<float>(ctx, fp.L2), c, at<float>(ctx, fp.L1), c,
                            at<float>(ctx, fp.W) + r, fp.m, c, c, c, 1.f), 0);
    }
    STAGE(run("gemm_rq"));
    for (int i : brand) {
      const auto& a = args[i];
      const auto& fp = ctx->f[a.factor];
      const int mm = fp.d.r + a.c;
      const float* W = at<float>(ctx, fp.W);
      GemmProb pc = gp(W, fp.m, W, fp.m, at<float>(ctx, fp.eig.K), mm, mm, mm, a.c, a.beta);
      if (a.alpha != 0.f) {   // + diag(alpha D, 0) in the epilogue (Eq.(7) with rho D)
        pc.diag_vec = a.D_in; pc.diag_a = a.alpha; pc.diag_n = fp.d.r;
      }
      gs.add(false, true, pc, 0);
    }
    STAGE(run("gemm_core"));
    for (int i : brand) {
      const auto& a = args[i];
      const auto& fp = ctx->f[a.factor];
      const int mm = fp.d.r + a.c;
      eg.push_back(eig_prob(ctx, fp.eig, mm, rout_of(a), at<float>(ctx, fp.eig.V), mm, a.D_out,
                            status_ptr(ctx, a.factor)));
    }
  }
  STAGE(run_eig(ctx, eg, st));
  // fold: V_Q = L2^{-T} V[r:r+c, :]  (so that Q V[r:, :] = Q1 V_Q with Q = Q1 L2^{-T})
  for (int i : brand) {
    const auto& a = args[i];
    const auto& fp = ctx->f[a.factor];
    const int r = fp.d.r, c = a.c, mm = r + c, ro = rout_of(a);
    gs.add(true, false, gp(at<float>(ctx, fp.L2i), c, at<float>(ctx, fp.eig.V) + r, mm,
                           at<float>(ctx, fp.Vf), c, c, ro, c, 1.f), 0);
  }
  if (!brand.empty()) STAGE(run("gemm_qfold"));
  // rotation: U_out = [U Q] V = U V[0:r, :] + Q1 V_Q
  for (int i : brand) {
    const auto& a = args[i];
    const auto& fp = ctx->f[a.factor];
    const int n = fp.d.n, r = fp.d.r, mm = r + a.c, ro = rout_of(a);
    const float* V = at<float>(ctx, fp.eig.V);
    const bool us = useUs(a);
    const float* U0 = us ? at<float>(ctx, fp.Us) : a.U_in;
    GemmProb p = gp(U0, us ? fp.nld : ldU(a), V, mm, at<float>(ctx, fp.Urot), fp.nld, n, ro, mm, 1.f);
    p.A2 = at<float>(ctx, fp.Qb); p.lda2 = fp.nld;
    p.B2 = at<float>(ctx, fp.Vf); p.ldb2 = a.c;
    p.k1 = r;
    gs.add(false, false, p, 0);
  }
  STAGE(run("gemm_rotate"));
  // orthonormality refresh (reading R8): U_out = U' (3/2 I - 1/2 U'^T U'), one Newton-Schulz
  // step.  In exact arithmetic U' is orthonormal and this is the identity map; in fp32 it
  // removes the per-step departure (~1e-6..1e-5 from the GEMMs) instead of letting it
  // accumulate along the chain, at 4 n r^2 flops.
  for (int i = 0; i < count; ++i) {
    const auto& a = args[i];
    if (a.flags & BKFAC_BRAND_NO_REFRESH) continue;
    const auto& fp = ctx->f[a.factor];
    const int n = fp.d.n, r = rout_of(a);
    const float* Ur = at<float>(ctx, fp.Urot);
    GemmProb p = gp(Ur, fp.nld, Ur, fp.nld, at<float>(ctx, fp.Gref), r, r, r, n, 1.f);
    p.sym = 1;
    gemm_ws(p, at<float>(ctx, fp.wsr));
    gs.add(true, false, p, fp.wsr_elems);
  }
  STAGE(run("gemm_refresh_gram"));
  for (int i = 0; i < count; ++i) {
    const auto& a = args[i];
    const auto& fp = ctx->f[a.factor];
    const int n = fp.d.n, r = rout_of(a);
    const float* Ur = at<float>(ctx, fp.Urot);
    if (a.flags & BKFAC_BRAND_NO_REFRESH) {
      EwProb e{};
      e.Y = a.U_out; e.ldy = ldU(a); e.X = Ur; e.ldx = fp.nld; e.rows = n; e.cols = r; e.op = EW_COPY;
      ew.push_back(e);
      continue;
    }
    GemmProb pf = gp(Ur, fp.nld, at<float>(ctx, fp.Gref), r, a.U_out, ldU(a), n, r, r, -0.5f, Ur, fp.nld, 1.5f);
    pf.status = status_ptr(ctx, a.factor);   // the new basis passes this epilogue
    gs.add(false, false, pf, 0);
  }
  STAGE(run("gemm_refresh"));
  if (!ew.empty()) STAGE(run_ew(ctx, ew, st, "ew_copy_out"));
done:
#undef STAGE
  if (dev_prev != ctx->device) cudaSetDevice(dev_prev);
  return rs;
}

// ------------------------------------------------------------------------- dense EA
bkfac_status bkfac_ea_accumulate(bkfac_ctx ctx, int factor, float* K, const float* M, int c,
                                 float rho, void* stream) {
  if (!ctx || !K || !M) return BKFAC_ERR_INVALID_ARG;
  if (!ctx->ws) return BKFAC_ERR_WORKSPACE;
  if (factor < 0 || factor >= (int)ctx->f.size()) return BKFAC_ERR_INVALID_ARG;
  const auto& fp = ctx->f[factor];
  if (!(fp.d.flags & BKFAC_FACTOR_DENSE_EA)) return BKFAC_ERR_INVALID_ARG;
  if (c <= 0 || c > fp.d.c_max) return BKFAC_ERR_DIM;
  if (!(rho >= 0.f && rho < 1.f)) return BKFAC_ERR_INVALID_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int n = fp.d.n;
  GemmStage gs;
  GemmProb pe = gp(M, n, M, n, K, n, n, n, c, 1.f - rho, K, n, rho);
  pe.status = status_ptr(ctx, factor);
  pe.sym = 1;   // K and M M^T are symmetric: lower tiles computed, mirrored
  gs.add(false, true, pe, 0);
  return run_gemms(ctx, gs, st, "gemm_ea");
}

namespace {
// brand / nbrand: the same call's Brand updates (bkfac_brand_ea_update, EA beside the
// eigensolver): an EA item whose M is a Brand item's M reads the 16-byte-aligned copy the
// Brand update has already made of it (odd n), so the loaders take the vector path
bkfac_status ea_stage(bkfac_ctx ctx, const bkfac_ea_args* args, int count, GemmStage& gs,
                      const bkfac_brand_args* brand = nullptr, int nbrand = 0) {
  for (int i = 0; i < count; ++i) {
    const auto& a = args[i];
    if (a.factor < 0 || a.factor >= (int)ctx->f.size() || !a.K_dense || !a.M)
      return BKFAC_ERR_INVALID_ARG;
    const auto& fp = ctx->f[a.factor];
    if (!(fp.d.flags & BKFAC_FACTOR_DENSE_EA)) return BKFAC_ERR_INVALID_ARG;
    if (a.c <= 0 || a.c > fp.d.c_max) return BKFAC_ERR_DIM;
    if (!(a.rho >= 0.f && a.rho < 1.f)) return BKFAC_ERR_INVALID_ARG;
    const int n = fp.d.n;
    if (!ld_ok(a.ld_M, n)) return BKFAC_ERR_DIM;
    const float* Mp = a.M;
    int ldm = ldx(a.ld_M, n);
    for (int j = 0; j < nbrand; ++j)
      if (brand[j].factor == a.factor && brand[j].M == a.M && brand[j].c == a.c && fp.Ms &&
          !fp.dense && ldx(brand[j].ld_M, n) == ldm && !al16(a.M, ldm)) {
        Mp = at<float>(ctx, fp.Ms);
        ldm = fp.nld;
      }
    GemmProb pe = gp(Mp, ldm, Mp, ldm, a.K_dense, n, n, n, a.c, 1.f - a.rho, a.K_dense, n, a.rho);
    pe.status = status_ptr(ctx, a.factor);
    pe.sym = 1;   // K and M M^T are symmetric: lower tiles computed, mirrored
    gs.add(false, true, pe, 0);
  }
  return BKFAC_OK;
}
}  // namespace

bkfac_status bkfac_ea_accumulate_batch(bkfac_ctx ctx, const bkfac_ea_args* args, int count,
                                       void* stream) {
  if (!ctx || count < 0 || (count > 0 && !args)) return BKFAC_ERR_INVALID_ARG;
  if (!ctx->ws) return BKFAC_ERR_WORKSPACE;
  GemmStage gs;
  const bkfac_status r = ea_stage(ctx, args, count, gs);
  if (r != BKFAC_OK || count == 0) return r;
  return run_gemms(ctx, gs, static_cast<cudaStream_t>(stream), "gemm_ea");
}

bkfac_status bkfac_brand_ea_update(bkfac_ctx ctx, const bkfac_brand_args* args, int count,
                                   const bkfac_ea_args* ea_args, int ea_count, void* stream) {
  if (!ctx || ea_count < 0 || (ea_count > 0 && !ea_args)) return BKFAC_ERR_INVALID_ARG;
  if (!ctx->ws) return BKFAC_ERR_WORKSPACE;
  for (int i = 0; i < ea_count; ++i)
    for (int j = 0; j < count && args; ++j)
      if (ea_args[i].K_dense == args[j].U_out || ea_args[i].K_dense == args[j].U_in)
        return BKFAC_ERR_ALIAS;
  // 0 (default): EA GEMM on a side stream beside the tridiagonalisation, grid capped at the
  // SMs its clusters leave idle; 2: the same, uncapped; 1: EA first, serially, full grid
  const int ea_mode = ctx->ea_mode;
  GemmStage gs;
  // beside the eigensolver the Brand update's aligned copies of M already exist
  bkfac_status r = ea_mode == 1 ? ea_stage(ctx, ea_args, ea_count, gs)
                                : ea_stage(ctx, ea_args, ea_count, gs, args, args ? count : 0);
  if (r != BKFAC_OK) return r;
  if (ea_count == 0) return bkfac_brand_update(ctx, args, count, stream);
  if (ea_mode == 1) {
    r = run_gemms(ctx, gs, static_cast<cudaStream_t>(stream), "gemm_ea");
    return r != BKFAC_OK ? r : bkfac_brand_update(ctx, args, count, stream);
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev_prev = 0;
  cudaGetDevice(&dev_prev);
  if (dev_prev != ctx->device) cudaSetDevice(ctx->device);
  bool launched = false;
  ctx->pending_ea = [&](int busy) -> bkfac_status {
    if (!cuda_ok(cudaStreamWaitEvent(ctx->ea_stream, ctx->ev_ea_fork, 0)))   // recorded by run_eig
      return BKFAC_ERR_CUDA;
    const int ea_cap = ctx->ea_cap;
    ctx->grid_cap = ea_mode == 2 ? 0 : (ea_mode == 3 || ea_mode == 4) ? -1
                  : (ea_cap > 0 ? ea_cap : std::max(kNumSM / 8, kNumSM - busy));
    ctx->ea_join_early = ea_mode == 4;
    const bkfac_status re = run_gemms(ctx, gs, ctx->ea_stream, "gemm_ea");
    ctx->grid_cap = 0;
    if (re != BKFAC_OK) return re;
    if (!cuda_ok(cudaEventRecord(ctx->ev_ea_done, ctx->ea_stream))) return BKFAC_ERR_CUDA;
    launched = true;
    return BKFAC_OK;
  };
  r = bkfac_brand_update(ctx, args, count, stream);
  ctx->pending_ea = nullptr;
  ctx->grid_cap = 0;
  ctx->ea_join_early = false;
  if (r == BKFAC_OK) {
    if (launched) {
      if (!cuda_ok(cudaStreamWaitEvent(st, ctx->ev_ea_done, 0))) r = BKFAC_ERR_CUDA;
    } else {
      r = run_gemms(ctx, gs, st, "gemm_ea");   // no eigensolver ran (count == 0)
    }
  }
  if (dev_prev != ctx->device) cudaSetDevice(dev_prev);
  return r;
}

// ------------------------------------------------------------------------- light correction
// Algorithm 6 on the RSVD scratch of the factor (the two never run in the same call):
// Yr <- U_c (gather), Qr <- K U_c, eig_r.K <- U_c^T K U_c (split-K), EVD (eig_r, all n_crc pairs,
// vectors into Br, values into Tr), Q2r <- U_c V, scatter into U and D.
bkfac_status bkfac_light_correction(bkfac_ctx ctx, const bkfac_correct_args* args, int count,
                                    void* stream) {
  if (!ctx || count < 0 || (count > 0 && !args)) return BKFAC_ERR_INVALID_ARG;
  if (!ctx->ws) return BKFAC_ERR_WORKSPACE;
  for (int i = 0; i < count; ++i) {
    const auto& a = args[i];
    if (a.factor < 0 || a.factor >= (int)ctx->f.size()) return BKFAC_ERR_INVALID_ARG;
    const auto& fp = ctx->f[a.factor];
    if (!fp.rsvd) return BKFAC_ERR_INVALID_ARG;
    if (!a.K_dense || !a.U || !a.D || !a.col_idx) return BKFAC_ERR_INVALID_ARG;
    if (a.n_crc < 1 || a.n_crc > fp.d.r) return BKFAC_ERR_DIM;
    if (!ld_ok(a.ld_U, fp.d.n)) return BKFAC_ERR_DIM;
    for (int j = 0; j < i; ++j)
      if (args[j].factor == a.factor) return BKFAC_ERR_INVALID_ARG;
  }
  if (count == 0) return BKFAC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev_prev = 0;
  cudaGetDevice(&dev_prev);
  if (dev_prev != ctx->device) cudaSetDevice(ctx->device);
  bkfac_status rs = BKFAC_OK;
  GemmStage gs;
  std::vector<EigProb> eg;
  static thread_local ColIdxBatch cb;
  auto colidx = [&](int mode, const char* tag) -> bkfac_status {
    prof_begin(ctx, tag, st, 0.0, 0.0);
    for (int i0 = 0; i0 < count; i0 += NF_MAXP) {
      const int nb = std::min(count - i0, NF_MAXP);
      cb.nprob = nb;
      for (int k = 0; k < nb; ++k) {
        const auto& a = args[i0 + k];
        const auto& fp = ctx->f[a.factor];
        const int n = fp.d.n;
        ColIdxProb q{};
        q.rows = n; q.idx = a.col_idx; q.n = a.n_crc; q.r = fp.d.r; q.mode = mode;
        q.status = status_ptr(ctx, a.factor);
        if (mode == 0) { q.src = a.U; q.lds = ldx(a.ld_U, n); q.dst = at<float>(ctx, fp.Yr); q.ldd = n; }
        else {
          q.src = at<float>(ctx, fp.Q2r); q.lds = n; q.dst = a.U; q.ldd = ldx(a.ld_U, n);
          q.dsrc = at<float>(ctx, fp.Tr); q.ddst = a.D;
        }
        cb.p[k] = q;
      }
      colidx_kernel<<<dim3(64, (unsigned)nb), 256, 0, st>>>(cb);
      LAUNCH_CHECK(ctx);
    }
    prof_end(ctx, st);
    return BKFAC_OK;
  };
#define STAGE(x) do { if ((rs = (x)) != BKFAC_OK) goto done; } while (0)
  STAGE(colidx(0, "crc_gather"));
  for (int i = 0; i < count; ++i) {   // Y = K U_c
    const auto& a = args[i];
    const auto& fp = ctx->f[a.factor];
    const int n = fp.d.n;
    GemmProb p = gp(a.K_dense, n, at<float>(ctx, fp.Yr), n, at<float>(ctx, fp.Qr), n, n, a.n_crc, n, 1.f);
    p.status = status_ptr(ctx, a.factor);
    gs.add(false, false, p, 0);
  }
  STAGE(run_gemms(ctx, gs, st, "gemm_crc_mul"));
  for (int i = 0; i < count; ++i) {   // M_S = U_c^T Y
    const auto& a = args[i];
    const auto& fp = ctx->f[a.factor];
    const int n = fp.d.n;
    GemmProb p = gp(at<float>(ctx, fp.Yr), n, at<float>(ctx, fp.Qr), n, at<float>(ctx, fp.eig_r.K),
                    a.n_crc, a.n_crc, a.n_crc, n, 1.f);   // straight into the eigensolver's input
    gemm_ws(p, at<float>(ctx, fp.ws_r));
    gs.add(true, false, p, fp.ws_r_elems);
  }
  STAGE(run_gemms(ctx, gs, st, "gemm_crc_proj"));
  for (int i = 0; i < count; ++i) {   // EVD(M_S): all n_crc pairs (vectors into Br, values into Tr)
    const auto& a = args[i];
    const auto& fp = ctx->f[a.factor];
    eg.push_back(eig_prob(ctx, fp.eig_r, a.n_crc, a.n_crc, at<float>(ctx, fp.Br), a.n_crc,
                          at<float>(ctx, fp.Tr), status_ptr(ctx, a.factor)));
  }
  STAGE(run_eig(ctx, eg, st));
  for (int i = 0; i < count; ++i) {   // U_c V
    const auto& a = args[i];
    const auto& fp = ctx->f[a.factor];
    const int n = fp.d.n;
    gs.add(false, false, gp(at<float>(ctx, fp.Yr), n, at<float>(ctx, fp.Br), a.n_crc,
                            at<float>(ctx, fp.Q2r), n, n, a.n_crc, a.n_crc, 1.f), 0);
  }
  STAGE(run_gemms(ctx, gs, st, "gemm_crc_rot"));
  STAGE(colidx(1, "crc_scatter"));
done:
#undef STAGE
  if (dev_prev != ctx->device) cudaSetDevice(dev_prev);
  return rs;
}

// ------------------------------------------------------------------------- RSVD
bkfac_status bkfac_rsvd_overwrite_batch(bkfac_ctx ctx, const bkfac_rsvd_args* args, int count,
                                        void* stream) {
  if (!ctx || count < 0 || (count > 0 && !args)) return BKFAC_ERR_INVALID_ARG;
  if (!ctx->ws) return BKFAC_ERR_WORKSPACE;
  int qmax = 0;
  for (int i = 0; i < count; ++i) {
    const auto& a = args[i];
    if (!a.K_dense || !a.U_out || !a.D_out) return BKFAC_ERR_INVALID_ARG;
    if (a.factor >= 0 && a.factor < (int)ctx->f.size() && !ld_ok(a.ld_U, ctx->f[a.factor].d.n))
      return BKFAC_ERR_DIM;
    if (a.factor < 0 || a.factor >= (int)ctx->f.size()) return BKFAC_ERR_INVALID_ARG;
    const auto& fp = ctx->f[a.factor];
    if (!fp.rsvd) return BKFAC_ERR_INVALID_ARG;
    if (a.oversample < 0 || a.power_iters < 0 || a.power_iters > 64) return BKFAC_ERR_INVALID_ARG;
    const int l = fp.d.r + a.oversample;
    if (l > fp.d.n) return BKFAC_ERR_RANK;
    if (l > fp.lmax) return BKFAC_ERR_UNSUPPORTED;
    for (int j = 0; j < i; ++j)
      if (args[j].factor == a.factor) return BKFAC_ERR_INVALID_ARG;
    qmax = std::max(qmax, a.power_iters);
  }
  if (count == 0) return BKFAC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  GemmStage gs;
  std::vector<CholProb> ch;
  std::vector<EigProb> eg;
  std::vector<EwProb> ew;
  bkfac_status rs;
  struct Loc { int n, r, l; int* status; float *Y, *Q, *Q2, *T, *ws; const FactorPlan* fp; };
  std::vector<Loc> L(count);
  // sketch width l = n: the range is all of R^n, Q = I and the RSVD is the exact EVD of
  // K (Alg 5 with nothing to sketch); those factors skip the range finder entirely.
  std::vector<int> rf, exact;
  for (int i = 0; i < count; ++i) {
    const auto& fp = ctx->f[args[i].factor];
    L[i] = Loc{fp.d.n, fp.d.r, fp.d.r + args[i].oversample, status_ptr(ctx, args[i].factor),
               at<float>(ctx, fp.Yr), at<float>(ctx, fp.Qr), at<float>(ctx, fp.Q2r),
               at<float>(ctx, fp.Tr), at<float>(ctx, fp.ws_r), &fp};
    (L[i].l == L[i].n ? exact : rf).push_back(i);
  }
  // Omega -> Q (Philox sketch); Y = K Omega
  {
    double bytes = 0.0;
    for (int i : rf) bytes += 4.0 * L[i].n * (double)L[i].l;
    prof_begin(ctx, "rsvd_sketch", st, 0.0, bytes);
    for (int i : rf) {
      philox_sketch_kernel<<<256, 256, 0, st>>>(L[i].Q, (long)L[i].n * L[i].l, args[i].seed,
                                               args[i].counter);
      LAUNCH_CHECK(ctx);
    }
    prof_end(ctx, st);
  }
  for (int i : rf) {
    GemmProb pk = gp(args[i].K_dense, L[i].n, L[i].Q, L[i].n, L[i].Y, L[i].n, L[i].n, L[i].l,
                     L[i].n, 1.f);
    gs.add(false, false, pk, 0);
  }
  if ((rs = run_gemms(ctx, gs, st, "gemm_rsvd_mul")) != BKFAC_OK) return rs;
  // shifted CholeskyQR3 of X (the power-iteration block K Q is ill-conditioned by
  // design): X -> Qout (shifted) -> Q2 -> Qout, for the factors in `act`
  auto orth = [&](const std::vector<int>& act, bool fromY) -> bkfac_status {
    for (int pass = 0; pass < 3; ++pass) {
      for (int i : act) {
        const float* In = pass == 0 ? (fromY ? L[i].Y : L[i].Q) : (pass == 1 ? L[i].Q : L[i].Q2);
        GemmProb p = gp(In, L[i].n, In, L[i].n, at<float>(ctx, L[i].fp->Gr), L[i].l, L[i].l, L[i].l,
                        L[i].n, 1.f);
        gemm_ws(p, L[i].ws);
        gs.add(true, false, p, L[i].fp->ws_r_elems);
      }
      bkfac_status s2 = run_gemms(ctx, gs, st, "gemm_rsvd_gram");
      if (s2 != BKFAC_OK) return s2;
      for (int i : act)
        ch.push_back(chol_prob(ctx, at<float>(ctx, L[i].fp->Gr), L[i].l, L[i].fp->L1r, L[i].fp->L1ir,
                               L[i].fp->cscr_r, L[i].status,
                               pass == 0 ? (float)L[i].l * 1.1920929e-7f : 0.f));
      if ((s2 = run_chol(ctx, ch, st)) != BKFAC_OK) return s2;
      for (int i : act) {
        const float* In = pass == 0 ? (fromY ? L[i].Y : L[i].Q) : (pass == 1 ? L[i].Q : L[i].Q2);
        float* Out = pass == 1 ? L[i].Q2 : L[i].Q;
        gs.add(false, true, gp(In, L[i].n, at<float>(ctx, L[i].fp->L1ir), L[i].l, Out, L[i].n, L[i].n,
                               L[i].l, L[i].l, 1.f), 0);
      }
      if ((s2 = run_gemms(ctx, gs, st, "gemm_rsvd_qmul")) != BKFAC_OK) return s2;
    }
    return BKFAC_OK;
  };
  // note: pass 0 reads Y and writes Q, so X and Qout never alias
  for (int q = 0; q < qmax; ++q) {
    std::vector<int> act;
    for (int i : rf)
      if (q < args[i].power_iters) act.push_back(i);
    if (act.empty()) continue;
    if ((rs = orth(act, true)) != BKFAC_OK) return rs;
    for (int i : act)
      gs.add(false, false, gp(args[i].K_dense, L[i].n, L[i].Q, L[i].n, L[i].Y, L[i].n, L[i].n,
                              L[i].l, L[i].n, 1.f), 0);
    if ((rs = run_gemms(ctx, gs, st, "gemm_rsvd_mul")) != BKFAC_OK) return rs;
  }
  if (!rf.empty() && (rs = orth(rf, true)) != BKFAC_OK) return rs;
  // B = Q^T K Q ; EVD(B) ; U = Q V_r
  for (int i : rf)
    gs.add(false, false, gp(args[i].K_dense, L[i].n, L[i].Q, L[i].n, L[i].T, L[i].n, L[i].n, L[i].l,
                            L[i].n, 1.f), 0);
  if ((rs = run_gemms(ctx, gs, st, "gemm_rsvd_mul")) != BKFAC_OK) return rs;
  for (int i : rf) {
    GemmProb p = gp(L[i].Q, L[i].n, L[i].T, L[i].n, at<float>(ctx, L[i].fp->eig_r.K), L[i].l, L[i].l,
                    L[i].l, L[i].n, 1.f);
    gemm_ws(p, L[i].ws);
    gs.add(true, false, p, L[i].fp->ws_r_elems);
  }
  if ((rs = run_gemms(ctx, gs, st, "gemm_rsvd_proj")) != BKFAC_OK) return rs;
  for (int i : exact) {   // B = K itself
    EwProb e{};
    e.Y = at<float>(ctx, L[i].fp->eig_r.K); e.ldy = L[i].n; e.X = args[i].K_dense; e.ldx = L[i].n;
    e.rows = L[i].n; e.cols = L[i].n; e.op = EW_COPY;
    ew.push_back(e);
  }
  if (!ew.empty() && (rs = run_ew(ctx, ew, st, "ew_rsvd_exact")) != BKFAC_OK) return rs;
  for (int i = 0; i < count; ++i) {
    const bool ex = L[i].l == L[i].n;
    eg.push_back(eig_prob(ctx, L[i].fp->eig_r, L[i].l, L[i].r,
                          ex ? args[i].U_out : at<float>(ctx, L[i].fp->eig_r.V),
                          ex ? ldx(args[i].ld_U, L[i].n) : L[i].l, args[i].D_out, L[i].status));
  }
  if ((rs = run_eig(ctx, eg, st)) != BKFAC_OK) return rs;
  for (int i : rf)
    gs.add(false, false, gp(L[i].Q, L[i].n, at<float>(ctx, L[i].fp->eig_r.V), L[i].l, args[i].U_out,
                            ldx(args[i].ld_U, L[i].n), L[i].n, L[i].r, L[i].l, 1.f), 0);
  return run_gemms(ctx, gs, st, "gemm_rsvd_rot");
}

bkfac_status bkfac_rsvd_overwrite(bkfac_ctx ctx, int factor, const float* K, int oversample,
                                  int power_iters, uint64_t seed, uint64_t counter, float* U_out,
                                  float* D_out, void* stream) {
  bkfac_rsvd_args a{factor, K, oversample, power_iters, seed, counter, U_out, D_out};
  return bkfac_rsvd_overwrite_batch(ctx, &a, 1, stream);
}

bkfac_status bkfac_gaussian_sketch(float* Om, int n, int l, uint64_t seed, uint64_t counter,
                                   void* stream) {
  if (!Om || n <= 0 || l <= 0) return BKFAC_ERR_INVALID_ARG;
  philox_sketch_kernel<<<1024, 256, 0, static_cast<cudaStream_t>(stream)>>>(Om, (long)n * l, seed,
                                                                            counter);
  if (!cuda_ok(cudaGetLastError())) return BKFAC_ERR_CUDA;
  return BKFAC_OK;
}

// ------------------------------------------------------------------------- precondition
#ifndef BKFAC_PREC_PROJ_PROMO
// K chunks per TMEM accumulation block of Y = J U_A, Xt = J^T U_G.  The same 256-term blocks
// as the output GEMM and every other contraction: the accumulate biases of the projections
// and of the output product partly cancel inside span(U_G) x span(U_A), and 256 / 256 measured
// best of 18 combinations (relative error of U_G^T S U_A at lambda = 0.01: 3.0e-4; 1.0e-3 with
// 512-term projections, 0.85e-3 with 32-term output blocks; tools/prec_block_error.py).
// 16 (512-term blocks) is 1.6 ms faster on gemm_prec_proj and nothing on the power-capped step.
#define BKFAC_PREC_PROJ_PROMO TC_PROMO
#endif
bkfac_status bkfac_precondition(bkfac_ctx ctx, const bkfac_precond_args* args, int count,
                                void* stream) {
  if (!ctx || (count > 0 && !args) || count < 0) return BKFAC_ERR_INVALID_ARG;
  if (!ctx->ws) return BKFAC_ERR_WORKSPACE;
  for (int i = 0; i < count; ++i) {
    const auto& a = args[i];
    if (a.layer < 0 || a.layer >= (int)ctx->l.size()) return BKFAC_ERR_INVALID_ARG;
    const auto& d = ctx->l[a.layer].d;
    if (!a.J || !a.S) return BKFAC_ERR_INVALID_ARG;
    if ((d.r_A > 0 && (!a.U_A || !a.D_A)) || (d.r_G > 0 && (!a.U_G || !a.D_G)))
      return BKFAC_ERR_INVALID_ARG;
    if (!(a.lambda_A > 0.f) || !(a.lambda_G > 0.f)) return BKFAC_ERR_INVALID_ARG;
    if (a.S == a.J) return BKFAC_ERR_ALIAS;
    if (!ld_ok(a.ld_UG, d.d_G) || !ld_ok(a.ld_UA, d.d_A) || !ld_ok(a.ld_J, d.d_A) ||
        !ld_ok(a.ld_S, d.d_A))
      return BKFAC_ERR_DIM;
    for (int j = 0; j < i; ++j)
      if (args[j].layer == a.layer) return BKFAC_ERR_INVALID_ARG;
  }
  if (count == 0) return BKFAC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  static thread_local PrecScalBatch psb;
  bkfac_status rs;
  GemmStage gs;
  // S1: scalars
  prof_begin(ctx, "prec_scalars", st, 0.0, 0.0);
  for (int i0 = 0; i0 < count; i0 += PS_MAXP) {
    const int n = std::min(count - i0, PS_MAXP);
    psb.nprob = 0;
    for (int i = i0; i < i0 + n; ++i) {
      const auto& a = args[i];
      const auto& lp = ctx->l[a.layer];
      PrecScalProb q{};
      q.D[0] = a.D_A; q.r[0] = lp.d.r_A; q.lam[0] = a.lambda_A; q.s[0] = at<float>(ctx, lp.sA);
      q.D[1] = a.D_G; q.r[1] = lp.d.r_G; q.lam[1] = a.lambda_G; q.s[1] = at<float>(ctx, lp.sG);
      q.flags = a.flags;
      q.lam_out = at<float>(ctx, lp.lam);   // {lambda_A, lambda_G, 1 / (lambda_G lambda_A)}
      psb.p[psb.nprob++] = q;
    }
    prec_scalars_kernel<<<psb.nprob, 256, 0, st>>>(psb);
    LAUNCH_CHECK(ctx);
  }
  prof_end(ctx, st);
  // S2: Y = J U_A (d_G x r_A), Xt = J^T U_G (d_A x r_G)
  for (int i = 0; i < count; ++i) {
    const auto& a = args[i];
    const auto& lp = ctx->l[a.layer];
    const int dG = lp.d.d_G, dA = lp.d.d_A, rA = lp.d.r_A, rG = lp.d.r_G;
    float* lam = at<float>(ctx, lp.lam);   // {lamA, lamG, 1/(lamG lamA), 1/lamA, 1/lamG}
    if (rA > 0) {   // Y' = (J U_A) diag(sA) / lamG  (scaling in the epilogue)
      GemmProb p = gp(a.J, ldx(a.ld_J, dA), a.U_A, ldx(a.ld_UA, dA), at<float>(ctx, lp.Y), lp.ldY, dG, rA, dA, 1.f);
      p.col_scale = at<float>(ctx, lp.sA); p.alpha_dev = lam + 4;
      p.promo = BKFAC_PREC_PROJ_PROMO;
      gemm_ws(p, at<float>(ctx, lp.ws));
      gs.add(true, false, p, lp.ws_elems);
    }
    if (rG > 0) {   // Xt' = (J^T U_G) diag(sG) / lamA
      GemmProb p = gp(a.J, ldx(a.ld_J, dA), a.U_G, ldx(a.ld_UG, dG), at<float>(ctx, lp.Xt), lp.ldXt, dA, rG, dG, 1.f);
      p.col_scale = at<float>(ctx, lp.sG); p.alpha_dev = lam + 3;
      p.promo = BKFAC_PREC_PROJ_PROMO;
      gs.add(false, false, p, 0);
    }
  }
  if ((rs = run_gemms(ctx, gs, st, "gemm_prec_proj")) != BKFAC_OK) return rs;
  // S3: Z' = diag(sG) U_G^T (Y diag(sA)) = lamG diag(sG) (U_G^T Y')  (r_G x r_A)
  for (int i = 0; i < count; ++i) {
    const auto& a = args[i];
    const auto& lp = ctx->l[a.layer];
    const int dG = lp.d.d_G, rA = lp.d.r_A, rG = lp.d.r_G;
    if (rA > 0 && rG > 0) {
      GemmProb p = gp(a.U_G, ldx(a.ld_UG, dG), at<float>(ctx, lp.Y), lp.ldY, at<float>(ctx, lp.Z), rG, rG, rA, dG, 1.f);
      p.row_scale = at<float>(ctx, lp.sG); p.alpha_dev = at<float>(ctx, lp.lam) + 1;
      gs.add(true, false, p, 0);
    }
  }
  if ((rs = run_gemms(ctx, gs, st, "gemm_prec_z")) != BKFAC_OK) return rs;
  // S5: Y' += U_G Z'
  for (int i = 0; i < count; ++i) {
    const auto& a = args[i];
    const auto& lp = ctx->l[a.layer];
    const int dG = lp.d.d_G, rA = lp.d.r_A, rG = lp.d.r_G;
    if (rA > 0 && rG > 0) {
      float* Y = at<float>(ctx, lp.Y);
      gs.add(false, false, gp(a.U_G, ldx(a.ld_UG, dG), at<float>(ctx, lp.Z), rG, Y, lp.ldY, dG, rA, rG, 1.f,
                              Y, lp.ldY, 1.f), 0);
    }
  }
  if ((rs = run_gemms(ctx, gs, st, "gemm_prec_small")) != BKFAC_OK) return rs;
  // S7: S^T (d_A x d_G) = [U_A | Xt'] [Y'^T ; U_G^T] + coef J^T
  for (int i = 0; i < count; ++i) {
    const auto& a = args[i];
    const auto& lp = ctx->l[a.layer];
    const int dG = lp.d.d_G, dA = lp.d.d_A, rA = lp.d.r_A, rG = lp.d.r_G;
    float* lam = at<float>(ctx, lp.lam);
    const int ldUA = ldx(a.ld_UA, dA), ldUG = ldx(a.ld_UG, dG);
    GemmProb p = gp(rA > 0 ? a.U_A : at<float>(ctx, lp.Xt), rA > 0 ? ldUA : lp.ldXt,
                    rA > 0 ? at<float>(ctx, lp.Y) : a.U_G, rA > 0 ? lp.ldY : ldUG, a.S,
                    ldx(a.ld_S, dA), dA, dG, rA + rG, 1.f, a.J, ldx(a.ld_J, dA), 1.f);
    p.A2 = at<float>(ctx, lp.Xt); p.lda2 = lp.ldXt;
    p.B2 = a.U_G ? a.U_G : at<float>(ctx, lp.Y); p.ldb2 = a.U_G ? ldUG : lp.ldY;
    p.k1 = rA;
    p.beta_dev = lam + 2;
    p.stream_c = 1;   // J read and S written once: evict-first, the operands stay in L2
    // BKFAC_OPT_PREC_BLOCK > 0: that many 32-term chunks per TMEM accumulation block (>= K / 32:
    // the whole K in one block, no promotion passes, the tile's output overlaps the next tile's
    // whole mainloop: 43.65 -> 40.8 ms at configs[4]).  Not the default: the low-rank term
    // cancels most of J / (lam lam) inside span(U_G) x span(U_A), and the longer block's
    // accumulate bias shows there (relative error of U_G^T S U_A 3.0e-4 -> 1.2e-3 at lam = 0.01,
    // tests/test_gpu_parity.py::test_precondition_output_block_length).
    p.promo = ctx->prec_block;
    p.status = status_ptr(ctx, (int)ctx->f.size() + a.layer);   // every element of J passes here
    gs.add(false, true, p, 0);
  }
  return run_gemms(ctx, gs, st, "gemm_prec_out");
}

bkfac_status bkfac_precondition_factored(bkfac_ctx ctx, const bkfac_precond_factored_args* args,
                                         int count, void* stream) {
  if (!ctx || (count > 0 && !args) || count < 0) return BKFAC_ERR_INVALID_ARG;
  if (!ctx->ws) return BKFAC_ERR_WORKSPACE;
  for (int i = 0; i < count; ++i) {
    const auto& a = args[i];
    if (a.layer < 0 || a.layer >= (int)ctx->l.size()) return BKFAC_ERR_INVALID_ARG;
    const auto& d = ctx->l[a.layer].d;
    if (!a.G || !a.A || !a.S) return BKFAC_ERR_INVALID_ARG;
    if ((d.r_A > 0 && (!a.U_A || !a.D_A)) || (d.r_G > 0 && (!a.U_G || !a.D_G)))
      return BKFAC_ERR_INVALID_ARG;
    if (!(a.lambda_A > 0.f) || !(a.lambda_G > 0.f)) return BKFAC_ERR_INVALID_ARG;
    if (a.n <= 0 || a.n > d.n_max) return BKFAC_ERR_DIM;
    if (a.S == a.G || a.S == a.A) return BKFAC_ERR_ALIAS;
    if (!ld_ok(a.ld_UG, d.d_G) || !ld_ok(a.ld_UA, d.d_A) || !ld_ok(a.ld_G, d.d_G) ||
        !ld_ok(a.ld_A, d.d_A) || !ld_ok(a.ld_S, d.d_A))
      return BKFAC_ERR_DIM;
    for (int j = 0; j < i; ++j)
      if (args[j].layer == a.layer) return BKFAC_ERR_INVALID_ARG;
  }
  if (count == 0) return BKFAC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  static thread_local PrecScalBatch psb;
  bkfac_status rs;
  GemmStage gs;
  // scalars (s_A, s_G, lambdas, 1/lambdas) as bkfac_precondition
  prof_begin(ctx, "prec_scalars", st, 0.0, 0.0);
  for (int i0 = 0; i0 < count; i0 += PS_MAXP) {
    const int n = std::min(count - i0, PS_MAXP);
    psb.nprob = 0;
    for (int i = i0; i < i0 + n; ++i) {
      const auto& a = args[i];
      const auto& lp = ctx->l[a.layer];
      PrecScalProb q{};
      q.D[0] = a.D_A; q.r[0] = lp.d.r_A; q.lam[0] = a.lambda_A; q.s[0] = at<float>(ctx, lp.sA);
      q.D[1] = a.D_G; q.r[1] = lp.d.r_G; q.lam[1] = a.lambda_G; q.s[1] = at<float>(ctx, lp.sG);
      q.flags = a.flags;
      q.lam_out = at<float>(ctx, lp.lam);
      psb.p[psb.nprob++] = q;
    }
    prec_scalars_kernel<<<psb.nprob, 256, 0, st>>>(psb);
    LAUNCH_CHECK(ctx);
  }
  prof_end(ctx, st);
  // P_G = G^T U_G (n x r_G), P_A = A^T U_A (n x r_A): long K (d), small output -> split-K
  for (int i = 0; i < count; ++i) {
    const auto& a = args[i];
    const auto& lp = ctx->l[a.layer];
    const int dG = lp.d.d_G, dA = lp.d.d_A, rA = lp.d.r_A, rG = lp.d.r_G, n = a.n;
    if (rG > 0) {   // P_G diag(s_G), the scaling in the epilogue
      GemmProb p = gp(a.G, ldx(a.ld_G, dG), a.U_G, ldx(a.ld_UG, dG), at<float>(ctx, lp.fPG), n, n, rG, dG, 1.f);
      p.col_scale = at<float>(ctx, lp.sG);
      gemm_ws(p, at<float>(ctx, lp.fws));
      gs.add(true, false, p, lp.fws_elems);
    }
    if (rA > 0) {
      GemmProb p = gp(a.A, ldx(a.ld_A, dA), a.U_A, ldx(a.ld_UA, dA), at<float>(ctx, lp.fPA), n, n, rA, dA, 1.f);
      p.col_scale = at<float>(ctx, lp.sA);
      gemm_ws(p, at<float>(ctx, lp.fws2));
      gs.add(true, false, p, lp.fws_elems);
    }
  }
  if ((rs = run_gemms(ctx, gs, st, "gemm_f2_proj")) != BKFAC_OK) return rs;
  // G_b = U_G P_G^T + G / lambda_G, A_b = U_A P_A^T + A / lambda_A (device-scalar beta)
  for (int i = 0; i < count; ++i) {
    const auto& a = args[i];
    const auto& lp = ctx->l[a.layer];
    const int dG = lp.d.d_G, dA = lp.d.d_A, rA = lp.d.r_A, rG = lp.d.r_G, n = a.n;
    float* lam = at<float>(ctx, lp.lam);
    GemmProb pg = gp(rG > 0 ? a.U_G : a.G, rG > 0 ? ldx(a.ld_UG, dG) : ldx(a.ld_G, dG), at<float>(ctx, lp.fPG), n,
                     at<float>(ctx, lp.fGb), dG, dG, n, rG, 1.f, a.G, ldx(a.ld_G, dG), 1.f);
    pg.beta_dev = lam + 4;
    pg.status = status_ptr(ctx, (int)ctx->f.size() + a.layer);   // every element of G passes here
    gs.add(false, true, pg, 0);
    GemmProb pa = gp(rA > 0 ? a.U_A : a.A, rA > 0 ? ldx(a.ld_UA, dA) : ldx(a.ld_A, dA), at<float>(ctx, lp.fPA), n,
                     at<float>(ctx, lp.fAb), dA, dA, n, rA, 1.f, a.A, ldx(a.ld_A, dA), 1.f);
    pa.beta_dev = lam + 3;
    pa.status = status_ptr(ctx, (int)ctx->f.size() + a.layer);
    gs.add(false, true, pa, 0);
  }
  if ((rs = run_gemms(ctx, gs, st, "gemm_f2_apply")) != BKFAC_OK) return rs;
  // S^T (d_A x d_G) = A_b G_b^T
  for (int i = 0; i < count; ++i) {
    const auto& a = args[i];
    const auto& lp = ctx->l[a.layer];
    const int dG = lp.d.d_G, dA = lp.d.d_A, n = a.n;
    gs.add(false, true, gp(at<float>(ctx, lp.fAb), dA, at<float>(ctx, lp.fGb), dG, a.S, ldx(a.ld_S, dA), dA, dG,
                           n, 1.f), 0);
  }
  return run_gemms(ctx, gs, st, "gemm_f2_out");
}

// ------------------------------------------------------------------------- GEMM primitive
bkfac_status bkfac_gemm(int transA, int transB, int M, int N, int K, float alpha, const float* A,
                        int lda, const float* B, int ldb, float beta, float* C, int ldc, float* ws,
                        size_t ws_bytes, int path, void* stream) {
  if (M < 0 || N < 0 || K < 0 || !C || (K > 0 && (!A || !B))) return BKFAC_ERR_INVALID_ARG;
  if (path != BKFAC_GEMM_TCGEN05 && path != BKFAC_GEMM_SIMT && path != BKFAC_GEMM_TCGEN05_PAIR)
    return BKFAC_ERR_INVALID_ARG;
  if (ldc < std::max(M, 1) || lda < 1 || ldb < 1) return BKFAC_ERR_DIM;
  if (M == 0 || N == 0) return BKFAC_OK;
  bkfac_ctx_s tmp;   // launch bookkeeping only; no workspace
  tmp.use_tc = path != BKFAC_GEMM_SIMT;
  if (path == BKFAC_GEMM_TCGEN05_PAIR) tmp.pair_mode = 2;
  if (tmp.use_tc) {   // once per process (thread-safe static initialisation)
    static const bool attrs = [] { const bool ok = tc_init_attributes(); cudaGetLastError(); return ok; }();
    (void)attrs;
  }
  GemmStage gs;
  GemmProb p = gp(A, lda, B, ldb, C, ldc, M, N, K, alpha, C, ldc, beta);
  const long cap = ws ? (long)(ws_bytes / sizeof(float)) : 0;
  if (ws && cap > 0) gemm_ws(p, ws);
  gs.add(transA != 0, transB != 0, p, cap);
  return run_gemms(&tmp, gs, static_cast<cudaStream_t>(stream), "gemm_user");
}

#ifdef BKFAC_TC_TIMING
void bkfac_debug_tc(unsigned long long* host, int reset) {
  if (reset) { static unsigned long long z[148 * 8]; cudaMemcpyToSymbol(g_tc_dbg, z, sizeof(z)); return; }
  cudaMemcpyFromSymbol(host, g_tc_dbg, sizeof(unsigned long long) * 148 * 8);
}
#endif
#if defined(BKFAC_CHASE_TIMING) || defined(BKFAC_Q2_TIMING) || defined(BKFAC_PANEL_TIMING)
void bkfac_debug_chase(unsigned long long* host, int reset) {
  if (reset) { static unsigned long long z[8]; cudaMemcpyToSymbol(g_chase_dbg, z, sizeof(z)); return; }
  cudaMemcpyFromSymbol(host, g_chase_dbg, sizeof(unsigned long long) * 8);
}
#endif
#ifdef BKFAC_CHOL_TIMING
void bkfac_debug_chol(unsigned long long* host, int reset) {
  if (reset) { static unsigned long long z[8]; cudaMemcpyToSymbol(g_chol_dbg, z, sizeof(z)); return; }
  cudaMemcpyFromSymbol(host, g_chol_dbg, sizeof(unsigned long long) * 8);
}
#endif
#ifdef BKFAC_SYT_TIMING
// tuning builds only (not part of the ABI): device address of a factor's eigensolver
// scratch, where BKFAC_SYT_TIMING kernels leave per-phase cycle sums.
void* bkfac_debug_eig_scratch(bkfac_ctx ctx, int factor) {
  return at<double>(ctx, ctx->f[factor].eig.Y);
}
void bkfac_debug_d2h(void* dst, const void* src, size_t bytes) {
  cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost);
}
#endif

// ------------------------------------------------------------------------- check
bkfac_status bkfac_check(bkfac_ctx ctx, void* stream, int* first_bad, int* info_bits) {
  if (!ctx) return BKFAC_ERR_INVALID_ARG;
  if (!ctx->ws) return BKFAC_ERR_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t n = ctx->f.size() + ctx->l.size() + 1;
  if (!cuda_ok(cudaMemcpyAsync(ctx->host_status, ctx->ws + ctx->status_off, sizeof(int) * n,
                               cudaMemcpyDeviceToHost, st)))
    return BKFAC_ERR_CUDA;
  if (!cuda_ok(cudaStreamSynchronize(st))) return BKFAC_ERR_CUDA;
  int bad = -1, info = 0;
  for (size_t i = 0; i < n; ++i) {
    info |= ctx->host_status[i];
    if (bad < 0 && (ctx->host_status[i] & ST_ERROR_MASK)) bad = (int)i;
  }
  if (first_bad) *first_bad = bad;
  if (info_bits) *info_bits = info;
  return bad >= 0 ? BKFAC_ERR_NUMERIC : BKFAC_OK;
}

}  // extern "C"
