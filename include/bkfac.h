/*
 * bkfac.h — C ABI of the B200-native B-KFAC hot path (arxiv 2210.08494).
 *
 * What it computes (BASELINE.json north_star; PAPER.md = /root/reference/PAPER.md):
 *   - bkfac_brand_update: the per-step symmetric Brand low-rank eigen-update of an
 *     exponential-average (EA) K-factor: the top-r eigendecomposition of
 *         alpha * U_in diag(D_in) U_in^T + beta * M M^T
 *     (Alg 3; Alg 4, :536-552, which passes (U, rho*D, sqrt(1-rho)*A);
 *     the B-process Eq.(10), :580-589).  Per step alpha = rho, beta = 1 - rho; at the
 *     first step alpha = 0, beta = 1 (Mtilde_{B,0} = M_0 M_0^T, :584; kappa(0) = 1, :362).
 *     When r + c >= n the B-update is "not applicable" (:457, :493); the library then
 *     forms the n x n sum densely and eigendecomposes it (same result, SURVEY §8(a) a6').
 *   - bkfac_ea_accumulate: the dense EA update K <- rho K + (1 - rho) M M^T
 *     (Alg 1 lines 5/9, :381, :390; Eq.(8) :563-568).  rho = 0 gives K = M M^T (k = 0).
 *   - bkfac_rsvd_overwrite: the B-R-KFAC overwrite (Alg 5, :641-646): randomized range
 *     finder on the dense EA factor (Alg 1 line 13, :397): Gaussian sketch + power
 *     iterations, symmetric projection, small EVD, top-r.
 *   - bkfac_precondition: S = Gamma~^{-1} J A~^{-1} with the regularised low-rank
 *     inverses of Alg 1 lines 16-17 (:403-405), J = Mat(g) (:359, :401), optionally with
 *     spectrum continuation (:711) and relative lambda (lambda = lambda * max D, :940).
 *
 * Conventions
 *   - All float buffers are DEVICE memory owned by the caller, fp32.
 *   - "col-major a x b" = each length-a column is contiguous (a PyTorch tensor of
 *     shape (b, a)).  U (n x r), M (n x c), K_dense (n x n, symmetric) are col-major.
 *     J and S are row-major d_G x d_A (PyTorch weight.grad layout).
 *   - Leading dimensions.  The ld_* fields of the argument structs give the distance in
 *     floats between consecutive columns of a col-major operand (rows of J / S); 0 means
 *     packed (the row count; d_A for J / S), otherwise ld >= that (BKFAC_ERR_DIM).  With a
 *     16-byte-aligned base and ld a multiple of 4 the contractions read the operand with
 *     16-byte loads; odd packed layouts (n = 4097, d_A = 16385, ...) cost an internal
 *     aligned copy (Brand operands) or the 4-byte load path (preconditioner operands), so
 *     callers should allocate with ld rounded up to a multiple of 32.  Padding entries are
 *     never read and never written (except U_out's columns beyond r_out, zero-filled).
 *   - D arrays have length r, are non-increasing and >= 0 on output.
 *   - The library never allocates device memory: the caller allocates the workspace
 *     (bkfac_workspace_bytes) and registers it (bkfac_set_workspace).  The context
 *     retains no caller pointer beyond a call except that workspace.
 *   - Calls are asynchronous and stream-ordered on `stream` (a cudaStream_t, passed
 *     as void* so this header needs no CUDA include).  Argument validation is
 *     synchronous and returns immediately with an error code; no work is enqueued
 *     on error.  Device-side numeric trouble (non-finite inputs, eigensolver
 *     failure) sets a per-factor status word reported by bkfac_check.
 *   - A context is not thread-safe; use one per device/thread.
 */
#ifndef BKFAC_H
#define BKFAC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bkfac_ctx_s* bkfac_ctx;

typedef enum {
  BKFAC_OK = 0,
  BKFAC_ERR_INVALID_ARG = 1,  /* null pointer, alpha < 0, beta <= 0, lambda <= 0, bad index */
  BKFAC_ERR_DIM = 2,          /* c > c_max, r > n, dimension mismatch with the descriptor    */
  BKFAC_ERR_RANK = 3,         /* r + oversample > n (RSVD)                                    */
  BKFAC_ERR_ALIAS = 4,        /* U_out aliases U_in (or D_out aliases D_in)                   */
  BKFAC_ERR_WORKSPACE = 5,    /* workspace missing or too small                               */
  BKFAC_ERR_CUDA = 6,         /* a CUDA runtime call failed                                   */
  BKFAC_ERR_NUMERIC = 7,      /* device status word reports non-finite data / no convergence  */
  BKFAC_ERR_UNSUPPORTED = 8   /* shape outside what this build supports                       */
} bkfac_status;

/* bkfac_factor_desc.flags */
#define BKFAC_FACTOR_DENSE_EA 1   /* the factor may be RSVD-overwritten: reserve RSVD workspace */
/* Paper-faithful output rank (NEXT-f1, Alg 4 :540-548, :655-656): the
 * factor's basis has r_out = min(n, r + c_max) columns.  A Brand update with batch c writes
 * the min(n, r + c) eigenpairs of M~_B = alpha U_r D_r U_r^T + beta M M^T -- its whole
 * spectrum, i.e. the rank-(r + c) matrix the paper preconditions with -- into U_out
 * (n x r_out) and D_out (r_out), zero-filling columns / entries beyond that; it reads
 * U_in / D_in through their first r columns / entries (the truncation to r that precedes
 * every Brand step, Alg 4 lines 2-4).  Layers preconditioned with such factors declare
 * r_G / r_A = r_out; the zero columns contribute nothing. */
#define BKFAC_FACTOR_FULL_RANK 2

/* bkfac_brand_args.flags */
#define BKFAC_BRAND_NO_REORTH 1   /* skip the second (CGS2) projection against U           */
#define BKFAC_BRAND_NO_REFRESH 2  /* skip the orthonormality refresh of U_out (R8)  */

/* bkfac_precond_args.flags */
#define BKFAC_PRECOND_CONTINUATION 1    /* lambda <- lambda + min D, D <- D - min D (:711)  */
#define BKFAC_PRECOND_LAMBDA_RELATIVE 2 /* lambda <- lambda * max D (phi_lambda, :940)      */

/* One K-factor: dimension n, target rank r (1 <= r <= n), largest batch c_max.       */
typedef struct { int n; int r; int c_max; int flags; } bkfac_factor_desc;

/* One preconditioned layer: gradient J is d_G x d_A (row-major); ranks of its factors;
 * n_max > 0 reserves workspace for bkfac_precondition_factored with up to n_max samples. */
typedef struct { int d_G; int d_A; int r_G; int r_A; int n_max; } bkfac_layer_desc;

/* Creates a context on CUDA device `device` for `nfactors` factors and `nlayers`
 * layers.  Descriptors are copied.  Returns BKFAC_ERR_DIM on invalid shapes. */
bkfac_status bkfac_init(bkfac_ctx* out, const bkfac_factor_desc* factors, int nfactors,
                        const bkfac_layer_desc* layers, int nlayers, int device);

/* Bytes of device workspace needed so that every factor and layer can be processed
 * in a single batched call (all of them concurrently). */
/* Run-time options of a context (defaults: the tuned configuration).  Synchronous host-side
 * state; affects calls issued afterwards.  BKFAC_ERR_INVALID_ARG for an unknown option or an
 * out-of-range value.
 *   BKFAC_OPT_TWO_STAGE   eigensolver reduction: 0 auto (two-stage dense->band->tridiagonal,
 *                         sbr.cuh, for orders whose one-stage tiles do not fit a cluster's
 *                         shared memory, 864 < m <= 1632, when at least 20 such problems share
 *                         the launch; fewer run the one-stage kernel on CTA clusters), 1
 *                         one-stage only, 2 two-stage for every order it supports
 *                         (34 <= m <= 1632).  Pinned (1 or 2), a factor's result does not depend
 *                         on the batch it shares a call with (bitwise); auto trades that for
 *                         strong scaling.
 *   BKFAC_OPT_GT_CLUSTER  1..8: largest cluster of the global-tile one-stage tridiagonalisation
 *                         and of the global-tile Cholesky (default 8)
 *   BKFAC_OPT_GEMM_PAIR   0 never / 1 auto (default) / 2 always: CTA-pair 256 x 256 GEMM tiles
 *   BKFAC_OPT_GEMM_SIMT   != 0: every contraction on the fp32 CUDA-core GEMM (comparison)
 *   BKFAC_OPT_EA_MODE     bkfac_brand_ea_update's EA placement: 0 beside the eigensolver on the
 *                         SMs it leaves idle (default), 1 serially first, 2 beside uncapped,
 *                         3 one CTA per tile, 4 as 3 with the join right after the reduction
 *   BKFAC_OPT_EA_CAP      > 0: the EA grid cap in CTAs instead of the idle-SM count
 *   BKFAC_OPT_SYT_CLUSTER > 0: wider clusters for the shared-memory tridiagonalisation (tuning)
 *   BKFAC_OPT_BT_SIMT     != 0: back-transform Gram/T products on the fp32 SIMT GEMM
 *   BKFAC_OPT_CHOL_BLOCKED Cholesky of orders > 256: 1 (default) blocked with the panel solve,
 *                         trailing SYRK and inverse on the tcgen05 GEMM, 0 one tiled CTA or
 *                         cluster per factor on CUDA cores
 *   BKFAC_OPT_NVTX        != 0: every stage of every call inside a host NVTX range named by
 *                         its stage tag (profiling: ncu --nvtx --nvtx-include "<tag>/")
 *   BKFAC_OPT_SBR_X       two-stage band reduction: 1 (default) X = A22 V and the block update
 *                         in their own kernels on the lower triangle only (warp-level tensor-core
 *                         MMA, 3xTF32), 0 both on the tcgen05 GEMM (full symmetric storage,
 *                         mirrored update)
 *   BKFAC_OPT_GEMM_CAP    0 (default): persistent tcgen05 GEMM grids span all SMs; 2..148: at
 *                         most this many CTAs (two calls running concurrently on two streams --
 *                         the stack's pipelined preconditioning -- each keep their own SMs).
 *                         Tile work and arithmetic are unchanged (bitwise the same results).
 *   BKFAC_OPT_PREC_BLOCK  0 (default): bkfac_precondition's output GEMM accumulates K = r_A + r_G
 *                         in TMEM blocks of 256 terms, each added to a running sum with
 *                         round-to-nearest, like every other contraction; 1..4096: blocks of
 *                         this many 32-term chunks (>= K / 32: one block -- about 7 % faster
 *                         on that GEMM, but with the accumulate bias of the longer block
 *                         the error of S's components inside
 *                         span(U_G) x span(U_A), where the low-rank term cancels most of
 *                         J / (lambda lambda), grows 4x: 3.0e-4 -> 1.2e-3 at lambda = 0.01) */
#define BKFAC_OPT_TWO_STAGE 1
#define BKFAC_OPT_GT_CLUSTER 2
#define BKFAC_OPT_GEMM_PAIR 3
#define BKFAC_OPT_GEMM_SIMT 4
#define BKFAC_OPT_EA_MODE 5
#define BKFAC_OPT_EA_CAP 6
#define BKFAC_OPT_SYT_CLUSTER 7
#define BKFAC_OPT_BT_SIMT 8
#define BKFAC_OPT_CHOL_BLOCKED 9
#define BKFAC_OPT_NVTX 10
#define BKFAC_OPT_SBR_X 11
#define BKFAC_OPT_GEMM_CAP 12
#define BKFAC_OPT_PREC_BLOCK 13
bkfac_status bkfac_set_option(bkfac_ctx ctx, int option, int value);

size_t bkfac_workspace_bytes(bkfac_ctx ctx);

/* Registers caller-owned device memory (>= bkfac_workspace_bytes, 256-B aligned).
 * Also holds the per-factor status words; they are cleared here. */
bkfac_status bkfac_set_workspace(bkfac_ctx ctx, void* dev_ptr, size_t bytes);

bkfac_status bkfac_destroy(bkfac_ctx ctx);

/* U_out (n x r col-major), D_out (r) = top_r( alpha U_in diag(D_in) U_in^T + beta M M^T ).
 * U_in must have orthonormal columns (any orthonormal basis with D_in = 0 at init).
 * M is col-major n x c, c <= c_max.  U_out must not alias U_in (BKFAC_ERR_ALIAS); the
 * caller ping-pongs two buffers.  Eigenvector signs are unspecified.  `count`
 * updates (distinct factors) run as one batch. */
typedef struct {
  int factor;
  const float* U_in; const float* D_in;
  const float* M; int c;
  float* U_out; float* D_out;
  float alpha; float beta;
  int flags;
  int ld_U;   /* leading dimension of U_in and U_out (0: n) */
  int ld_M;   /* leading dimension of M (0: n) */
} bkfac_brand_args;
bkfac_status bkfac_brand_update(bkfac_ctx ctx, const bkfac_brand_args* args, int count,
                                void* stream);

/* K_dense (n x n) <- rho K_dense + (1 - rho) M M^T.  Requires BKFAC_FACTOR_DENSE_EA. */
bkfac_status bkfac_ea_accumulate(bkfac_ctx ctx, int factor, float* K_dense, const float* M,
                                 int c, float rho, void* stream);

/* Batched form of bkfac_ea_accumulate: `count` distinct factors in one grouped launch. */
typedef struct {
  int factor; float* K_dense; const float* M; int c; float rho;
  int ld_M;   /* leading dimension of M (0: n); K_dense is packed */
} bkfac_ea_args;
bkfac_status bkfac_ea_accumulate_batch(bkfac_ctx ctx, const bkfac_ea_args* args, int count,
                                       void* stream);

/* bkfac_brand_update(args, count) and bkfac_ea_accumulate_batch(ea_args, ea_count) of one
 * step (Alg 5 lines 5-6 / Alg 1 lines 16-17) in one call.
 * Same results as the two calls in sequence on `stream`; the EA GEMM runs on an internal
 * stream, forked when the Brand path reaches its eigensolver and capped to the SMs the
 * tridiagonalisation leaves idle, and joined before the call's work completes on
 * `stream`.  No K_dense may alias a U_in / U_out (BKFAC_ERR_ALIAS). */
bkfac_status bkfac_brand_ea_update(bkfac_ctx ctx, const bkfac_brand_args* args, int count,
                                   const bkfac_ea_args* ea_args, int ea_count, void* stream);

/* U_out (n x r), D_out (r) <- RSVD of K_dense with l = r + oversample sketch columns and
 * `power_iters` re-orthonormalised power iterations.  The Gaussian sketch is
 * Philox4x32-10 keyed by `seed`, stream `counter`. */
bkfac_status bkfac_rsvd_overwrite(bkfac_ctx ctx, int factor, const float* K_dense,
                                  int oversample, int power_iters, uint64_t seed,
                                  uint64_t counter, float* U_out, float* D_out, void* stream);

/* Batched form of bkfac_rsvd_overwrite: `count` distinct factors, stage by stage. */
typedef struct {
  int factor; const float* K_dense; int oversample; int power_iters;
  uint64_t seed; uint64_t counter; float* U_out; float* D_out;
  int ld_U;   /* leading dimension of U_out (0: n); K_dense is packed */
} bkfac_rsvd_args;
bkfac_status bkfac_rsvd_overwrite_batch(bkfac_ctx ctx, const bkfac_rsvd_args* args, int count,
                                        void* stream);

/* NEXT-f3, Algorithm 6, the light correction of B-KFAC-C (Alg 7,
 * :691-701): for the n_crc modes col_idx[0..n_crc) (distinct, in [0, r); the random choice
 * of line 2, drawn by the caller), M_S = U_c^T K_dense U_c with U_c = U[:, col_idx];
 * U_S D_S U_S^T = EVD(M_S); U[:, col_idx] <- U_c U_S, D[col_idx] <- max(D_S, 0).  U (n x r
 * col-major; a full-rank factor's leading r columns) and D are updated in place; other
 * columns are untouched and U stays orthonormal.  col_idx is a device int32 array; an
 * index outside [0, r) sets the factor's status (BKFAC_ERR_NUMERIC from bkfac_check).
 * Requires BKFAC_FACTOR_DENSE_EA; 1 <= n_crc <= r. */
typedef struct {
  int factor; const float* K_dense; float* U; float* D; const int* col_idx; int n_crc;
  int ld_U;   /* leading dimension of U (0: n); K_dense is packed */
} bkfac_correct_args;
bkfac_status bkfac_light_correction(bkfac_ctx ctx, const bkfac_correct_args* args, int count,
                                    void* stream);

/* Omega (n x l col-major) <- the RSVD Gaussian test matrix for (seed, counter): the
 * sketch step of bkfac_rsvd_overwrite exposed on its own (Philox4x32-10, key = seed,
 * counter words (e/4 lo, e/4 hi, counter lo, counter hi) for element e = j*n + i;
 * Box-Muller in fp64 on the word pair ((e%4)/2)*2, cos for even e, sin for odd e). */
bkfac_status bkfac_gaussian_sketch(float* Omega, int n, int l, uint64_t seed, uint64_t counter,
                                   void* stream);

/* S (d_G x d_A row-major) = Gamma~^{-1} J A~^{-1}, with
 *   A~^{-1} = U_A diag((D_A + lambda_A)^{-1} - 1/lambda_A) U_A^T + I/lambda_A  (and Gamma).
 * S must not alias J.  `layer` indexes the layer descriptors given to bkfac_init. */
typedef struct {
  int layer;
  const float* U_G; const float* D_G; float lambda_G;
  const float* U_A; const float* D_A; float lambda_A;
  const float* J; float* S;
  int flags;
  int ld_UG; int ld_UA;   /* leading dimensions of U_G (0: d_G) and U_A (0: d_A) */
  int ld_J; int ld_S;     /* row strides of J and S (0: d_A) */
} bkfac_precond_args;
bkfac_status bkfac_precondition(bkfac_ctx ctx, const bkfac_precond_args* args, int count,
                                void* stream);

/* NEXT-f2, Algorithm 8 (Eq.(20)-(21)): the same S = Gamma~^{-1} Mat(g)
 * A~^{-1} when the gradient arrives factored, Mat(g) = G A^T, without ever forming it:
 *   A_b = A~^{-1} A = U_A diag(s_A) U_A^T A + A / lambda_A     (d_A x n)
 *   G_b = Gamma~^{-1} G = U_G diag(s_G) U_G^T G + G / lambda_G (d_G x n)
 *   S   = G_b A_b^T                                             (d_G x d_A row-major)
 * O(r (d_G + d_A) n) for the inverse applications.  G (d_G x n) and A (d_A x n) are
 * col-major (the per-sample matrices whose Gram products are the K-factor statistics:
 * the M of the layer's two factors); n <= the layer's n_max (BKFAC_ERR_DIM otherwise).
 * Flags as bkfac_precondition.  S must not alias G or A. */
typedef struct {
  int layer;
  const float* U_G; const float* D_G; float lambda_G;
  const float* U_A; const float* D_A; float lambda_A;
  const float* G; const float* A; int n;
  float* S;
  int flags;
  int ld_UG; int ld_UA;   /* leading dimensions of U_G (0: d_G) and U_A (0: d_A) */
  int ld_G; int ld_A;     /* leading dimensions of G (0: d_G) and A (0: d_A) */
  int ld_S;               /* row stride of S (0: d_A) */
} bkfac_precond_factored_args;
bkfac_status bkfac_precondition_factored(bkfac_ctx ctx, const bkfac_precond_factored_args* args,
                                         int count, void* stream);

/* The fp32-accurate GEMM every contraction above runs on, exposed for testing and for
 * callers that need the same arithmetic:  C = alpha op(A) op(B) + beta C  (BLAS col-major;
 * op(X) = X^T when trans* != 0; C is M x N with leading dimension ldc >= M).
 * path BKFAC_GEMM_TCGEN05: 3xTF32 on tcgen05 tensor cores (the hot-path kernel);
 * path BKFAC_GEMM_SIMT: fp32 FFMA on CUDA cores (comparison baseline);
 * path BKFAC_GEMM_TCGEN05_PAIR: the tcgen05 kernel forced onto CTA-pair 256 x 256 tiles
 * (cta_group::2), which the library otherwise picks only for large long-K stages (tests).
 * ws (device, optional, ws_bytes) enables deterministic split-K when K is long and the
 * output small; without it the product runs unsplit.  Asynchronous on `stream`. */
#define BKFAC_GEMM_TCGEN05 0
#define BKFAC_GEMM_SIMT 1
#define BKFAC_GEMM_TCGEN05_PAIR 2
bkfac_status bkfac_gemm(int transA, int transB, int M, int N, int K, float alpha, const float* A,
                        int lda, const float* B, int ldb, float beta, float* C, int ldc, float* ws,
                        size_t ws_bytes, int path, void* stream);

/* Synchronises `stream`, reads the per-factor status words.  Returns BKFAC_OK or
 * BKFAC_ERR_NUMERIC (first offending factor in *first_bad_factor, else -1).
 * Informational bits (e.g. a Cholesky pivot dropped for a rank-deficient residual)
 * are returned in *info_bits (OR over factors) without failing. */
bkfac_status bkfac_check(bkfac_ctx ctx, void* stream, int* first_bad_factor, int* info_bits);

/* Number of kernels this context has launched since creation (host-side counter). */
uint64_t bkfac_launch_count(bkfac_ctx ctx);

/* Optional per-stage timing: when enabled, every stage (a group of launches of one
 * kernel family) is bracketed by CUDA events recorded on the launching stream, with
 * its algorithmic flop and byte counts. */
typedef struct {
  char name[32];
  long long calls;      /* stage executions                */
  long long launches;   /* kernel launches inside them      */
  double ms;            /* summed event-timed duration      */
  double flops;         /* algorithmic flops                */
  double bytes;         /* algorithmic bytes                */
} bkfac_stage_stat;
bkfac_status bkfac_profile_enable(bkfac_ctx ctx, int enable);   /* also clears records */
/* Synchronises the recorded events, aggregates per stage name into out[0..max_out),
 * clears the records and returns the number of distinct stages (-1 on error). */
int bkfac_profile_read(bkfac_ctx ctx, bkfac_stage_stat* out, int max_out);
/* Number of stage records so far (-1 on error). */
int bkfac_profile_count(bkfac_ctx ctx);
/* As bkfac_profile_read over records [begin, end) only, and without clearing them.  Events
 * recorded while profiling was on during a CUDA-graph capture are graph nodes: every replay
 * re-records them, so reading a graph's record range after each (synchronised) replay gives
 * that replay's per-stage times.  Returns the number of distinct stages (-1 on error). */
int bkfac_profile_read_range(bkfac_ctx ctx, int begin, int end, bkfac_stage_stat* out,
                             int max_out);

const char* bkfac_status_string(bkfac_status s);

/* Build identification string (compile flags / arch). */
const char* bkfac_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* BKFAC_H */
