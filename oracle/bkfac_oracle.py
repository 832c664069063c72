"""Plain, slow, obviously-correct fp64 oracle of the B-KFAC hot path.

TEST INFRASTRUCTURE ONLY — imported solely by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (``cpu_baseline`` / ``--impl reference``).  It shares no code,
header, table or constant generator with the CUDA path; neither imports the other.

Every function cites the passage of ``PAPER.md`` (arxiv 2210.08494) it follows.
Library primitives used as single steps: ``@`` (matmul), ``numpy.linalg.eigh``
(dense symmetric EVD, LAPACK syevd), ``numpy.linalg.qr`` (Householder QR, LAPACK
geqrf/orgqr), ``numpy.argsort``.  No blocking, fusion or reordering beyond what the
paper's formulas state.

Pins (see ``tests/test_oracle_pins.py``): closed forms (Eq.(8)'s unrolled sum, S.2),
Brand exactness Eq.(7) by dense reconstruction, brute-force Jacobi EVD on tiny
inputs, r >= n  =>  B-process == exact EA, error recursion S.7, Prop 3.1, Prop 3.2
(expansions + PSD brackets), the "M~_B beats B" inequality (:655-656), Prop 4.1
decomposition and E_k = 0, Prop 4.2 bound and worst-case equality, RSVD exactness
on low-rank input, Philox4x32-10 known-answer vectors, and the Kronecker identity
(Eq.(4) context) for the preconditioner.  Every function is pinned;
none is "parity unpinned".

Conventions: matrices are float64 numpy arrays in mathematical orientation
(an n x c matrix has shape (n, c)).  A low-rank PSD representation is (U, D) with
U (n x r) orthonormal and D (r,) non-increasing, >= 0.
"""
from __future__ import annotations

import math
from typing import Iterable, List, Optional, Sequence, Tuple

import numpy as np

f64 = np.float64

# --------------------------------------------------------------------------
# Dense EA K-factor  (Eq.(5); :563-570 Eq.(8); S.1 :33-40)
# --------------------------------------------------------------------------


def ea_update(Mcal_prev: Optional[np.ndarray], M: np.ndarray, rho: float) -> np.ndarray:
    """One step of Eq.(8):
    Mcal_0 = M_0 M_0^T;  Mcal_j = rho*Mcal_{j-1} + (1-rho) M_j M_j^T  (j >= 1).
    ``Mcal_prev is None`` marks j = 0 (kappa(0) = 1)."""
    M = np.asarray(M, dtype=f64)
    G = M @ M.T
    if Mcal_prev is None:
        return G
    return rho * np.asarray(Mcal_prev, dtype=f64) + (1.0 - rho) * G


def ea_process(Ms: Sequence[np.ndarray], rho: float) -> List[np.ndarray]:
    """The exact EA process Mcal_0..Mcal_k of Eq.(8)."""
    out: List[np.ndarray] = []
    prev = None
    for M in Ms:
        prev = ea_update(prev, M, rho)
        out.append(prev)
    return out


# --------------------------------------------------------------------------
# Dense symmetric EVD and truncation (Alg 3 line "EVD(M_S)" PAPER.md:505;
# truncation "retaining only the first r modes" PAPER.md:534, Alg 4 :540-543)
# --------------------------------------------------------------------------


def sym_evd(X: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """Full symmetric EVD, eigenvalues sorted non-increasing (library primitive
    numpy.linalg.eigh on the symmetrised input)."""
    X = np.asarray(X, dtype=f64)
    X = 0.5 * (X + X.T)
    w, V = np.linalg.eigh(X)
    order = np.argsort(-w, kind="stable")
    return V[:, order], w[order]


def truncate(U: np.ndarray, D: np.ndarray, r: int) -> Tuple[np.ndarray, np.ndarray]:
    """Keep the first r modes (Alg 4 lines 2-4)."""
    return U[:, :r].copy(), D[:r].copy()


def top_r(X: np.ndarray, r: int) -> Tuple[np.ndarray, np.ndarray]:
    """Optimal rank-r truncation of a symmetric PSD matrix: U_{X,r}, D clamped >= 0
    (the eigenvalues of a PSD matrix are non-negative)."""
    V, w = sym_evd(X)
    U, D = truncate(V, w, r)
    return U, np.maximum(D, 0.0)


def densify(U: np.ndarray, D: np.ndarray) -> np.ndarray:
    """U diag(D) U^T."""
    U = np.asarray(U, dtype=f64)
    return (U * np.asarray(D, dtype=f64)[None, :]) @ U.T


# --------------------------------------------------------------------------
# B-process, tier D (definition): Eq.(10), S.4 :55-65
# --------------------------------------------------------------------------


def bprocess_dense(Ms: Sequence[np.ndarray], rho: float, r: int,
                   overwrite: Optional[dict] = None):
    """Yield, for i = 0, 1, ..., the dense matrices (Mtilde_{B,i}, B_i) of Eq.(10)
    (PAPER.md:582-586):

        Mtilde_{B,0} = M_0 M_0^T,
        B_i          = U_{Mt,r} U_{Mt,r}^T Mtilde_{B,i} U_{Mt,r} U_{Mt,r}^T   (top-r truncation)
        Mtilde_{B,i+1} = rho * B_i + (1 - rho) M_{i+1} M_{i+1}^T.

    ``overwrite`` maps i -> a dense rank-r matrix X_i that replaces B_i (the
    B-R-KFAC over-write B_i = Mtilde_{R,i,r}, Alg 5 :641-646)."""
    Mt = None
    for i, M in enumerate(Ms):
        M = np.asarray(M, dtype=f64)
        if i == 0:
            Mt = M @ M.T
        else:
            Mt = rho * B + (1.0 - rho) * (M @ M.T)  # noqa: F821  (B from previous i)
        U, D = top_r(Mt, r)
        B = densify(U, D)
        if overwrite is not None and i in overwrite:
            B = np.asarray(overwrite[i], dtype=f64)
        yield Mt, B


def bprocess_dense_reps(Ms: Sequence[np.ndarray], rho: float, r: int):
    """(U_r, D_r) of B_i for every i, tier D."""
    out = []
    for Mt, _B in bprocess_dense(Ms, rho, r):
        out.append(top_r(Mt, r))
    return out


# --------------------------------------------------------------------------
# Symmetric Brand, tier B (recursion): Alg 3 PAPER.md:491-514 with Eq.(7)
# :431-450 (B <- A, V <- U), scaled per Alg 4 :546 (U, rho*D, sqrt(1-rho)*A)
# --------------------------------------------------------------------------


def symmetric_brand(U: np.ndarray, D: np.ndarray, A: np.ndarray, reorth: bool = True):
    """Algorithm 3, unweighted: exact EVD of X^ = U D U^T + A A^T.

    Line 1 (:497): P = U^T A ("U^T Z", Z read as A); A_perp = A - U P.
      With ``reorth`` one classical Gram-Schmidt re-projection is applied (the
      paper is silent); in exact arithmetic it is a no-op.
    Line 2 (:499): Q_A R_A = QR(A_perp)  (Householder; footnote :451 allows any).
    Line 3 (:503): M_S = [[I, U^T A],[0, R_A]] diag(D, I) [[I, U^T A],[0, R_A]]^T.
    Line 4 (:505): U_M D_M U_M^T = EVD(M_S).
    Line 5 (:507-509): U^ = [U Q_A] U_M, D^ = D_M.
    Requires r + n < d (Alg 3 input, :493).  Returns all r + n modes, sorted."""
    U = np.asarray(U, dtype=f64)
    D = np.asarray(D, dtype=f64)
    A = np.asarray(A, dtype=f64)
    d, r = U.shape
    n = A.shape[1]
    if r + n >= d:
        raise ValueError("symmetric Brand needs r + n < d (PAPER.md:493)")
    P = U.T @ A
    A_perp = A - U @ P
    if reorth:
        P2 = U.T @ A_perp
        A_perp = A_perp - U @ P2
        P = P + P2
    Q_A, R_A = np.linalg.qr(A_perp, mode="reduced")
    left = np.block([[np.eye(r), P], [np.zeros((n, r)), R_A]])
    mid = np.block([[np.diag(D), np.zeros((r, n))], [np.zeros((n, r)), np.eye(n)]])
    M_S = left @ mid @ left.T
    U_M, D_M = sym_evd(M_S)
    U_hat = np.hstack([U, Q_A]) @ U_M
    return U_hat, D_M


def brand_update(U: np.ndarray, D: np.ndarray, M: np.ndarray, alpha: float, beta: float,
                 r_out: int, reorth: bool = True) -> Tuple[np.ndarray, np.ndarray]:
    """The hot-path operation (BASELINE.json north_star):
    top-r_out eigendecomposition of alpha * U diag(D) U^T + beta * M M^T.

    Per step alpha = rho, beta = 1 - rho (Alg 4 :546 passes rho*D and sqrt(1-rho)*A);
    at init alpha = 0, beta = 1 (Mtilde_{B,0} = M_0 M_0^T, :584; kappa(0) = 1, :362).
    When r + c < n: Symmetric Brand (Alg 3) then truncation (Alg 4 :540-543).
    When r + c >= n the B-update is not applicable (:457, :493, :705); the result is
    then the definition itself: dense EVD of the n x n sum (SURVEY §8(a) a6')."""
    U = np.asarray(U, dtype=f64)
    D = np.asarray(D, dtype=f64)
    M = np.asarray(M, dtype=f64)
    n, r = U.shape
    c = M.shape[1]
    if r + c < n:
        Uh, Dh = symmetric_brand(U, alpha * D, math.sqrt(beta) * M, reorth=reorth)
        Uo, Do = truncate(Uh, Dh, r_out)
        return Uo, np.maximum(Do, 0.0)
    X = alpha * densify(U, D) + beta * (M @ M.T)
    return top_r(X, r_out)


def brand_core(U: np.ndarray, D: np.ndarray, M: np.ndarray, alpha: float, beta: float,
               reorth: bool = True):
    """Exposes (Q_A, M_S) of Alg 3 for pins of Eq.(7)."""
    U = np.asarray(U, dtype=f64)
    A = math.sqrt(beta) * np.asarray(M, dtype=f64)
    r = U.shape[1]
    n = A.shape[1]
    P = U.T @ A
    A_perp = A - U @ P
    if reorth:
        P2 = U.T @ A_perp
        A_perp = A_perp - U @ P2
        P = P + P2
    Q_A, R_A = np.linalg.qr(A_perp, mode="reduced")
    left = np.block([[np.eye(r), P], [np.zeros((n, r)), R_A]])
    mid = np.block([[alpha * np.diag(np.asarray(D, dtype=f64)), np.zeros((r, n))],
                    [np.zeros((n, r)), np.eye(n)]])
    return Q_A, left @ mid @ left.T


# --------------------------------------------------------------------------
# Counter-based Gaussian sketch for the RSVD.  The GPU side
# implements the same published generator independently (Philox4x32-10,
# Salmon et al. 2011) — random numbers the method draws are an input.
# --------------------------------------------------------------------------

_PHILOX_M0 = 0xD2511F53
_PHILOX_M1 = 0xCD9E8D57
_PHILOX_W0 = 0x9E3779B9
_PHILOX_W1 = 0xBB67AE85
_MASK32 = 0xFFFFFFFF


def philox4x32_10(ctr: np.ndarray, key: Tuple[int, int]) -> np.ndarray:
    """Philox4x32 with 10 rounds.  ``ctr``: uint64 array (..., 4) holding 32-bit
    words; ``key``: two 32-bit words.  Returns uint64 array (..., 4)."""
    c = np.array(ctr, dtype=np.uint64) & np.uint64(_MASK32)
    k0 = np.uint64(key[0] & _MASK32)
    k1 = np.uint64(key[1] & _MASK32)
    m0 = np.uint64(_PHILOX_M0)
    m1 = np.uint64(_PHILOX_M1)
    mask = np.uint64(_MASK32)
    for rnd in range(10):
        if rnd > 0:
            k0 = (k0 + np.uint64(_PHILOX_W0)) & mask
            k1 = (k1 + np.uint64(_PHILOX_W1)) & mask
        p0 = m0 * c[..., 0]
        p1 = m1 * c[..., 2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & mask
        hi1, lo1 = p1 >> np.uint64(32), p1 & mask
        c = np.stack([hi1 ^ c[..., 1] ^ k0, lo1, hi0 ^ c[..., 3] ^ k1, lo0], axis=-1)
    return c


def gaussian_sketch(n: int, l: int, seed: int, counter: int) -> np.ndarray:
    """Omega ~ N(0,1)^{n x l} as float32 (then promoted), column-major element
    index e = j*n + i.  Philox4x32-10 with key = (seed lo, seed hi) and counter
    (e//4 lo, e//4 hi, counter lo, counter hi); word pair (2p, 2p+1), p = (e%4)//2,
    gives uniforms u = (x + 0.5) 2^-32 and Box-Muller in fp64:
    z = sqrt(-2 ln u_a) * (cos if e even else sin)(2 pi u_b); z is rounded to fp32."""
    e = np.arange(n * l, dtype=np.uint64)
    blk = e >> np.uint64(2)
    ctr = np.stack([blk & np.uint64(_MASK32), blk >> np.uint64(32),
                    np.full_like(blk, counter & _MASK32),
                    np.full_like(blk, (counter >> 32) & _MASK32)], axis=-1)
    x = philox4x32_10(ctr, (seed & _MASK32, (seed >> 32) & _MASK32))
    t = (e & np.uint64(3)).astype(np.int64)
    p = t >> 1
    xa = np.take_along_axis(x, (2 * p)[:, None], axis=1)[:, 0].astype(f64)
    xb = np.take_along_axis(x, (2 * p + 1)[:, None], axis=1)[:, 0].astype(f64)
    ua = (xa + 0.5) * 2.0 ** -32
    ub = (xb + 0.5) * 2.0 ** -32
    rad = np.sqrt(-2.0 * np.log(ua))
    th = 2.0 * math.pi * ub
    z = np.where((t & 1) == 0, rad * np.cos(th), rad * np.sin(th))
    z32 = z.astype(np.float32)
    return z32.reshape(l, n).T.astype(f64)  # column-major fill


# --------------------------------------------------------------------------
# RSVD overwrite (Alg 1 line 13 :397; Alg 5 :641-646)
# --------------------------------------------------------------------------


def rsvd_overwrite(Mcal: np.ndarray, r: int, oversample: int, power_iters: int,
                   seed: int, counter: int, Omega: Optional[np.ndarray] = None):
    """Randomized range finder on the dense EA factor (symmetric variant):
    Y = Mcal Omega; q times {Q = orth(Y); Y = Mcal Q}; Q = orth(Y);
    B = Q^T Mcal Q; EVD(B); U = Q V_{1..r}, D = Lambda_{1..r} (clamped >= 0)."""
    Mcal = np.asarray(Mcal, dtype=f64)
    n = Mcal.shape[0]
    l = r + oversample
    if l > n:
        raise ValueError("r + oversample must be <= n (SPEC.md:70)")
    if Omega is None:
        Omega = gaussian_sketch(n, l, seed, counter)
    Y = Mcal @ Omega
    for _ in range(power_iters):
        Q, _ = np.linalg.qr(Y, mode="reduced")
        Y = Mcal @ Q
    Q, _ = np.linalg.qr(Y, mode="reduced")
    B = Q.T @ Mcal @ Q
    V, w = sym_evd(B)
    return Q @ V[:, :r], np.maximum(w[:r], 0.0)


# --------------------------------------------------------------------------
# Light correction, Algorithm 6 -- B-KFAC-C, Algorithm 7 (:691-701)
# --------------------------------------------------------------------------


def light_correction(U: np.ndarray, D: np.ndarray, Mcal: np.ndarray,
                     col_idx: Sequence[int]) -> Tuple[np.ndarray, np.ndarray]:
    """Algorithm 6.  col_idx (n_crc distinct indices < r) is the random
    choice of line 2, passed in.  Line 4: M_S = U_c^T Mcal U_c with U_c = U[:, col_idx];
    line 5: U_S D_S U_S^T = EVD(M_S); line 7: the representation is corrected in that
    subspace -- U[:, col_idx] <- U_c U_S (the EVD's U expressed in the original basis,
    the reading that keeps U n x r), D[col_idx] <- D_S.  Other columns are unchanged."""
    U = np.array(U, dtype=f64, copy=True)
    D = np.array(D, dtype=f64, copy=True)
    idx = np.asarray(col_idx, dtype=np.int64)
    Uc = U[:, idx]
    MS = Uc.T @ np.asarray(Mcal, dtype=f64) @ Uc
    US, DS = sym_evd(MS)
    U[:, idx] = Uc @ US
    D[idx] = DS
    return U, D


# --------------------------------------------------------------------------
# Regularised low-rank inverse application (Alg 1 lines 16-17 :403-405;
# identity (A (x) Gamma)^{-1} g = vec(Gamma^{-1} Mat(g) A^{-1}), :359;
# spectrum continuation :711; relative lambda = lambda_max * phi, :940)
# --------------------------------------------------------------------------


def reg_params(D: np.ndarray, lam: float, continuation: bool = False,
               lam_relative: bool = False) -> Tuple[np.ndarray, float]:
    """Effective (D, lambda).  Relative mode: lambda = lam * max(D) (§6 :940).
    Continuation (:711): lambda <- lambda + min_i D_i, D <- D - min_i D_i."""
    D = np.asarray(D, dtype=f64).copy()
    if lam_relative:
        lam = float(lam) * (float(D.max()) if D.size else 0.0)
    if continuation and D.size:
        dmin = float(D.min())
        lam = lam + dmin
        D = D - dmin
    return D, float(lam)


def apply_inverse_right(J: np.ndarray, U: np.ndarray, D: np.ndarray, lam: float) -> np.ndarray:
    """Alg 1 line 16 (:403): J U [(D + lam I)^{-1} - lam^{-1} I] U^T + lam^{-1} J."""
    J = np.asarray(J, dtype=f64)
    U = np.asarray(U, dtype=f64)
    s = 1.0 / (np.asarray(D, dtype=f64) + lam) - 1.0 / lam
    return ((J @ U) * s[None, :]) @ U.T + J / lam


def apply_inverse_left(Mk: np.ndarray, U: np.ndarray, D: np.ndarray, lam: float) -> np.ndarray:
    """Alg 1 line 17 (:405): U [(D + lam I)^{-1} - lam^{-1} I] U^T M + lam^{-1} M."""
    Mk = np.asarray(Mk, dtype=f64)
    U = np.asarray(U, dtype=f64)
    s = 1.0 / (np.asarray(D, dtype=f64) + lam) - 1.0 / lam
    return U @ ((U.T @ Mk) * s[:, None]) + Mk / lam


def precondition(J: np.ndarray, U_G: np.ndarray, D_G: np.ndarray, lam_G: float,
                 U_A: np.ndarray, D_A: np.ndarray, lam_A: float,
                 continuation: bool = False, lam_relative: bool = False) -> np.ndarray:
    """S = Gamma~^{-1} J A~^{-1} (Alg 1 lines 16-17), J = Mat(g)
    of shape d_Gamma x d_A."""
    DA, lA = reg_params(D_A, lam_A, continuation, lam_relative)
    DG, lG = reg_params(D_G, lam_G, continuation, lam_relative)
    Mk = apply_inverse_right(J, U_A, DA, lA)
    return apply_inverse_left(Mk, U_G, DG, lG)


def precondition_factored(G: np.ndarray, A: np.ndarray, U_G: np.ndarray, D_G: np.ndarray,
                          lam_G: float, U_A: np.ndarray, D_A: np.ndarray, lam_A: float,
                          continuation: bool = False, lam_relative: bool = False) -> np.ndarray:
    """Algorithm 8 (Eq.(20)-(21)), linear in d: the gradient arrives
    factored, Mat(g) = G A^T with G (d_Gamma x n_M), A (d_A x n_M), and
      A^T_bold = A^T V_A [(D_A + lam I)^{-1} - lam^{-1} I] V_A^T + lam^{-1} A^T
      G_bold   = V_G [(D_G + lam I)^{-1} - lam^{-1} I] V_G^T G + lam^{-1} G
      S        = G_bold A^T_bold.
    Effective (D, lambda) as in ``precondition`` (reg_params)."""
    G = np.asarray(G, dtype=f64)
    A = np.asarray(A, dtype=f64)
    DA, lA = reg_params(D_A, lam_A, continuation, lam_relative)
    DG, lG = reg_params(D_G, lam_G, continuation, lam_relative)
    UA = np.asarray(U_A, dtype=f64)
    UG = np.asarray(U_G, dtype=f64)
    sA = 1.0 / (DA + lA) - 1.0 / lA
    sG = 1.0 / (DG + lG) - 1.0 / lG
    At_bold = ((A.T @ UA) * sA[None, :]) @ UA.T + A.T / lA
    G_bold = UG @ ((UG.T @ G) * sG[:, None]) + G / lG
    return G_bold @ At_bold


# --------------------------------------------------------------------------
# §4.2 error protocol metrics -- NEXT-f4
# --------------------------------------------------------------------------


def reg_inverse_dense(U: np.ndarray, D: np.ndarray, lam: float, continuation: bool = False,
                      lam_relative: bool = False) -> np.ndarray:
    """The regularised inverse of a low-rank representation as a dense matrix
    (Alg 1 lines 16-17, :403-405): U diag((D + lam)^{-1} - lam^{-1}) U^T + I / lam, with the
    effective (D, lam) of reg_params."""
    U = np.asarray(U, dtype=f64)
    De, le = reg_params(D, lam, continuation, lam_relative)
    s = 1.0 / (De + le) - 1.0 / le
    return (U * s[None, :]) @ U.T + np.eye(U.shape[0]) / le


def error_metrics(approx_A, approx_G, ref_A, ref_G, J: np.ndarray) -> Tuple[float, float, float, float]:
    """§4.2 metrics: (1) ||A~^{-1} - A^{-1}_ref||_F / ||A^{-1}_ref||_F,
    (2) the same for Gamma, (3) ||s~ - s_ref||_F / ||s_ref||_F, (4) 1 - cos(angle(s~, s_ref)),
    with s = Gamma^{-1} J A^{-1} (the step of Alg 1 lines 14-17).  Each argument approx_* /
    ref_* is (U, D, lam, continuation); the inverses are formed densely."""
    Ai, Gi = reg_inverse_dense(*approx_A), reg_inverse_dense(*approx_G)
    Ar, Gr = reg_inverse_dense(*ref_A), reg_inverse_dense(*ref_G)
    J = np.asarray(J, dtype=f64)
    s_t = Gi @ J @ Ai
    s_r = Gr @ J @ Ar
    m1 = float(np.linalg.norm(Ai - Ar) / np.linalg.norm(Ar))
    m2 = float(np.linalg.norm(Gi - Gr) / np.linalg.norm(Gr))
    nr = float(np.linalg.norm(s_r))
    if nr == 0.0:
        raise ValueError("ZeroReference: the reference step is zero (SPEC.md:342)")
    m3 = float(np.linalg.norm(s_t - s_r) / nr)
    m4 = float(1.0 - np.sum(s_t * s_r) / (np.linalg.norm(s_t) * nr))
    return m1, m2, m3, m4


# --------------------------------------------------------------------------
# Stack driver: init, Brand each step, optional RSVD overwrite
# of the dense EA factor every T steps (Alg 5), preconditioning each step.
# --------------------------------------------------------------------------


class FactorChain:
    """B-KFAC / B-R-KFAC chain of one K-factor, fp64."""

    def __init__(self, n: int, r: int, rho: float, keep_dense: bool = False,
                 rsvd_every: int = 0, oversample: int = 10, power_iters: int = 2,
                 rsvd_seed: int = 0):
        self.n, self.r, self.rho = n, r, rho
        self.keep_dense = keep_dense or rsvd_every > 0
        self.rsvd_every = rsvd_every
        self.oversample, self.power_iters, self.rsvd_seed = oversample, power_iters, rsvd_seed
        self.k = -1
        self.U: Optional[np.ndarray] = None
        self.D: Optional[np.ndarray] = None
        self.Mcal: Optional[np.ndarray] = None
        self.n_overwrites = 0

    def step(self, M: np.ndarray, U0: Optional[np.ndarray] = None):
        """Advance to step k+1 with incoming M (n x c)."""
        self.k += 1
        k = self.k
        if k == 0:
            U0 = np.asarray(U0, dtype=f64) if U0 is not None else np.eye(self.n, self.r)
            self.U, self.D = brand_update(U0, np.zeros(U0.shape[1]), M, 0.0, 1.0, self.r)
        else:
            if self.rsvd_every and k % self.rsvd_every == 0:
                # Alg 5 (:641-646): overwrite with RSVD(Mcal_{k-1}), then B-update.
                # sketch width l = r + r_o capped at n (reading R7: l = n is the
                # exact EVD of Mcal_{k-1}, the limit of the range finder)
                ro = min(self.oversample, self.n - self.r)
                self.U, self.D = rsvd_overwrite(self.Mcal, self.r, ro,
                                                self.power_iters, self.rsvd_seed,
                                                self.n_overwrites)
                self.n_overwrites += 1
            self.U, self.D = brand_update(self.U, self.D, M, self.rho, 1.0 - self.rho, self.r)
        if self.keep_dense:
            self.Mcal = ea_update(self.Mcal if k > 0 else None, M, self.rho)
        return self.U, self.D
