"""Pins of the fp64 oracle against what the paper and the mathematics fix.

None of these compares the oracle with itself: each uses a closed form, an identity
stated in the paper, brute force on tiny inputs, a worked example (tests/golden/),
or a property the paper proves.  CPU only (not marked gpu)."""
import json
import math
import os

import numpy as np
import pytest

import oracle as O
import synth
from tests._util import (eig_rel_err, jacobi_evd, lowrank_diff_fro, lowrank_rel_err,
                         principal_subspace_dist)

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _spec():
    with open(os.path.join(GOLD, "spec_examples.json")) as f:
        return json.load(f)


def _stream(n, c, steps, seed, k=None, decay=0.8, sigma=0.05):
    f = synth.random_case(n, c, 1, seed, k=k, decay=decay, sigma=sigma)
    return [f.batch(i).astype(np.float64) for i in range(steps)]


# ---------------------------------------------------------------- EA (Eq. 8)

def test_ea_recursion_equals_unrolled_sum():
    """Eq.(8) recursion vs its unrolled form sum_i kappa(i) rho^{k-i} M_i M_i^T
    (S.2 :43), kappa(i) = 1 - rho 1{i>0} (:362)."""
    rho = 0.95
    Ms = _stream(24, 3, 11, 1)
    proc = O.ea_process(Ms, rho)
    for k in range(len(Ms)):
        closed = sum((1.0 - rho * (i > 0)) * rho ** (k - i) * Ms[i] @ Ms[i].T
                     for i in range(k + 1))
        assert np.abs(proc[k] - closed).max() <= 1e-12 * np.abs(closed).max()
        # trace recursion: tr(Mcal_k) = rho tr(Mcal_{k-1}) + (1-rho)||M_k||_F^2
        if k > 0:
            t = rho * np.trace(proc[k - 1]) + (1 - rho) * np.sum(Ms[k] ** 2)
            assert abs(np.trace(proc[k]) - t) <= 1e-12 * abs(t)


def test_ea_fixed_point_and_zero_update():
    rho = 0.9
    I = np.eye(5)
    assert np.allclose(O.ea_update(I, np.eye(5), rho), I, atol=1e-15)
    Mc = np.diag([1.0, 2.0, 3.0])
    assert np.allclose(O.ea_update(Mc, np.zeros((3, 2)), rho), rho * Mc, atol=1e-15)


# ---------------------------------------------------------------- dense EVD

def test_evd_closed_form_toeplitz_and_diag():
    sp = _spec()
    n = sp["toeplitz_121"]["n"]
    T = 2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
    V, w = O.sym_evd(T)
    kk = np.arange(1, n + 1)
    exact = np.sort(2 - 2 * np.cos(kk * np.pi / (n + 1)))[::-1]
    assert np.abs(w - exact).max() < 1e-13
    for j in range(n):   # eigenvector of 2-2cos(k pi/(n+1)) is sin(i k pi/(n+1))
        kj = int(round(np.arccos((2 - w[j]) / 2) * (n + 1) / np.pi))
        vec = np.sin(np.arange(1, n + 1) * kj * np.pi / (n + 1))
        vec /= np.linalg.norm(vec)
        assert abs(abs(vec @ V[:, j]) - 1) < 1e-12
    _, w = O.sym_evd(np.diag(sp["evd_diag"]["diag"]).astype(float))
    assert list(w) == sp["evd_diag"]["D"]


def test_evd_matches_bruteforce_jacobi():
    rng = np.random.default_rng(3)
    for n in (3, 6, 9):
        X = rng.standard_normal((n, n))
        X = X + X.T
        V, w = O.sym_evd(X)
        Vj, wj = jacobi_evd(X)
        assert np.abs(w - wj).max() < 1e-11 * np.abs(wj).max()
        assert np.abs(X @ V - V * w[None, :]).max() < 1e-12 * np.abs(w).max()


def test_truncate_worked_example():
    sp = _spec()["truncate"]
    D = np.array(sp["D"], float)
    U = np.eye(len(D))
    Ut, Dt = O.truncate(U, D, sp["r"])
    assert list(Dt) == sp["kept"]
    err = np.linalg.norm(O.densify(U, D) - O.densify(Ut, Dt)) ** 2
    assert abs(err - sp["error_fro_squared"]) < 1e-12
    fl = _spec()["frob_lowrank"]
    Q, _ = np.linalg.qr(np.random.default_rng(0).standard_normal((6, 2)))
    assert abs(np.linalg.norm(O.densify(Q, np.array(fl["D"], float))) - fl["norm"]) < 1e-12


# ---------------------------------------------------------------- Brand (Alg 3)

@pytest.mark.parametrize("case", range(40))
def test_brand_exactness_eq7(case):
    """Brand is exact: [U Q_A] M_S [U Q_A]^T equals
    alpha U D U^T + beta M M^T, and the returned r+n modes densify to it."""
    rng = np.random.default_rng(100 + case)
    d = int(rng.integers(8, 40))
    r = int(rng.integers(1, d // 2))
    n = int(rng.integers(1, d - r))
    U, _ = np.linalg.qr(rng.standard_normal((d, r)))
    D = np.sort(rng.random(r) * 5)[::-1]
    M = rng.standard_normal((d, n))
    alpha, beta = 0.95, 0.05
    target = alpha * (U * D) @ U.T + beta * M @ M.T
    Q_A, M_S = O.brand_core(U, D, M, alpha, beta)
    UQ = np.hstack([U, Q_A])
    assert np.abs(UQ @ M_S @ UQ.T - target).max() < 1e-12 * np.abs(target).max()
    Uh, Dh = O.symmetric_brand(U, alpha * D, math.sqrt(beta) * M)
    assert np.abs(O.densify(Uh, Dh) - target).max() < 1e-11 * np.abs(target).max()
    assert np.abs(Uh.T @ Uh - np.eye(r + n)).max() < 1e-12


def test_brand_top_r_equals_bruteforce_on_tiny_inputs():
    """North star pin: on tiny inputs the result equals brute-force dense EVD of
    rho B_i + (1 - rho) M M^T (here by a pure-Python Jacobi, not LAPACK)."""
    rng = np.random.default_rng(7)
    for _ in range(6):
        d, r, c = 10, 3, 2
        U, _ = np.linalg.qr(rng.standard_normal((d, r)))
        D = np.array([3.0, 1.5, 0.4])
        M = rng.standard_normal((d, c))
        Ub, Db = O.brand_update(U, D, M, 0.95, 0.05, r)
        X = 0.95 * (U * D) @ U.T + 0.05 * M @ M.T
        Vj, wj = jacobi_evd(X)
        assert np.abs(Db - wj[:r]).max() < 1e-12 * wj[0]
        assert lowrank_diff_fro(Vj[:, :r], wj[:r], Ub, Db) < 1e-11 * wj[0]


def test_brand_zero_update_and_empty_basis():
    """A = 0 leaves the rep unchanged; U with D = 0 (phantom basis,
    SURVEY c4) gives the EVD of A A^T."""
    rng = np.random.default_rng(11)
    d, r, c = 30, 5, 4
    U, _ = np.linalg.qr(rng.standard_normal((d, r)))
    D = np.array([5.0, 4.0, 3.0, 2.0, 1.0])
    Ub, Db = O.brand_update(U, D, np.zeros((d, c)), 1.0, 1.0, r)
    assert np.abs(Db - D).max() < 1e-12
    assert lowrank_diff_fro(U, D, Ub, Db) < 1e-12
    M = rng.standard_normal((d, c))
    Ub, Db = O.brand_update(synth.phantom_basis(d, r), np.zeros(r), M, 0.0, 1.0, r)
    Vj, wj = jacobi_evd(M @ M.T) if d <= 12 else (None, None)
    w = np.linalg.svd(M, compute_uv=False) ** 2            # sigma_i(M)^2 = eig(M M^T)
    assert np.abs(Db[:c] - w).max() < 1e-12 * w[0]
    assert np.abs(Db[c:]).max() < 1e-12 * w[0]


def test_dense_path_equals_definition_when_r_plus_c_ge_n():
    rng = np.random.default_rng(5)
    d, r, c = 12, 6, 8           # r + c >= d: B-update not applicable (:457, :493)
    U, _ = np.linalg.qr(rng.standard_normal((d, r)))
    D = np.sort(rng.random(r))[::-1]
    M = rng.standard_normal((d, c))
    Ub, Db = O.brand_update(U, D, M, 0.9, 0.1, r)
    Vj, wj = jacobi_evd(0.9 * (U * D) @ U.T + 0.1 * M @ M.T)
    assert np.abs(Db - wj[:r]).max() < 1e-12 * wj[0]


# ---------------------------------------------------------------- B-process

def _chain(Ms, rho, r, U0=None):
    n = Ms[0].shape[0]
    ch = O.FactorChain(n, r, rho)
    return [ch.step(M, U0) for M in Ms]


def test_tierB_chain_equals_tierD_definition():
    """The Brand recursion (Alg 3 + Alg 4) reproduces the B-process definition
    Eq.(10) step by step."""
    rho = 0.95
    for (n, c, r) in [(64, 8, 16), (40, 3, 12)]:
        Ms = _stream(n, c, 12, 21 + n, decay=0.7)
        reps_b = _chain(Ms, rho, r)
        reps_d = O.bprocess_dense_reps(Ms, rho, r)
        for (Ub, Db), (Ud, Dd) in zip(reps_b, reps_d):
            assert lowrank_rel_err(Ud, Dd, Ub, Db) < 1e-11
            assert eig_rel_err(Dd, Db) < 1e-12


def test_r_ge_n_bprocess_equals_exact_ea():
    """With r >= n nothing is ever truncated, so the B-process equals the exact EA
    factor (north star pin)."""
    rho = 0.9
    Ms = _stream(10, 3, 8, 31)
    ea = O.ea_process(Ms, rho)
    for (U, D), Mk in zip(_chain(Ms, rho, 10), ea):
        assert np.abs(O.densify(U, D) - Mk).max() < 1e-12 * np.abs(Mk).max()


def test_error_recursion_S7():
    """S.7: Mcal_{i+m} - Mt_{B,i+m} = rho (Mcal_{i+m-1} - B_{i+m-1})."""
    rho = 0.95
    Ms = _stream(30, 4, 10, 41)
    ea = O.ea_process(Ms, rho)
    seq = list(O.bprocess_dense(Ms, rho, 6))
    for j in range(1, len(Ms)):
        lhs = ea[j] - seq[j][0]
        rhs = rho * (ea[j - 1] - seq[j - 1][1])
        assert np.abs(lhs - rhs).max() < 1e-12 * np.abs(ea[j]).max()


def _min_eig(X):
    return float(np.linalg.eigvalsh(0.5 * (X + X.T)).min())


def test_prop32_expansions_and_psd_brackets():
    """Prop 3.2: Eq.(12)/(13) equal the directly computed errors
    for an overwrite-at-i run (exact truncation, footnote :106) and a pure run; every
    bracketed term is symmetric PSD (:623)."""
    rho = 0.9
    r = 5
    Ms = _stream(24, 3, 12, 51, decay=0.85)
    ea = O.ea_process(Ms, rho)
    i = 4
    pure = list(O.bprocess_dense(Ms, rho, r))
    Ur, Dr = O.top_r(ea[i], r)
    MR = O.densify(Ur, Dr)                           # Mtilde_{R,i,r}
    over = list(O.bprocess_dense(Ms, rho, r, overwrite={i: MR}))
    scale = np.abs(ea[-1]).max()
    for q in range(1, len(Ms) - i):
        E_pure = ea[i + q] - pure[i + q][0]
        exp_pure = rho ** q * (ea[i] - pure[i][1]) + sum(
            rho ** (q - j) * (pure[i + j][0] - pure[i + j][1]) for j in range(1, q))
        assert np.abs(E_pure - exp_pure).max() < 1e-12 * scale
        E_over = ea[i + q] - over[i + q][0]
        exp_over = rho ** q * (ea[i] - MR) + sum(
            rho ** (q - j) * (over[i + j][0] - over[i + j][1]) for j in range(1, q))
        assert np.abs(E_over - exp_over).max() < 1e-12 * scale
        for X in [ea[i] - pure[i][1], ea[i] - MR, E_pure, E_over] + \
                 [pure[i + j][0] - pure[i + j][1] for j in range(1, q)]:
            assert np.abs(X - X.T).max() < 1e-13 * scale
            assert _min_eig(X) > -1e-12 * scale


def test_prop31_and_MB_beats_B():
    """Prop 3.1 in Frobenius and spectral norms, and the
    inequality ||M - B|| >= ||M - Mt_B|| of PAPER.md:655-656."""
    rho = 0.95
    r, c = 4, 3
    Ms = _stream(20, c, 15, 61, decay=0.9)
    ea = O.ea_process(Ms, rho)
    for k, (Mt, B) in enumerate(O.bprocess_dense(Ms, rho, r)):
        Mk = ea[k]
        Ur, Dr = O.top_r(Mk, r)
        Urc, Drc = O.top_r(Mk, r + c)
        for ordn in ("fro", 2):
            nrm = lambda X: np.linalg.norm(X, ordn)
            tol = 1e-12 * np.abs(Mk).max()
            assert nrm(Mk - B) >= nrm(Mk - O.densify(Ur, Dr)) - tol
            assert nrm(Mk - Mt) >= nrm(Mk - O.densify(Urc, Drc)) - tol
            assert nrm(Mk - B) >= nrm(Mk - Mt) - tol


def test_prop41_decomposition_and_prop42_bound():
    """Prop 4.1: after an RSVD (exact truncation) at k = 0,
    Mcal_k - Mt_k = sum_i kappa(i) rho^{k-i} E_i with E_0 = Mcal_0 - Mt_{R;0,r} and,
    for B-updates, E_i = (Mt_i - B_i)/(1-rho), E_k = 0; for no update
    E_j = M_j M_j^T - Mt_{R;0,r}.  Prop 4.2 (:757-764): ||E_j||_F <= ||M_j M_j^T||_F."""
    rho, r = 0.9, 4
    Ms = _stream(18, 3, 9, 71)
    ea = O.ea_process(Ms, rho)
    U0, D0 = O.top_r(ea[0], r)
    MR0 = O.densify(U0, D0)
    seq = list(O.bprocess_dense(Ms, rho, r, overwrite={0: MR0}))
    k = len(Ms) - 1
    kappa = lambda i: 1.0 - rho * (i > 0)
    E = [ea[0] - MR0] + [(seq[i][0] - seq[i][1]) / (1 - rho) for i in range(1, k)] + [0 * MR0]
    lhs = ea[k] - seq[k][0]
    rhs = sum(kappa(i) * rho ** (k - i) * E[i] for i in range(k + 1))
    assert np.abs(lhs - rhs).max() < 1e-12 * np.abs(ea[k]).max()
    for j in range(1, k):
        assert np.linalg.norm(E[j]) <= np.linalg.norm(Ms[j] @ Ms[j].T) * (1 + 1e-12)
    # no update after the RSVD: Mt_k = Mt_{R;0,r}
    rhs_nu = sum(kappa(i) * rho ** (k - i) * (Ms[i] @ Ms[i].T - MR0) for i in range(k + 1))
    rhs_nu += rho ** k * (ea[0] - Ms[0] @ Ms[0].T)   # E_0 = Mcal_0 - MR0 (= M0M0^T - MR0)
    assert np.abs((ea[k] - MR0) - rhs_nu).max() < 1e-12 * np.abs(ea[k]).max()


def test_prop42_worst_case_equality():
    """S.25 construction: if V_{M_j}^T U_{Mcal_0,r} = 0 then the
    no-update error reaches sqrt(||M_j M_j^T||^2 + ||Mt_{R,0,r}||^2)."""
    rng = np.random.default_rng(81)
    n, c, r = 20, 3, 4
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    M0 = Q[:, :6] @ rng.standard_normal((6, c + 3))
    U0, D0 = O.top_r(M0 @ M0.T, r)
    comp = np.linalg.qr(np.hstack([U0, rng.standard_normal((n, n - r))]))[0][:, r:]
    Mj = comp[:, :c] @ rng.standard_normal((c, c))
    Ej = Mj @ Mj.T - O.densify(U0, D0)
    expect = math.sqrt(np.linalg.norm(Mj @ Mj.T) ** 2 + np.linalg.norm(D0) ** 2)
    assert abs(np.linalg.norm(Ej) - expect) < 1e-12 * expect


# ---------------------------------------------------------------- RSVD

def test_philox_known_answers():
    with open(os.path.join(GOLD, "philox4x32_10_kat.json")) as f:
        kat = json.load(f)
    for case in kat["cases"]:
        ctr = np.array([[int(x, 16) for x in case["ctr"]]], dtype=np.uint64)
        key = tuple(int(x, 16) for x in case["key"])
        out = O.philox4x32_10(ctr, key)[0]
        assert [int(v) for v in out] == [int(x, 16) for x in case["out"]]


def test_gaussian_sketch_is_standard_normal_and_deterministic():
    Om = O.gaussian_sketch(4000, 25, seed=7, counter=3)
    assert Om.shape == (4000, 25)
    assert abs(Om.mean()) < 0.01 and abs(Om.std() - 1) < 0.01
    assert abs(np.mean(Om ** 4) - 3) < 0.1            # Gaussian kurtosis
    assert np.array_equal(Om, O.gaussian_sketch(4000, 25, seed=7, counter=3))
    assert not np.array_equal(Om, O.gaussian_sketch(4000, 25, seed=7, counter=4))
    assert np.array_equal(Om.astype(np.float32).astype(np.float64), Om)


def test_rsvd_exact_on_low_rank_and_zero():
    """exact on rank <= r input; zero input gives zero."""
    rng = np.random.default_rng(91)
    X = rng.standard_normal((40, 2))
    Mc = X @ X.T
    U, D = O.rsvd_overwrite(Mc, 2, 4, 2, seed=1, counter=0)
    assert np.abs(O.densify(U, D) - Mc).max() < 1e-10 * np.abs(Mc).max()
    U, D = O.rsvd_overwrite(np.zeros((40, 40)), 3, 4, 1, seed=1, counter=0)
    assert np.all(D == 0)


def test_rsvd_near_optimal_on_decaying_spectrum():
    """64x64 with lambda_i = 0.5^i, r = 8: error within 1.05x of the
    optimal truncation; more power iterations do not hurt."""
    rng = np.random.default_rng(92)
    Q, _ = np.linalg.qr(rng.standard_normal((64, 64)))
    lam = 0.5 ** np.arange(64)
    Mc = (Q * lam) @ Q.T
    opt = math.sqrt(np.sum(lam[8:] ** 2))
    U, D = O.rsvd_overwrite(Mc, 8, 10, 2, seed=5, counter=0)
    err = np.linalg.norm(Mc - O.densify(U, D))
    assert err <= 1.05 * opt


# ---------------------------------------------------------------- preconditioning

def test_precondition_kronecker_identity():
    """(A (x) Gamma)^{-1} g = vec(Gamma^{-1} Mat(g) A^{-1}), with the
    regularised low-rank factors of Alg 1 lines 16-17 densified: solve the
    Kronecker system directly on d <= 16."""
    rng = np.random.default_rng(101)
    dG, dA, rG, rA = 6, 9, 3, 4
    UG, _ = np.linalg.qr(rng.standard_normal((dG, rG)))
    UA, _ = np.linalg.qr(rng.standard_normal((dA, rA)))
    DG, DA = np.array([3.0, 1.0, 0.5]), np.array([2.0, 1.5, 0.2, 0.1])
    lG, lA = 0.3, 0.2
    J = rng.standard_normal((dG, dA))
    for cont in (False, True):
        S = O.precondition(J, UG, DG, lG, UA, DA, lA, continuation=cont)
        DGe, lGe = O.reg_params(DG, lG, cont)
        DAe, lAe = O.reg_params(DA, lA, cont)
        Gam = O.densify(UG, DGe) + lGe * np.eye(dG)
        Acal = O.densify(UA, DAe) + lAe * np.eye(dA)
        vecS = np.linalg.solve(np.kron(Acal, Gam), J.reshape(-1, order="F"))
        assert np.abs(S - vecS.reshape(dG, dA, order="F")).max() < 1e-12 * np.abs(S).max()
        # residual form: (Gamma~ + lam I) S (A~ + lam I) = J
        assert np.abs(Gam @ S @ Acal - J).max() < 1e-12 * np.abs(J).max()


def test_precondition_factored_alg8_kronecker():
    """Algorithm 8: with Mat(g) = G A^T given factored, the linear-time
    application equals the Kronecker solve (A~ (x) Gamma~)^{-1} vec(G A^T) (:359), with and
    without continuation / relative lambda."""
    rng = np.random.default_rng(202)
    dG, dA, rG, rA, nM = 7, 10, 3, 4, 5
    UG, _ = np.linalg.qr(rng.standard_normal((dG, rG)))
    UA, _ = np.linalg.qr(rng.standard_normal((dA, rA)))
    DG, DA = np.array([2.0, 0.7, 0.3]), np.array([3.0, 1.0, 0.4, 0.05])
    lG, lA = 0.25, 0.15
    G = rng.standard_normal((dG, nM))
    A = rng.standard_normal((dA, nM))
    for cont, rel in ((False, False), (True, False), (False, True)):
        S = O.precondition_factored(G, A, UG, DG, lG, UA, DA, lA, continuation=cont, lam_relative=rel)
        DGe, lGe = O.reg_params(DG, lG, cont, rel)
        DAe, lAe = O.reg_params(DA, lA, cont, rel)
        Gam = O.densify(UG, DGe) + lGe * np.eye(dG)
        Acal = O.densify(UA, DAe) + lAe * np.eye(dA)
        vecS = np.linalg.solve(np.kron(Acal, Gam), (G @ A.T).reshape(-1, order="F"))
        assert np.abs(S - vecS.reshape(dG, dA, order="F")).max() < 1e-12 * np.abs(S).max()


def test_precondition_worked_examples():
    sp = _spec()
    e = sp["apply_inverse_e1"]
    n = e["n"]
    U = np.zeros((n, 1)); U[0, 0] = 1.0
    out = O.apply_inverse_right(np.eye(n), U, np.array(e["D"]), e["lambda"])
    assert np.allclose(np.diag(out), e["column_scales"], atol=1e-15)
    z = sp["apply_inverse_zero_rep"]
    J = np.random.default_rng(1).standard_normal((4, 5))
    S = O.precondition(J, np.zeros((4, 2)), np.zeros(2), z["lambda"],
                       np.zeros((5, 2)), np.zeros(2), z["lambda"])
    assert np.abs(S - J * z["scale"] ** 2).max() < 1e-15
    c = sp["continuation"]
    De, le = O.reg_params(np.array(c["D"], float), c["lambda"], continuation=True)
    assert np.allclose(De, c["D_eff"]) and abs(le - c["lambda_eff"]) < 1e-15
    De, le = O.reg_params(np.array([5.0, 1.0]), 0.1, lam_relative=True)
    assert abs(le - 0.5) < 1e-15          # phi=0.1, max D = 5 -> 0.5


# ---------------------------------------------------------------- light correction (Alg 6)

def test_light_correction_pins():
    """Algorithm 6 and its footnote (:683): after correcting the modes
    col_idx, the error E = Mcal - U D U^T has U_c^T E U_c = 0 on the chosen subspace, so
    ||E||_F cannot increase; U stays orthonormal; correcting every mode of a factor whose
    Mcal lives in span(U) recovers Mcal exactly."""
    rng = np.random.default_rng(303)
    n, r, ncrc = 40, 10, 4
    X = rng.standard_normal((n, 25))
    Mcal = X @ X.T
    U, _ = np.linalg.qr(rng.standard_normal((n, r)))
    D = np.sort(rng.random(r))[::-1] * 50
    idx = rng.choice(r, ncrc, replace=False)
    Uc0 = U[:, idx]
    U2, D2 = O.light_correction(U, D, Mcal, idx)
    E0 = Mcal - O.densify(U, D)
    E1 = Mcal - O.densify(U2, D2)
    assert np.abs(Uc0.T @ E1 @ Uc0).max() < 1e-10 * np.abs(Mcal).max()
    assert np.linalg.norm(E1) <= np.linalg.norm(E0) + 1e-9
    assert np.abs(U2.T @ U2 - np.eye(r)).max() < 1e-12
    others = np.setdiff1d(np.arange(r), idx)
    assert np.array_equal(U2[:, others], U[:, others]) and np.array_equal(D2[others], D[others])
    # full correction of an Mcal inside span(U): exact
    W = U @ rng.standard_normal((r, r))
    M2 = W @ W.T
    U3, D3 = O.light_correction(U, np.zeros(r), M2, np.arange(r))
    assert np.abs(O.densify(U3, D3) - M2).max() < 1e-10 * np.abs(M2).max()


# ---------------------------------------------------------------- §4.2 error metrics

def test_error_metrics_pins():
    """SPEC.md:343-346 examples: approx == ref -> all zero; approx = 2 x ref as an operator
    -> m3 = 1, m4 = 0; m4 is invariant under positive rescaling; the dense inverse form
    equals a direct inverse of U D U^T + lam I (independent of reg_inverse_dense's formula)."""
    rng = np.random.default_rng(404)
    dA, dG, rA, rG = 12, 9, 4, 3
    UA, _ = np.linalg.qr(rng.standard_normal((dA, rA)))
    UG, _ = np.linalg.qr(rng.standard_normal((dG, rG)))
    DA, DG = np.array([5.0, 2.0, 1.0, 0.5]), np.array([3.0, 1.0, 0.2])
    J = rng.standard_normal((dG, dA))
    a, g = (UA, DA, 0.1, False), (UG, DG, 0.2, False)
    assert max(abs(x) for x in O.error_metrics(a, g, a, g, J)) < 1e-14
    Xi = O.reg_inverse_dense(UA, DA, 0.1)
    assert np.abs(Xi - np.linalg.inv(UA @ np.diag(DA) @ UA.T + 0.1 * np.eye(dA))).max() < 1e-12
    # "2 x ref as an operator": the approximate Gamma inverse is twice the reference one.
    # lam/2 with D/2 gives (U D/2 U^T + lam/2 I)^{-1} = 2 (U D U^T + lam I)^{-1}
    g2 = (UG, DG / 2, 0.1, False)
    m1, m2, m3, m4 = O.error_metrics(a, g2, a, g, J)
    assert abs(m2 - 1.0) < 1e-12 and abs(m3 - 1.0) < 1e-12 and abs(m4) < 1e-12 and m1 == 0.0
    # m4 scale invariance: scale the approximate A inverse by 7 (D/7, lam/7)
    b = (UA, DA * 1.3, 0.1, True)
    b7 = (UA, DA * 1.3 / 7, 0.1 / 7, True)
    m4a = O.error_metrics(b, g, a, g, J)[3]
    m4b = O.error_metrics(b7, g, a, g, J)[3]
    assert abs(m4a - m4b) < 1e-12


# ---------------------------------------------------------------- B-R-KFAC chain

def test_brkfac_chain_overwrite_equals_rsvd_then_brand():
    """Alg 5: at k % T == 0 the rep is overwritten by the RSVD
    of Mcal_{k-1} and then B-updated with M_k; the exact-EA factor is maintained."""
    rho, r = 0.95, 6
    Ms = _stream(48, 4, 7, 111)
    ch = O.FactorChain(48, r, rho, rsvd_every=3, oversample=5, power_iters=2, rsvd_seed=9)
    reps = [ch.step(M) for M in Ms]
    ea = O.ea_process(Ms, rho)
    assert np.abs(ch.Mcal - ea[-1]).max() < 1e-12 * np.abs(ea[-1]).max()
    # step 6: overwrite from Mcal_5 (2nd overwrite, counter 1) then Brand with M_6
    Ur, Dr = O.rsvd_overwrite(ea[5], r, 5, 2, 9, 1)
    Ub, Db = O.brand_update(Ur, Dr, Ms[6], rho, 1 - rho, r)
    assert lowrank_rel_err(Ub, Db, *reps[6]) < 1e-12


def test_tierB_equals_tierD_on_cfg1_shapes():
    """Config 1 (BASELINE.json configs[0]): both factors, 20 chained steps."""
    cfg = synth.cfg1_toy()
    for f in cfg.factors:
        Ms = [f.batch(i).astype(np.float64) for i in range(cfg.steps)]
        reps_b = _chain(Ms, cfg.rho, f.r, U0=synth.phantom_basis(f.n, f.r))
        reps_d = O.bprocess_dense_reps(Ms, cfg.rho, f.r)
        for (Ub, Db), (Ud, Dd) in zip(reps_b, reps_d):
            assert lowrank_rel_err(Ud, Dd, Ub, Db) < 1e-10
