"""Test-side helpers: comparison metrics and a brute-force Jacobi EVD.

Nothing here is used by the oracle or by the CUDA path."""
from __future__ import annotations

import math

import numpy as np


def lowrank_diff_fro(U1, D1, U2, D2) -> float:
    """||U1 diag(D1) U1^T - U2 diag(D2) U2^T||_F without densifying and without
    assuming orthonormality (SURVEY §8(c) "parity metric pitfall"): with
    [U1 U2] = Q R (fp64 QR), the difference equals Q R diag(D1, -D2) R^T Q^T."""
    U1 = np.asarray(U1, dtype=np.float64)
    U2 = np.asarray(U2, dtype=np.float64)
    D = np.concatenate([np.asarray(D1, np.float64), -np.asarray(D2, np.float64)])
    _, R = np.linalg.qr(np.hstack([U1, U2]), mode="reduced")
    return float(np.linalg.norm((R * D[None, :]) @ R.T))


def lowrank_rel_err(U_ref, D_ref, U, D) -> float:
    """Relative Frobenius error of the reconstructed U D U^T against the reference."""
    return lowrank_diff_fro(U_ref, D_ref, U, D) / max(float(np.linalg.norm(D_ref)), 1e-300)


def eig_rel_err(D_ref, D) -> float:
    """Normwise eigenvalue error max_i |dD_i| / D_1."""
    D_ref = np.asarray(D_ref, np.float64)
    D = np.asarray(D, np.float64)
    return float(np.max(np.abs(D_ref - D)) / max(abs(D_ref[0]), 1e-300))


def jacobi_evd(A, sweeps: int = 60, tol: float = 1e-15):
    """Cyclic Jacobi eigenvalue algorithm in pure Python loops (tiny n only).
    Brute force independent of LAPACK: used to pin the oracle's EVD steps."""
    n = len(A)
    a = [[float(A[i][j]) for j in range(n)] for i in range(n)]
    v = [[1.0 if i == j else 0.0 for j in range(n)] for i in range(n)]
    for _ in range(sweeps):
        off = sum(a[i][j] ** 2 for i in range(n) for j in range(n) if i != j)
        if off < tol * tol * max(1e-300, sum(a[i][i] ** 2 for i in range(n))):
            break
        for p in range(n - 1):
            for q in range(p + 1, n):
                if a[p][q] == 0.0:
                    continue
                theta = (a[q][q] - a[p][p]) / (2.0 * a[p][q])
                t = math.copysign(1.0, theta) / (abs(theta) + math.sqrt(theta * theta + 1.0))
                c = 1.0 / math.sqrt(t * t + 1.0)
                s = t * c
                for k in range(n):
                    akp, akq = a[k][p], a[k][q]
                    a[k][p] = c * akp - s * akq
                    a[k][q] = s * akp + c * akq
                for k in range(n):
                    apk, aqk = a[p][k], a[q][k]
                    a[p][k] = c * apk - s * aqk
                    a[q][k] = s * apk + c * aqk
                for k in range(n):
                    vkp, vkq = v[k][p], v[k][q]
                    v[k][p] = c * vkp - s * vkq
                    v[k][q] = s * vkp + c * vkq
    w = np.array([a[i][i] for i in range(n)])
    V = np.array(v)
    order = np.argsort(-w, kind="stable")
    return V[:, order], w[order]


def principal_subspace_dist(U1, U2) -> float:
    """sin of the largest principal angle between span(U1) and span(U2)."""
    Q1, _ = np.linalg.qr(np.asarray(U1, np.float64))
    Q2, _ = np.linalg.qr(np.asarray(U2, np.float64))
    s = np.linalg.svd(Q1.T @ Q2, compute_uv=False)
    return float(math.sqrt(max(0.0, 1.0 - float(np.min(s)) ** 2)))
