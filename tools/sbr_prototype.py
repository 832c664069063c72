"""numpy prototype of csrc/sbr.cuh (two-stage tridiagonalisation) used to check the
algorithm's logic on the CPU: panel QR + two-sided block update to band b, bulge chasing with
the reflector bookkeeping of the kernel, Q2 applied in the kernel's diamond order, Q1 by the
geqrf-layout reflectors with offset b.  Not part of the library or the tests."""
import numpy as np


def house(x):
    alpha = x[0]
    xn2 = float(np.dot(x[1:], x[1:]))
    v = np.zeros_like(x); v[0] = 1.0
    if len(x) <= 1 or xn2 == 0.0:
        return v, 0.0, alpha
    beta = -np.copysign(np.sqrt(alpha * alpha + xn2), alpha)
    tau = (beta - alpha) / beta
    v[1:] = x[1:] / (alpha - beta)
    return v, tau, beta


def sbr(K, b):
    A = K.copy(); m = len(A)
    refl = []  # (col k, v (len m - k - b), tau)
    npan = (m - 2) // b if m - 2 >= b else 0
    for j in range(npan):
        c0, r0 = j * b, (j + 1) * b
        L = m - r0
        P = A[r0:, c0:c0 + b].copy()
        V = np.zeros((L, b)); taus = np.zeros(b)
        for i in range(min(b, L)):
            v, tau, beta = house(P[i:, i])
            if tau != 0.0:
                P[i:, i:] -= tau * np.outer(v, v @ P[i:, i:])
            V[i:, i] = v; taus[i] = tau
            refl.append((c0 + i, v, tau))
        # T (dlarft)
        T = np.zeros((b, b))
        for i in range(b):
            T[:i, i] = -taus[i] * T[:i, :i] @ (V[:, :i].T @ V[:, i])
            T[i, i] = taus[i]
        A22 = A[r0:, r0:]
        X = A22 @ V
        Y = X @ T
        W = Y - 0.5 * V @ (T.T @ (V.T @ Y))
        A[r0:, r0:] = A22 - V @ W.T - W @ V.T
        A[r0:, c0:c0 + b] = np.triu(P)  # R (band), zeros below
        A[c0:c0 + b, r0:] = A[r0:, c0:c0 + b].T
    return A, refl


def chase(Bm, b):
    A = Bm.copy(); m = len(A)
    Vq = {}
    for j in range(m - 2):
        k = 0; u = None; tu = 0.0
        while True:
            s = j + 1 + k * b
            if s >= m:
                break
            nk = min(b, m - s)
            if k == 0:
                x = A[s:s + nk, j].copy()
                v, tau, beta = house(x)
                A[s:s + nk, j] = 0; A[s, j] = beta
                A[j, s:s + nk] = A[s:s + nk, j]
            else:
                E = A[s:s + nk, s - b:s].copy()
                E = E - tu * np.outer(E @ u, u)
                v, tau, beta = house(E[:, 0].copy())
                E = E - tau * np.outer(v, v @ E)
                E[1:, 0] = 0; E[0, 0] = beta
                A[s:s + nk, s - b:s] = E; A[s - b:s, s:s + nk] = E.T
            if tau != 0:
                D = A[s:s + nk, s:s + nk]
                p = tau * D @ v
                w = p - 0.5 * tau * np.dot(p, v) * v
                A[s:s + nk, s:s + nk] = D - np.outer(v, w) - np.outer(w, v)
            vv = np.zeros(b); vv[:nk] = v
            Vq[(j, k)] = (vv, tau)
            u, tu = vv[:b], tau
            if nk < b:
                u = vv
            k += 1
    return A, Vq


def apply_q2(Z, Vq, m, b, G):
    Z = Z.copy()
    nsw = m - 2
    ngroups = (nsw + G - 1) // G
    for g in range(ngroups - 1, -1, -1):
        j0 = g * G; jn = min(G, nsw - j0)
        k = 0
        while True:
            rbase = j0 + 1 + k * b
            if rbase >= m:
                break
            for a in range(jn - 1, -1, -1):
                key = (j0 + a, k)
                if key not in Vq:
                    continue
                v, tau = Vq[key]
                s = j0 + a + 1 + k * b
                n = min(b, m - s)
                vv = v[:n]
                Z[s:s + n] -= tau * np.outer(vv, vv @ Z[s:s + n])
            k += 1
    return Z


def apply_q1(Z, refl, m, b):
    Z = Z.copy()
    for (k, v, tau) in reversed(refl):
        s = k + b
        Z[s:] -= tau * np.outer(v, v @ Z[s:])
    return Z


if __name__ == "__main__":
    rng = np.random.default_rng(0)
    for m, b in [(40, 32), (96, 32), (130, 32), (300, 32), (97, 8)]:
        X = rng.standard_normal((m, m)); K = X @ X.T / m
        Bm, refl = sbr(K, b)
        band_err = np.abs(np.tril(Bm, -b - 1)).max()
        T, Vq = chase(Bm, b)
        tri_err = np.abs(np.tril(T, -2)).max()
        w, Y = np.linalg.eigh(T)
        Z = apply_q2(Y, Vq, m, b, 32)
        Vfull = apply_q1(Z, refl, m, b)
        rec = np.linalg.norm(Vfull @ np.diag(w) @ Vfull.T - K) / np.linalg.norm(K)
        print(f"m={m} b={b}: band {band_err:.1e} tri {tri_err:.1e} reconstruction {rec:.1e} "
              f"eig {np.abs(np.sort(w) - np.linalg.eigvalsh(K)).max():.1e}")


def _debug():
    rng = np.random.default_rng(0)
    m, b = 96, 32
    X = rng.standard_normal((m, m)); K = X @ X.T / m
    Bm, refl = sbr(K, b)
    print("stage1 eig", np.abs(np.linalg.eigvalsh(Bm) - np.linalg.eigvalsh(K)).max(),
          "sym", np.abs(Bm - Bm.T).max())
    T, Vq = chase(Bm, b)
    print("stage2 eig", np.abs(np.linalg.eigvalsh(T) - np.linalg.eigvalsh(Bm)).max(),
          "sym", np.abs(T - T.T).max())
