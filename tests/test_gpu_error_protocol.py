"""NEXT-f4 parity: the §4.2 error protocol on the GPU
(paper_2210_08494_b200.error_protocol, every stage through the C ABI) against the same
protocol replayed with the fp64 oracle on the same fp32 inputs, schedule and random draws.

The metrics are relative errors between two approximations that both carry fp32-level
noise on the GPU side; the GPU and oracle metric agree to the propagated fp32 error of the
inverses (TOL_PREC = 1e-3 relative per step, R4), so each metric must match to
1e-3 relative plus an absolute floor of 2e-5 (fp32 noise on a relative error whose own
value is ~1e-5..1e-1)."""
import numpy as np
import pytest

import oracle as O
import synth

REL, ABS = 1e-3, 2e-5


def _oracle_protocol(fA, fG, layer, r, rho, lam, burn_in, window, algos, oversample, power_iters, seed):
    from paper_2210_08494_b200.error_protocol import correction_indices
    dims = (fA.n, fG.n)
    rr = (min(r, fA.n), min(r, fG.n))
    K = [None, None]
    rep = {a.name: [None, None] for a in algos}
    out = {a.name: [] for a in algos}
    for k in range(burn_in + window):
        Ms = (fA.batch(k).astype(np.float64), fG.batch(k).astype(np.float64))
        J = layer.grad(k).astype(np.float64)
        # B-R-KFAC (Alg 5): RSVD(Mcal_{k-1}), then the B-update with M_k
        for a in algos:
            if a.brand and a.rsvd and k > 0 and k % a.rsvd == 0:
                for i in range(2):
                    rep[a.name][i] = O.rsvd_overwrite(K[i], rr[i], min(oversample, dims[i] - rr[i]),
                                                      power_iters, seed, 2 * k + i)
        ex = []
        for i in range(2):
            K[i] = O.ea_update(K[i], Ms[i], rho)
            V, w = O.sym_evd(K[i])
            ex.append((V, np.maximum(w, 0.0)))
        for a in algos:
            for i in range(2):
                if a.evd:
                    if k % a.evd == 0:
                        rep[a.name][i] = ex[i]
                    continue
                if a.rsvd and not a.brand and k % a.rsvd == 0:   # R-KFAC: RSVD(Mcal_k)
                    rep[a.name][i] = O.rsvd_overwrite(K[i], rr[i], min(oversample, dims[i] - rr[i]),
                                                      power_iters, seed, 2 * k + i)
                    continue
                if a.brand:
                    if k == 0:
                        U0, D0 = synth.phantom_basis(dims[i], rr[i]).astype(np.float64), np.zeros(rr[i])
                        rep[a.name][i] = O.brand_update(U0, D0, Ms[i], 0.0, 1.0, rr[i])
                    else:
                        U, D = rep[a.name][i]
                        rep[a.name][i] = O.brand_update(U, D, Ms[i], rho, 1.0 - rho, rr[i])
                    if a.corct and k % a.corct == 0 and k > 0:
                        idx = correction_indices(rr[i], a.phi, seed, k, i).numpy()
                        U, D = rep[a.name][i]
                        rep[a.name][i] = O.light_correction(U, D, K[i], idx)
        if k < burn_in:
            continue
        for a in algos:
            (UA, DA), (UG, DG) = rep[a.name]
            cont = not a.evd
            out[a.name].append(O.error_metrics((UA, DA, lam, cont), (UG, DG, lam, cont),
                                               (ex[0][0], ex[0][1], lam, False),
                                               (ex[1][0], ex[1][1], lam, False), J))
    return out


@pytest.mark.gpu
def test_error_protocol_matches_oracle(cuda_lib):
    from paper_2210_08494_b200 import error_protocol as EP
    fA = synth.random_case(48, 8, 12, seed=11, k=10, decay=0.8, sigma=0.05)
    fG = synth.random_case(40, 8, 12, seed=12, k=10, decay=0.8, sigma=0.05)
    layer = synth.LayerSpec("tiny", 48, 40, 0, 1, 0.1, 13)
    algos = (EP.Algo("b-kfac", brand=True), EP.Algo("b-r-kfac", brand=True, rsvd=2),
             EP.Algo("b-kfac-c", brand=True, corct=2, phi=0.5), EP.Algo("r-kfac-T2", rsvd=2),
             EP.Algo("r-kfac-T1", rsvd=1), EP.Algo("r-kfac-T6", rsvd=6), EP.Algo("k-fac-T2", evd=2))
    kw = dict(r=12, rho=0.95, lam=0.1, burn_in=6, window=6, algos=algos, oversample=6,
              power_iters=2, seed=5)
    got = EP.run(fA, fG, layer, **kw)
    ref = _oracle_protocol(fA, fG, layer, **kw)
    for a in algos:
        g, o = np.asarray(got[a.name]), np.asarray(ref[a.name])
        assert g.shape == o.shape == (6, 4)
        assert np.all(np.isfinite(g))
        bad = np.abs(g - o) > REL * np.abs(o) + ABS
        assert not bad.any(), (a.name, g[bad], o[bad])
    # the window starts on every algorithm's heaviest update (:784): all R-KFAC
    # representations are the same RSVD of the same EA factor there (B-R-KFAC's overwrite
    # reads Mcal_{k-1} and is followed by a B-update, Alg 5)
    first = [np.asarray(got[n][0]) for n in ("r-kfac-T2", "r-kfac-T1", "r-kfac-T6")]
    for f in first[1:]:
        assert np.allclose(f, first[0], rtol=1e-4, atol=1e-6)


def test_paper_algorithm_periods():
    """:782's seven algorithms with T_updt = 10: periods in K-factor updates."""
    from paper_2210_08494_b200 import error_protocol as EP
    al = {a.name: a for a in EP.paper_algorithms()}
    assert set(al) == {"b-kfac", "b-r-kfac", "b-kfac-c", "r-kfac-T50", "r-kfac-T10",
                       "r-kfac-T300", "k-fac-T50"}
    assert al["b-r-kfac"].rsvd == 5 and al["b-kfac-c"].corct == 5 and al["b-kfac-c"].phi == 0.5
    assert al["r-kfac-T10"].rsvd == 1 and al["r-kfac-T300"].rsvd == 30 and al["k-fac-T50"].evd == 5
