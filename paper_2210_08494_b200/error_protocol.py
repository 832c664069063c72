"""NEXT-f4: the §4.2 numerical error protocol on synthetic K-factor
streams, run on the GPU through the C ABI.

Time unit.  The paper feeds new K-factor data every T_updt = 10 optimizer steps and holds
every inverse fixed in between (:776), so the error is piecewise constant over blocks of
10 steps.  The protocol here advances one K-factor UPDATE per iteration; every period of
:782 is divided by T_updt (T_RSVD = 50 -> 5 updates, T_inv = 300 -> 30 updates, ...), and
a 300-step window is 30 updates.

Benchmark (:776, "K-FAC with T_inv = T_updt"): the dense EA factors (bkfac_ea_accumulate,
Eq. 8) and their exact eigendecomposition after every update (bkfac_rsvd_overwrite with
rank n and sketch width l = n, R7); no truncation, no continuation.

Algorithms (:782), each fed the same M_A, M_Gamma stream:
  b-kfac          Brand update every update (T_Brand = T_updt, Alg 4)
  b-r-kfac        Brand update every update; every 5 updates it is preceded by the RSVD
                  overwrite of the previous EA factor Mcal_{k-1} (Alg 5, :641-646)
  b-kfac-c        Brand update, light correction every 5 updates, phi = 0.5 (Alg 6-7)
  r-kfac-T50      RSVD of the EA factor every 5 updates (Alg 2)
  r-kfac-T10      RSVD every update
  r-kfac-T300     RSVD once per 30 updates ("no update" inside the window)
  k-fac-T50       exact EVD every 5 updates (full rank)
Every algorithm's schedule is aligned so that its heaviest update happens at the first
update of the window (:784, "we always start our sequence ... exactly when the heaviest
update of the algorithm at hand is performed"): heavy work at k % period == 0 with the
window starting at k0 = burn_in, a multiple of every period.  Low-rank algorithms use
spectrum continuation (:711, :784); the benchmark and k-fac use plain lambda.

Metrics (1)-(4) of :778 per update in the window: relative Frobenius error of A^{-1} and
Gamma^{-1}, relative error of the step s = Gamma^{-1} J A^{-1}, and 1 - cos(angle).  The
steps come from bkfac_precondition; the dense inverse matrices of (1)-(2) are assembled by
bkfac_gemm; PyTorch only takes norms and differences of the results (evaluation glue,
outside the method's hot path).
"""
from __future__ import annotations

import dataclasses
from typing import Callable, Dict, List, Optional, Tuple

from . import binding


@dataclasses.dataclass(frozen=True)
class Algo:
    name: str
    brand: bool = False        # Brand update every K-factor update
    rsvd: int = 0              # RSVD overwrite period (updates), 0 = never
    corct: int = 0             # light-correction period (updates), 0 = never
    evd: int = 0               # exact-EVD period (updates), full rank
    phi: float = 0.5           # phi_corct


def paper_algorithms(t_updt: int = 10) -> Tuple[Algo, ...]:
    """The seven algorithms of :782 with their periods in K-factor updates."""
    u = lambda steps: max(1, steps // t_updt)
    return (Algo("b-kfac", brand=True),
            Algo("b-r-kfac", brand=True, rsvd=u(50)),
            Algo("b-kfac-c", brand=True, corct=u(50), phi=0.5),
            Algo("r-kfac-T50", rsvd=u(50)),
            Algo("r-kfac-T10", rsvd=u(10)),
            Algo("r-kfac-T300", rsvd=u(300)),
            Algo("k-fac-T50", evd=u(50)))


def correction_indices(r: int, phi: float, seed: int, k: int, factor: int):
    """Alg 6 line 2's random choice of n_crc = round(phi * r) distinct columns, drawn on
    the host from a generator keyed by (seed, k, factor) (B-KFAC-C)."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(seed * 1000003 + k * 7919 + factor)
    ncrc = max(1, int(round(phi * r)))
    return torch.randperm(r, generator=g)[:ncrc].to(torch.int32)


def _dense_inverse(U, D, lam: float, continuation: bool):
    """U diag((D' + lam')^{-1} - 1/lam') U^T + I/lam' as a dense n x n tensor, (D', lam') the
    continuation-adjusted pair (:711) when asked.  U is an (r, n) tensor (col-major n x r);
    the rank-r product runs on bkfac_gemm."""
    import torch
    n = U.shape[1]
    D = D.double()
    if continuation and D.numel():
        dmin = float(D.min())
        D, lam = D - dmin, lam + dmin
    s = (1.0 / (D + lam) - 1.0 / lam).float()
    X = torch.eye(n, device=U.device, dtype=torch.float32) / lam
    if U.shape[0]:
        Us = (U * s[:, None]).contiguous()
        binding.bkfac_gemm(False, True, 1.0, Us, U, 1.0, X)
    return X


def _metrics(Ai, Gi, Ar, Gr, s, sr) -> Tuple[float, float, float, float]:
    import torch
    n = lambda x: torch.linalg.norm(x.double())
    m1 = float(n(Ai - Ar) / n(Ar))
    m2 = float(n(Gi - Gr) / n(Gr))
    m3 = float(n(s - sr) / n(sr))
    m4 = float(1.0 - (s.double() * sr.double()).sum() / (n(s) * n(sr)))
    return m1, m2, m3, m4


def synthetic_stream(fA, fG, layer, device) -> Callable:
    """k -> (M_A (c, d_A), M_G (c, d_G), J (d_G, d_A)) device tensors from the seeded synth
    specs (the same generator family as the bench; DESIGN.md input recipe)."""
    import torch

    def gen(k):
        to = lambda x: torch.from_numpy(x).to(device)
        return (to(fA.batch(k).T.copy()), to(fG.batch(k).T.copy()), to(layer.grad(k)))
    return gen


def run(fA, fG, layer, r: int, rho: float, lam: float, burn_in: int = 30, window: int = 30,
        algos: Optional[Tuple[Algo, ...]] = None, oversample: int = 10, power_iters: int = 2,
        seed: int = 0, device: int = 0, gen: Optional[Callable] = None) -> Dict[str, List[tuple]]:
    """Runs burn_in + window K-factor updates; returns, per algorithm, the (m1, m2, m3, m4)
    of every update in the window.  fA / fG are synth.FactorSpec, layer a synth.LayerSpec."""
    import torch
    algos = paper_algorithms() if algos is None else algos
    dev = torch.device(f"cuda:{device}")
    d_A, d_G, c = fA.n, fG.n, fA.c
    dims = (d_A, d_G)
    rr = (min(r, d_A), min(r, d_G))
    for a in algos:
        for p in (a.rsvd, a.corct, a.evd):
            if p and burn_in % p:
                raise ValueError(f"burn_in must be a multiple of every period ({a.name}: {p})")
    gen = gen or synthetic_stream(fA, fG, layer, dev)
    fl = binding.BKFAC_FACTOR_DENSE_EA
    full = binding.Context([(d_A, d_A, c, fl), (d_G, d_G, c, fl)], [(d_G, d_A, d_G, d_A)], device=device)
    low = binding.Context([(d_A, rr[0], c, fl), (d_G, rr[1], c, fl)], [(d_G, d_A, rr[1], rr[0])],
                          device=device)
    K = [torch.zeros((n, n), device=dev) for n in dims]       # the EA factors (Eq. 8)
    ex = [[torch.zeros((n, n), device=dev), torch.zeros(n, device=dev)] for n in dims]
    rep = {a.name: [[torch.zeros((rr[i], n), device=dev), torch.zeros(rr[i], device=dev)]
                    for i, n in enumerate(dims)] for a in algos}
    for a in algos:
        if a.evd:
            rep[a.name] = [[torch.zeros((n, n), device=dev), torch.zeros(n, device=dev)] for n in dims]
    S_ref = torch.empty((d_G, d_A), device=dev)
    S = torch.empty((d_G, d_A), device=dev)
    out: Dict[str, List[tuple]] = {a.name: [] for a in algos}
    for k in range(burn_in + window):
        MA, MG, J = gen(k)
        Ms = (MA, MG)
        # B-R-KFAC (Alg 5, :641-646): the overwrite is RSVD(Mcal_{k-1}), taken before M_k is
        # accumulated; the B-update with M_k follows below as on every update
        for a in algos:
            if a.brand and a.rsvd and k > 0 and k % a.rsvd == 0:
                for i in range(2):
                    U, D = rep[a.name][i]
                    low.bkfac_rsvd_overwrite(i, K[i], min(oversample, dims[i] - rr[i]), power_iters,
                                             seed, 2 * k + i, U, D)
        for i in range(2):
            full.bkfac_ea_accumulate(i, K[i], Ms[i], rho if k else 0.0)
            full.bkfac_rsvd_overwrite(i, K[i], 0, 0, seed, k, ex[i][0], ex[i][1])
        for a in algos:
            for i in range(2):
                U, D = rep[a.name][i]
                if a.evd:
                    if k % a.evd == 0:
                        U.copy_(ex[i][0]); D.copy_(ex[i][1])
                    continue
                if a.rsvd and not a.brand and k % a.rsvd == 0:   # R-KFAC: RSVD(Mcal_k)
                    low.bkfac_rsvd_overwrite(i, K[i], min(oversample, dims[i] - rr[i]), power_iters,
                                             seed, 2 * k + i, U, D)
                    continue
                if a.brand:
                    if k == 0:   # Mtilde_{B,0} = M_0 M_0^T (:584): alpha = 0 on a phantom basis
                        U.zero_(); D.zero_()
                        U[torch.arange(rr[i]), torch.arange(rr[i])] = 1.0
                    Uo, Do = torch.empty_like(U), torch.empty_like(D)
                    low.bkfac_brand_update([dict(factor=i, U_in=U, D_in=D, M=Ms[i], U_out=Uo, D_out=Do,
                                                 alpha=rho if k else 0.0, beta=1.0 - rho if k else 1.0)])
                    U.copy_(Uo); D.copy_(Do)
                    if a.corct and k % a.corct == 0 and k > 0:
                        idx = correction_indices(rr[i], a.phi, seed, k, i).to(dev)
                        low.bkfac_light_correction([dict(factor=i, K=K[i], U=U, D=D, col_idx=idx)])
        if k < burn_in:
            continue
        full.bkfac_precondition([dict(layer=0, U_G=ex[1][0], D_G=ex[1][1], lambda_G=lam,
                                      U_A=ex[0][0], D_A=ex[0][1], lambda_A=lam, J=J, S=S_ref)])
        Ar = _dense_inverse(ex[0][0], ex[0][1], lam, False)
        Gr = _dense_inverse(ex[1][0], ex[1][1], lam, False)
        for a in algos:
            (UA, DA), (UG, DG) = rep[a.name]
            ctx = full if a.evd else low
            cont = not a.evd
            ctx.bkfac_precondition([dict(layer=0, U_G=UG, D_G=DG, lambda_G=lam, U_A=UA, D_A=DA,
                                         lambda_A=lam, J=J, S=S,
                                         flags=binding.BKFAC_PRECOND_CONTINUATION if cont else 0)])
            Ai = _dense_inverse(UA, DA, lam, cont)
            Gi = _dense_inverse(UG, DG, lam, cont)
            out[a.name].append(_metrics(Ai, Gi, Ar, Gr, S, S_ref))
    full.close(); low.close()
    return out


def summary(out: Dict[str, List[tuple]]) -> Dict[str, List[float]]:
    """Average of each metric over the window per algorithm (Table 1, "Avg. Error Metrics")."""
    return {a: [sum(x[i] for x in recs) / max(len(recs), 1) for i in range(4)]
            for a, recs in out.items()}
