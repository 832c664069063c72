"""Helpers for the GPU parity tests: move numpy (math-orientation) arrays through the
C ABI.  Conversions only; no arithmetic of the method."""
import numpy as np


def to_dev_cols(X):
    """numpy n x k (math orientation) -> CUDA tensor (k, n) == col-major n x k, fp32."""
    import torch
    return torch.from_numpy(np.ascontiguousarray(np.asarray(X, np.float32).T)).cuda()


def from_dev_cols(t):
    return t.detach().double().cpu().numpy().T.copy()


def to_dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, np.float32))).cuda()


def gpu_brand(ctx, factor, U, D, M, alpha, beta, flags=0):
    """Runs bkfac_brand_update on fp32 copies of (U, D, M); returns float64 numpy (U, D)."""
    import torch
    tU = to_dev_cols(U)
    tD = to_dev(D)
    tM = to_dev_cols(M)
    Uo = torch.empty_like(tU)
    Do = torch.empty_like(tD)
    ctx.bkfac_brand_update([dict(factor=factor, U_in=tU, D_in=tD, M=tM, U_out=Uo, D_out=Do,
                                 alpha=alpha, beta=beta, flags=flags)])
    torch.cuda.synchronize()
    return from_dev_cols(Uo), Do.double().cpu().numpy()
