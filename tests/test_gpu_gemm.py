"""GPU checks of the 3xTF32 tcgen05 GEMM (the kernel every contraction of the hot path
runs on) through the C ABI (bkfac_gemm), against fp64 numpy on the same fp32 inputs.

Tolerance: 3xTF32 drops only the lo*lo term (2^-22 relative per product) and
accumulates in fp32, whose rounding error grows like sqrt(K) u for random signs; we
require max |dC| / max (|A||B|) <= 1e-6 * max(1, sqrt(K)/8) -- at K = 4609 that is
8.5e-6, still ~60x below what single-pass TF32 (2^-11 ~ 5e-4 per product) gives."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [  # (M, N, K): several tiles, ragged tails in every dimension, long-K splits
    (128, 128, 32), (1, 1, 1), (77, 5, 3), (300, 260, 333), (220, 256, 4609),
    (4609, 256, 220), (129, 127, 1025), (512, 1024, 4097), (33, 1000, 64)]


def _mat(rng, rows, cols):
    return rng.standard_normal((rows, cols)).astype(np.float32)


def _run(ta, tb, M, N, K, alpha, beta, path, seed, with_ws=True):
    import torch
    from paper_2210_08494_b200 import binding
    rng = np.random.default_rng(seed)
    A = _mat(rng, M, K) if ta else _mat(rng, K, M)      # torch layouts (see binding)
    B = _mat(rng, K, N) if tb else _mat(rng, N, K)
    C0 = _mat(rng, N, M)
    tA, tB, tC = (torch.from_numpy(x).cuda() for x in (A, B, C0))
    ws = torch.empty(16 * M * N + 1024, device="cuda") if with_ws else None
    binding.bkfac_gemm(ta, tb, alpha, tA, tB, beta, tC, ws=ws, path=path)
    torch.cuda.synchronize()
    # col-major views: A_cm = A.T etc.
    Acm = A.T.astype(np.float64)
    Bcm = B.T.astype(np.float64)
    opA = Acm.T if ta else Acm
    opB = Bcm.T if tb else Bcm
    ref = alpha * opA @ opB + beta * C0.T.astype(np.float64)
    got = tC.cpu().numpy().T.astype(np.float64)
    scale = float((np.abs(opA) @ np.abs(opB)).max()) * abs(alpha) + abs(beta) * float(np.abs(C0).max())
    return float(np.abs(got - ref).max()) / max(scale, 1e-30) / max(1.0, np.sqrt(K) / 8)


@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False), (True, True)])
@pytest.mark.parametrize("shape", CASES)
def test_tc_gemm_matches_fp64(cuda_lib, ta, tb, shape):
    from paper_2210_08494_b200 import binding
    M, N, K = shape
    err = _run(ta, tb, M, N, K, 1.25, 0.5, binding.BKFAC_GEMM_TCGEN05, seed=M * 7 + N * 3 + K)
    assert err < 1e-6, f"3xTF32 error {err:.3e} (normalised)"


PAIR_CASES = [  # CTA-pair 256 x 256 tiles: several tiles per pair (> 74 tiles), K-blocks
    (2560, 2304, 1100), (300, 700, 64), (4097, 512, 1024), (257, 300, 300)]


@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False), (True, True)])
@pytest.mark.parametrize("shape", PAIR_CASES)
def test_tc_gemm_pair_tiles(cuda_lib, ta, tb, shape):
    """The cta_group::2 path (256 x 256 tiles, TMEM sum / accumulation buffers swapping roles
    per tile) forced on: ragged tails, one to 5 K-blocks per tile, CTA pairs that walk
    several tiles (the per-tile buffer alternation and its barrier phases)."""
    from paper_2210_08494_b200 import binding
    M, N, K = shape
    err = _run(ta, tb, M, N, K, 0.75, -0.5, binding.BKFAC_GEMM_TCGEN05_PAIR, seed=M + 5 * N + 11 * K)
    assert err < 1e-6, f"3xTF32 pair-tile error {err:.3e} (normalised)"


def test_tc_gemm_no_workspace_and_beta_zero(cuda_lib):
    from paper_2210_08494_b200 import binding
    err = _run(True, False, 220, 256, 4609, 1.0, 0.0, binding.BKFAC_GEMM_TCGEN05, seed=3,
               with_ws=False)
    assert err < 1e-6


def test_tc_gemm_is_deterministic(cuda_lib):
    """Split-K reduction order is fixed: two runs are bitwise equal."""
    import torch
    from paper_2210_08494_b200 import binding
    rng = np.random.default_rng(9)
    A = torch.from_numpy(_mat(rng, 220, 4609)).cuda()
    B = torch.from_numpy(_mat(rng, 256, 4609)).cuda()
    ws = torch.empty(16 * 220 * 256, device="cuda")
    outs = []
    for _ in range(2):
        C = torch.zeros((256, 220), device="cuda")
        binding.bkfac_gemm(True, False, 1.0, A, B, 0.0, C, ws=ws)
        outs.append(C)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])


def test_simt_path_same_contract(cuda_lib):
    from paper_2210_08494_b200 import binding
    err = _run(False, True, 300, 260, 333, 1.0, 1.0, binding.BKFAC_GEMM_SIMT, seed=4)
    assert err < 1e-6


@pytest.mark.parametrize("ta,tb", [(False, False), (True, True)])
def test_tc_gemm_misaligned_base(cuda_lib, ta, tb):
    """Operands whose base address is 4-byte but not 16-byte aligned (leading dimension
    a multiple of 4) must take the scalar loader path and still be exact to 3xTF32."""
    import torch
    from paper_2210_08494_b200 import binding
    M, N, K = 256, 192, 300
    rng = np.random.default_rng(21)
    A = _mat(rng, M, K) if ta else _mat(rng, K, M)
    B = _mat(rng, K, N) if tb else _mat(rng, N, K)
    bufA = torch.empty(A.size + 1, device="cuda"); bufB = torch.empty(B.size + 1, device="cuda")
    tA = bufA[1:].view(*A.shape); tA.copy_(torch.from_numpy(A))
    tB = bufB[1:].view(*B.shape); tB.copy_(torch.from_numpy(B))
    C = torch.zeros((N, M), device="cuda")
    binding.bkfac_gemm(ta, tb, 1.0, tA, tB, 0.0, C)
    torch.cuda.synchronize()
    opA = A.astype(np.float64) if ta else A.T.astype(np.float64)
    opB = B.T.astype(np.float64).T if tb else B.T.astype(np.float64)
    opA = A.T.T.astype(np.float64) if ta else A.T.astype(np.float64)
    opB = B.astype(np.float64) if tb else B.T.astype(np.float64)
    ref = opA @ opB
    got = C.cpu().numpy().T
    err = np.abs(got - ref).max() / (np.abs(opA) @ np.abs(opB)).max()
    assert err < 1e-6
