"""Seeded synthetic inputs shared by the oracle, the tests and the bench.

This module holds NO arithmetic of the method (no EA update, no Brand step, no
RSVD, no preconditioning).  It only draws the inputs the paper's workloads
consume, so that the fp64 oracle (``oracle/``) and the CUDA path
(``paper_2210_08494_b200``) can be fed identical fp32 data.

Recipe:

* The paper measures on CIFAR10 / VGG16_bn K-factors, which are
  not available here.  The stand-in is the "significant eigenspectrum decay"
  the paper relies on: every incoming statistic is

      M_k = L · diag(s) · W_k + sigma · N_k            (n x c, c = n_BS)

  with L (n x k) a fixed seeded orthonormal basis per factor, s_j = decay^j,
  W_k ~ N(0,1)^{k x c} and N_k ~ N(0,1)^{n x c} fresh every step.
* Gradients J (d_Gamma x d_A, PyTorch ``weight.grad`` layout) are N(0, var).
* Everything is cast to float32 before either side sees it.
* Seeds: base 20221015; factor seed = base*1000 + global factor index; the
  step stream is keyed by (factor seed, step) through numpy's SeedSequence,
  so factor inputs are identical at every GPU count.
"""
from __future__ import annotations

import dataclasses
import functools
from typing import List, Optional, Sequence, Tuple

import numpy as np

BASE_SEED = 20221015


def factor_seed(global_index: int) -> int:
    return BASE_SEED * 1000 + int(global_index)


def _rng(*key: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(k) for k in key])))


@functools.lru_cache(maxsize=256)
def orthonormal_basis(n: int, k: int, seed: int) -> np.ndarray:
    """Seeded n x k orthonormal basis (float64): QR of a Gaussian, diag(R) > 0."""
    g = _rng(seed, 0x0B0515).standard_normal((n, k))
    q, r = np.linalg.qr(g)
    q = q * np.sign(np.diag(r))[None, :]
    q.setflags(write=False)
    return q


@dataclasses.dataclass(frozen=True)
class FactorSpec:
    """One K-factor of a stack: dimension n, batch c = n_BS, target rank r."""
    name: str
    n: int
    c: int
    r: int
    k: int          # rank of the signal part of M
    decay: float    # s_j = decay**j
    sigma: float    # noise level
    seed: int

    def batch(self, step: int) -> np.ndarray:
        """M_step as float32, shape (n, c) (mathematical orientation)."""
        L = orthonormal_basis(self.n, self.k, self.seed)
        g = _rng(self.seed, 1, step)
        W = g.standard_normal((self.k, self.c))
        N = g.standard_normal((self.n, self.c))
        s = self.decay ** np.arange(self.k, dtype=np.float64)
        M = (L * s[None, :]) @ W + self.sigma * N
        return M.astype(np.float32)


@dataclasses.dataclass(frozen=True)
class LayerSpec:
    """One preconditioned layer: factors (A: d_A = in(+1), Gamma: d_G = out)."""
    name: str
    d_A: int
    d_G: int
    a_index: int      # index of its A factor in the stack's factor list
    g_index: int      # index of its Gamma factor
    grad_std: float
    seed: int

    def grad(self, step: int) -> np.ndarray:
        """J = Mat(g) as float32, shape (d_G, d_A) (PyTorch weight.grad layout)."""
        g = _rng(self.seed, 2, step)
        return (self.grad_std * g.standard_normal((self.d_G, self.d_A))).astype(np.float32)


@dataclasses.dataclass(frozen=True)
class StackConfig:
    name: str
    factors: Tuple[FactorSpec, ...]
    layers: Tuple[LayerSpec, ...]
    rho: float
    lam: float
    steps: int
    rsvd_every: int = 0          # 0 = never (pure B-KFAC)
    oversample: int = 10
    power_iters: int = 2


def _stack(name: str, layer_dims: Sequence[Tuple[str, int, int]], c: int, r_max: int,
           k: int, decay: float, sigma: float, rho: float, lam: float, steps: int,
           grad_std: float, rsvd_every: int = 0, oversample: int = 10,
           power_iters: int = 2) -> StackConfig:
    factors: List[FactorSpec] = []
    layers: List[LayerSpec] = []
    for li, (lname, d_A, d_G) in enumerate(layer_dims):
        ia = len(factors)
        factors.append(FactorSpec(f"{lname}.A", d_A, c, min(r_max, d_A), min(k, d_A),
                                  decay, sigma, factor_seed(ia)))
        ig = len(factors)
        factors.append(FactorSpec(f"{lname}.G", d_G, c, min(r_max, d_G), min(k, d_G),
                                  decay, sigma, factor_seed(ig)))
        layers.append(LayerSpec(lname, d_A, d_G, ia, ig, grad_std, factor_seed(10_000 + li)))
    return StackConfig(name, tuple(factors), tuple(layers), rho, lam, steps,
                       rsvd_every, oversample, power_iters)


# --- BASELINE.json configs ---------------------------------------------------

def cfg1_toy() -> StackConfig:
    """configs[0]: n=256 (A) / 128 (Gamma), n_BS=32, r=64, rho=0.95, lambda=0.1,
    20 chained steps, k=32, decay 0.9, noise 0.01; one gradient G (256x128) ~ N(0,1)
    preconditioned — read as J = G^T (128 x 256), SURVEY §8(c) G10."""
    return _stack("cfg1_toy", [("toy", 256, 128)], c=32, r_max=64, k=32, decay=0.9,
                  sigma=0.01, rho=0.95, lam=0.1, steps=20, grad_std=1.0)


def cfg2_conv() -> StackConfig:
    """configs[1]: single conv-layer A factor n=4609, n_BS=256, r=220, rho=0.95,
    k=64, decay 0.95, noise 0.05, 50 steps, RSVD (r_o=10, q=2) every 10 steps."""
    f = FactorSpec("conv.A", 4609, 256, 220, 64, 0.95, 0.05, factor_seed(0))
    return StackConfig("cfg2_conv", (f,), (), 0.95, 0.1, 50, rsvd_every=10,
                       oversample=10, power_iters=2)


VGG_CIN = (3, 64, 64, 128, 128, 256, 256, 256, 512, 512, 512, 512, 512)
VGG_COUT = (64, 64, 128, 128, 256, 256, 256, 512, 512, 512, 512, 512, 512)


def vgg16bn_layers() -> List[Tuple[str, int, int]]:
    dims = [(f"conv{i}", cin * 9 + 1, cout) for i, (cin, cout) in enumerate(zip(VGG_CIN, VGG_COUT))]
    dims += [("fc0", 513, 512), ("fc1", 513, 512), ("fc2", 513, 10)]
    return dims


def cfg3_vgg(steps: int = 20) -> StackConfig:
    """configs[2]: VGG16_bn stack, 16 layers / 32 factors, n_BS=256, r=min(220,n),
    rho=0.95, lambda=0.1, gradients ~ N(0, 1e-2)."""
    return _stack("cfg3_vgg16bn", vgg16bn_layers(), c=256, r_max=220, k=64, decay=0.95,
                  sigma=0.05, rho=0.95, lam=0.1, steps=steps, grad_std=0.1)


def cfg4_vgg_sharded(steps: int = 100) -> StackConfig:
    """configs[3]: cfg3 + dense EA maintained + RSVD overwrite every 25 steps."""
    c = cfg3_vgg(steps)
    return dataclasses.replace(c, name="cfg4_vgg16bn_rsvd", rsvd_every=25)


def cfg5_transformer(blocks: int = 24, steps: int = 50) -> StackConfig:
    """configs[4]: 24 blocks x (4097->16384, 16385->4096): 96 factors, 48 gradients,
    n_BS=1024, r=512, rho=0.97, lambda=0.01, k=256, decay 0.98, noise 0.02."""
    dims = []
    for b in range(blocks):
        dims.append((f"blk{b}.fc_in", 4097, 16384))
        dims.append((f"blk{b}.fc_out", 16385, 4096))
    return _stack("cfg5_transformer", dims, c=1024, r_max=512, k=256, decay=0.98,
                  sigma=0.02, rho=0.97, lam=0.01, steps=steps, grad_std=0.1)


def cfg5_rank_of_8() -> StackConfig:
    """One rank's share of configs[4] at 8 GPUs (layer sharding gives every rank 3 of the
    24 identical blocks): 12 factors, 6 layers -- the per-GPU work of the 8-GPU run, timed
    on one GPU to project strong scaling (the all-gather excluded)."""
    c = cfg5_transformer(blocks=3)
    return dataclasses.replace(c, name="cfg5_transformer_rank_of_8")


def cfg5_rank_of(world: int) -> StackConfig:
    """One rank's share of configs[4] at `world` GPUs (24 / world of the identical blocks)."""
    c = cfg5_transformer(blocks=24 // world)
    return dataclasses.replace(c, name=f"cfg5_transformer_rank_of_{world}")


CONFIGS = {
    "cfg1": cfg1_toy,
    "cfg2": cfg2_conv,
    "cfg3": cfg3_vgg,
    "cfg4": cfg4_vgg_sharded,
    "cfg5": cfg5_transformer,
    "cfg5r8": cfg5_rank_of_8,
    "cfg5r4": lambda: cfg5_rank_of(4),
    "cfg5r2": lambda: cfg5_rank_of(2),
}


def random_case(n: int, c: int, r: int, seed: int, k: Optional[int] = None,
                decay: float = 0.8, sigma: float = 0.05) -> FactorSpec:
    """A small factor for unit tests (same generator family)."""
    return FactorSpec(f"rand{n}x{c}r{r}", n, c, r, min(k or c, n), decay, sigma, seed)


def phantom_basis(n: int, r: int) -> np.ndarray:
    """Init basis for the first Brand step: any orthonormal n x r
    with D = 0 works; we use the first r columns of the identity."""
    U = np.zeros((n, r), dtype=np.float32)
    U[np.arange(r), np.arange(r)] = 1.0
    return U
