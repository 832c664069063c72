"""Input generators: deterministic, right shapes, fp32 (CPU)."""
import numpy as np

import synth


def test_generator_deterministic_and_fp32():
    f = synth.random_case(300, 16, 8, seed=5, k=12)
    a, b = f.batch(3), f.batch(3)
    assert a.dtype == np.float32 and a.shape == (300, 16)
    assert np.array_equal(a, b)
    assert not np.array_equal(a, f.batch(4))


def test_basis_orthonormal():
    L = synth.orthonormal_basis(200, 30, 77)
    assert np.abs(L.T @ L - np.eye(30)).max() < 1e-13


def test_configs_shapes():
    c3 = synth.cfg3_vgg()
    assert len(c3.factors) == 32 and len(c3.layers) == 16
    brand = [f for f in c3.factors if f.r + f.c < f.n]
    assert len(brand) == 23          # 23 Brand + 9 dense-path factors
    c5 = synth.cfg5_transformer()
    assert len(c5.factors) == 96 and len(c5.layers) == 48
    assert sorted({f.n for f in c5.factors}) == [4096, 4097, 16384, 16385]
    c1 = synth.cfg1_toy()
    assert [f.n for f in c1.factors] == [256, 128]
    assert (c1.layers[0].d_G, c1.layers[0].d_A) == (128, 256)


def test_rank_of_8_is_one_rank_share_of_cfg5():
    """cfg5r8 = what layer sharding gives one of 8 ranks of configs[4] (the per-rank
    projection of DESIGN.md section 8)."""
    from paper_2210_08494_b200.stack import layer_cost, shard_layers
    c5, r8 = synth.cfg5_transformer(), synth.cfg5_rank_of_8()
    assert len(r8.factors) == 12 and len(r8.layers) == 6
    costs = [layer_cost(c5.factors[L.a_index].n, c5.factors[L.g_index].n) for L in c5.layers]
    shards = shard_layers(costs, 8)
    assert sorted(len(s) for s in shards) == [6] * 8
    mine = sorted((c5.layers[i].d_G, c5.layers[i].d_A) for i in shards[0])
    assert mine == sorted((L.d_G, L.d_A) for L in r8.layers)

