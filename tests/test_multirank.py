"""The N > 1 path on CPU: world-size-2 gloo runs of the layer sharding and
the per-slot all-gather of preconditioned gradients, with the fp64 oracle standing in for
the CUDA kernels.  Every rank must end up with every layer's S, bitwise equal to the
single-process result (per-layer inputs are seeded by global index, so sharding never
changes a result), and the max-over-ranks timing reduction must pick the slowest rank."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import synth
from paper_2210_08494_b200.stack import SlotGather, layer_cost, shard_layers

# small layers of mixed shapes (d_G, d_A, r_G, r_A): uneven sizes exercise slot padding
LAYERS = [(16, 33, 4, 6), (8, 12, 3, 2), (24, 9, 5, 4), (12, 40, 2, 8), (10, 10, 10, 3)]
LAM = 0.1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _layer_result(li):
    """Preconditioned gradient of layer li from seeded factors (oracle as the kernels)."""
    dG, dA, rG, rA = LAYERS[li]
    rng = np.random.default_rng(1000 + li)
    fa = synth.random_case(dA, 5, rA, seed=2000 + li, k=min(dA, 4))
    fg = synth.random_case(dG, 5, rG, seed=3000 + li, k=min(dG, 4))
    UA, DA = O.brand_update(synth.phantom_basis(dA, rA), np.zeros(rA), fa.batch(0), 0.0, 1.0, rA)
    UG, DG = O.brand_update(synth.phantom_basis(dG, rG), np.zeros(rG), fg.batch(0), 0.0, 1.0, rG)
    J = rng.standard_normal((dG, dA))
    return O.precondition(J, UG, DG, LAM, UA, DA, LAM).astype(np.float32)


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        layers = [(dG, dA, 2 * i, 2 * i + 1) for i, (dG, dA, _, _) in enumerate(LAYERS)]
        costs = [layer_cost(dA, dG) for (dG, dA, _, _) in LAYERS]
        owned = shard_layers(costs, world)
        mine = {li: torch.from_numpy(_layer_result(li)) for li in owned[rank]}
        gather = SlotGather(layers, owned, rank, "cpu")
        full = gather.gather(mine)
        # max over ranks of a per-rank "elapsed time" (bench.py's reduction)
        t = torch.tensor([float(rank + 1) * 1.5], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out_q.put((rank, {li: v.numpy().copy() for li, v in full.items()}, float(t[0]),
                   gather.bytes_per_step()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_slot_allgather_bitwise_equal_to_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = {li: _layer_result(li) for li in range(len(LAYERS))}
    for rank, full, tmax, nbytes in results:
        assert sorted(full) == list(range(len(LAYERS))), f"rank {rank} misses layers"
        for li, S in full.items():
            assert S.shape == ref[li].shape
            assert np.array_equal(S, ref[li]), f"rank {rank} layer {li} differs"
        assert tmax == 1.5 * world                     # max over ranks, not the mean
        assert nbytes > 0


def test_sharding_covers_every_layer_once_and_is_deterministic():
    costs = [layer_cost(dA, dG) for (dG, dA, _, _) in LAYERS]
    for world in (1, 2, 3, 4):
        owned = shard_layers(costs, world)
        assert owned == shard_layers(costs, world)
        assert sorted(sum(owned, [])) == list(range(len(LAYERS)))


def _worker_overlap(rank, world, port, out_q):
    """The overlapped form bench.py uses: outputs bound to the double-buffered send slots,
    step k's gather started asynchronously and finished only before buffer set k & 1 is
    written again (two steps later) or at the end."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        layers = [(dG, dA, 2 * i, 2 * i + 1) for i, (dG, dA, _, _) in enumerate(LAYERS)]
        costs = [layer_cost(dA, dG) for (dG, dA, _, _) in LAYERS]
        owned = shard_layers(costs, world)
        gather = SlotGather(layers, owned, rank, "cpu")
        views = [gather.send_views(0), gather.send_views(1)]
        base = {li: torch.from_numpy(_layer_result(li)) for li in owned[rank]}
        results = []
        for k in range(4):
            b = k & 1
            if k >= 2:
                results.append({li: v.numpy().copy() for li, v in gather.finish(b).items()})
            for li in owned[rank]:           # "precondition straight into the send slot"
                views[b][li].copy_(base[li] * float(k + 1))
            gather.start(b)
        for b in (0, 1):
            results.append({li: v.numpy().copy() for li, v in gather.finish(b).items()})
        out_q.put((rank, results))
    finally:
        dist.destroy_process_group()


def test_slot_allgather_overlapped_double_buffer():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_overlap, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = {li: _layer_result(li) for li in range(len(LAYERS))}
    for rank, steps in results:
        assert len(steps) == 4
        for k, full in enumerate(steps):          # finished in step order 0, 1, 2, 3
            assert sorted(full) == list(range(len(LAYERS)))
            for li, S in full.items():
                assert np.array_equal(S, ref[li] * np.float32(k + 1)), (rank, k, li)


def test_pipeline_policy_per_rank_share():
    """stack.pipeline_sms: pipelined preconditioning only where the rank's Brand update leaves
    SMs idle (<= 48 factors); the cap leaves room for the Brand side (148 - P >= 96 SMs: the
    12 eight-CTA clusters of an 8-GPU rank's one-stage reduction)."""
    from paper_2210_08494_b200 import pipeline_sms
    assert pipeline_sms(96) == 0          # configs[4] on one GPU
    assert pipeline_sms(0) == 0
    assert pipeline_sms(48) == 52         # 2 GPUs
    assert pipeline_sms(24) == 44 and pipeline_sms(12) == 44
    for nf in range(1, 200):
        p = pipeline_sms(nf)
        assert p == 0 or (2 <= p and 148 - p >= 96)
