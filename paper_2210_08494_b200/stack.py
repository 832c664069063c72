"""Stack driver: B-KFAC / B-R-KFAC over many K-factors and layers.

Per step k (Alg 4 / Alg 5; Alg 1 lines 16-17, :401-405):
  * k == 0: Mtilde_{B,0} = M_0 M_0^T -> top-r  (alpha = 0, beta = 1, phantom basis)
  * k >= 1: if RSVD is due (k % T_RSVD == 0): (U, D) <- RSVD(Mcal_{k-1}), then
            Brand update with (alpha, beta) = (rho, 1 - rho)
  * dense EA factor Mcal_k (only when RSVD is enabled)
  * S = Gamma~^{-1} J A~^{-1} for every layer whose factors this rank owns.
Every call goes through the C ABI; this module only owns buffers and the schedule.

Multi-GPU: whole layers are assigned to ranks by greedy LPT on
n_A^3 + n_Gamma^3 (``shard_layers``); each rank updates its own factors and
preconditions its own layers; preconditioned gradients are all-gathered per slot.
"""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Tuple

from . import binding


def shard_layers(layer_costs: Sequence[float], world: int) -> List[List[int]]:
    """Greedy LPT: layers sorted by decreasing cost, each to the least-loaded rank
    (ties: lowest rank).  Deterministic; returns per-rank lists in ascending order."""
    order = sorted(range(len(layer_costs)), key=lambda i: (-layer_costs[i], i))
    loads = [0.0] * world
    owned: List[List[int]] = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda q: (loads[q], q))
        loads[r] += layer_costs[i]
        owned[r].append(i)
    return [sorted(o) for o in owned]


def layer_cost(n_A: int, n_G: int) -> float:
    return float(n_A) ** 3 + float(n_G) ** 3


LD_ALIGN = 32


def pipeline_sms(n_factors: int) -> int:
    """SMs for the pipelined preconditioning (BKFACStack.set_pipeline) of a rank that owns
    n_factors factors; 0 = unpipelined.  Pipelining pays where the Brand update leaves SMs
    idle -- few factors per GPU, whose latency-bound eigensolver kernels (one CTA or cluster
    per factor) do not fill 148 SMs; with 96 factors the Brand update fills the GPU and the
    split only slows both halves.  Measured on configs[4]: 96 factors 212 ms
    unpipelined vs 219 at 56 SMs; 48 factors 117.8 -> 109.2 (52 SMs); 24 factors 73.5 ->
    65.3 (44-48); 12 factors 41.4 -> 36.1-36.4 (42-46); the VGG stacks (32 factors) 4.67 ->
    4.54 ms (44)."""
    if n_factors > 48 or n_factors == 0:
        return 0
    return 52 if n_factors > 24 else 44


def padded(rows: int, cols: int, device, zero: bool = True):
    """A (rows, cols) float32 view of a (rows, cols rounded up to 32) buffer: the row
    stride is the operand's leading dimension (bkfac.h "Leading dimensions"), a multiple of
    32 floats, so every contraction reads it with 16-byte loads.  The padding is never read."""
    import torch
    ld = (cols + LD_ALIGN - 1) // LD_ALIGN * LD_ALIGN
    make = torch.zeros if zero else torch.empty
    return make((rows, ld), dtype=torch.float32, device=device)[:, :cols]


def full_rows(t):
    """The whole padded buffer behind a padded() view (rows x leading dimension)."""
    import torch
    return torch.as_strided(t, (t.shape[0], t.stride(0)), (t.stride(0), 1))


class BKFACStack:
    """Owns the per-factor state (ping-pong U/D buffers, optional dense EA factor) of
    the factors a rank owns and runs whole steps through the bkfac C ABI."""

    def __init__(self, factors: Sequence[Tuple[int, int, int]],
                 layers: Sequence[Tuple[int, int, int, int]],
                 rho: float, lam: float, rsvd_every: int = 0, oversample: int = 10,
                 power_iters: int = 2, precond_flags: int = 0, brand_flags: int = 0,
                 device: int = 0, rank: int = 0, world: int = 1, rsvd_seed: int = 20221015,
                 full_rank: bool = False, correct_every: int = 0, phi_crc: float = 0.5,
                 correct_seed: int = 20221016):
        """factors: (n, r, c_max) per global factor; layers: (d_G, d_A, g_index, a_index).

        full_rank=True is the paper's own preconditioner (NEXT-f1, PAPER.md:533-534,
        :655-656): every Brand step keeps all min(n, r + c) eigenpairs of M~_B and the layers
        are preconditioned with them; the next step truncates to r."""
        import torch
        self.torch = torch
        self.rho, self.lam = float(rho), float(lam)
        self.rsvd_every, self.oversample, self.power_iters = rsvd_every, oversample, power_iters
        self.precond_flags, self.brand_flags = precond_flags, brand_flags
        self.rsvd_seed = rsvd_seed
        self.device = device
        self.rank, self.world = rank, world
        self.factors = [tuple(f) for f in factors]
        self.layers = [tuple(l) for l in layers]
        costs = [layer_cost(self.factors[a][0], self.factors[g][0]) for (_, _, g, a) in self.layers]
        self.owned_layers_all = shard_layers(costs, world) if self.layers else [[] for _ in range(world)]
        self.my_layers = self.owned_layers_all[rank]
        owned_f = set()
        for li in self.my_layers:
            _, _, g, a = self.layers[li]
            owned_f.update([g, a])
        if not self.layers:   # factor-only workloads: round-robin on n^3
            fo = shard_layers([float(f[0]) ** 3 for f in self.factors], world)[rank]
            owned_f.update(fo)
        self.my_factors = sorted(owned_f)
        self.local = {g: i for i, g in enumerate(self.my_factors)}
        self.full_rank = full_rank
        # B-KFAC-C (NEXT-f3, Alg 7 :691-701): every correct_every steps, Algorithm 6 on
        # n_crc = max(1, round(phi_crc r)) random modes of every factor against the dense EA
        self.correct_every, self.phi_crc, self.correct_seed = correct_every, phi_crc, correct_seed
        if correct_every and not rsvd_every:
            raise ValueError("the light correction needs the dense EA factor (rsvd_every > 0)")
        flags = (binding.BKFAC_FACTOR_DENSE_EA if rsvd_every > 0 else 0) | \
                (binding.BKFAC_FACTOR_FULL_RANK if full_rank else 0)
        fdesc = [(self.factors[g][0], self.factors[g][1], self.factors[g][2], flags)
                 for g in self.my_factors]
        ldesc = []
        for li in self.my_layers:
            dG, dA, g, a = self.layers[li]
            # n_max: Algorithm 8 (factored gradients G = M_Gamma, A = M_A) needs both batches
            ldesc.append((dG, dA, self.rank_out(g), self.rank_out(a),
                          min(self.factors[g][2], self.factors[a][2])))
        self.ctx = binding.Context(fdesc, ldesc, device=device)
        dev = f"cuda:{device}"
        self.U = []
        self.D = []
        self.K = []
        for g in self.my_factors:
            n, r, _ = self.factors[g]
            ro = self.rank_out(g)
            self.U.append([padded(ro, n, dev) for _ in range(2)])
            self.D.append([torch.zeros((ro,), dtype=torch.float32, device=dev) for _ in range(2)])
            self.K.append(torch.zeros((n, n), dtype=torch.float32, device=dev) if rsvd_every > 0 else None)
        self.cur = [0] * len(self.my_factors)
        self.k = 0
        self.n_overwrites = 0
        self._graphs = {}
        self.last_profile_range = None
        # preconditioned gradients, two sets by step parity: step k's S stays valid while
        # step k+1 runs (a caller can read it back concurrently)
        self.S2 = [{}, {}]
        # pipelined preconditioning (set_pipeline): step k's gradients wait here and are
        # preconditioned by step k + 1's call, beside its Brand update
        self.pipe = 0
        self.prec_stream = None
        self._pend = None          # (step index, J of that step)
        for li in self.my_layers:
            dG, dA, _, _ = self.layers[li]
            for par in range(2):
                self.S2[par][li] = padded(dG, dA, dev, zero=False)

    def bind_outputs(self, by_parity: Sequence[Dict[int, "torch.Tensor"]]) -> None:
        """Precondition straight into caller buffers (e.g. SlotGather.send_views(b)): the
        S of step k goes to by_parity[k & 1][layer].  Call before any graph is captured."""
        if self._graphs:
            raise RuntimeError("bind_outputs after a CUDA graph was captured")
        for par in range(2):
            for li in self.my_layers:
                t = by_parity[par][li]
                dG, dA, _, _ = self.layers[li]
                if tuple(t.shape) != (dG, dA) or t.stride(1) != 1 or t.stride(0) < dA:
                    raise ValueError(f"output buffer of layer {li} must be a ({dG}, {dA}) tensor "
                                     "with unit stride along its rows")
                self.S2[par][li] = t

    def set_pipeline(self, prec_sms: int) -> None:
        """prec_sms > 0: pipelined steps.  The preconditioning of step k (Alg 1 lines 16-17,
        PAPER.md:401-405) needs step k's factors, so it cannot overlap step k's own Brand update;
        it does not touch step k + 1's (those are written into the other ping-pong buffer).  In
        pipelined mode step(M_k, J_k) therefore runs Brand(k) on the calling stream and the
        preconditioning of step k - 1 (J_{k-1}, the factors of step k - 1) on a second stream
        at the same time, the persistent GEMM grids split prec_sms : 148 - prec_sms SMs
        (BKFAC_OPT_GEMM_CAP), and returns S_{k-1}.  J_k must stay unchanged until the next call;
        ``flush()`` preconditions the last step.  The arithmetic of every call is unchanged,
        so each S is bitwise the S of the unpipelined schedule.  0 turns it off (call flush
        first)."""
        if prec_sms and not (2 <= prec_sms <= 146):
            raise ValueError("prec_sms must be in [2, 146]")
        if self._pend is not None:
            raise RuntimeError("set_pipeline with a preconditioning pending (call flush first)")
        if prec_sms and self.prec_stream is None:
            self.prec_stream = self.torch.cuda.Stream(device=self.device)
        if prec_sms != self.pipe:
            self._graphs = {}
        self.pipe = int(prec_sms)

    def _prec_items(self, J, k):
        items = []
        for lj, li in enumerate(self.my_layers):
            dG, dA, g, a = self.layers[li]
            UG, DG = self.state(g)
            UA, DA = self.state(a)
            items.append(dict(layer=lj, U_G=UG, D_G=DG, lambda_G=self.lam, U_A=UA, D_A=DA,
                              lambda_A=self.lam, J=J[li], S=self.S2[k & 1][li],
                              flags=self.precond_flags))
        return items

    def flush(self, stream=None) -> Dict[int, "torch.Tensor"]:
        """Pipelined mode: precondition the pending step (the last step() call's J) with the
        current factors on `stream`; returns its S ({} when nothing is pending)."""
        if self._pend is None:
            return {}
        kp, J = self._pend
        self._pend = None
        main = stream if stream is not None else self.torch.cuda.current_stream(self.device)
        self.ctx.bkfac_precondition(self._prec_items(J, kp), main)
        return {li: self.S2[kp & 1][li] for li in self.my_layers}

    # ---------------------------------------------------------------------------------
    def rank_out(self, g: int) -> int:
        n, r, c = self.factors[g]
        return min(n, r + c) if self.full_rank else r

    def state(self, g: int):
        i = self.local[g]
        return self.U[i][self.cur[i]], self.D[i][self.cur[i]]

    def set_state(self, g: int, U, D) -> None:
        i = self.local[g]
        self.U[i][self.cur[i]].copy_(U)
        self.D[i][self.cur[i]].copy_(D)

    def _phantom(self, i: int):
        U = self.U[i][self.cur[i]]
        U.zero_()
        r = self.factors[self.my_factors[i]][1]
        U[self.torch.arange(r), self.torch.arange(r)] = 1.0
        self.D[i][self.cur[i]].zero_()

    def step(self, M: Dict[int, "torch.Tensor"], J: Optional[Dict[int, "torch.Tensor"]] = None,
             stream=None, graph: bool = False, factored: bool = False,
             profile: bool = False) -> Dict[int, "torch.Tensor"]:
        """One step over the owned factors (M keyed by global factor index, each (c, n))
        and owned layers (J keyed by global layer index, each (d_G, d_A)).

        graph=True replays a CUDA graph of the step's launches (captured on first use per
        U/D ping-pong parity and input buffers -- the inputs must be the same tensors on
        every replay, refilled in place).  The initial step and RSVD-overwrite steps always
        run eagerly; the library's per-stage profiling must be off while graphs are used.

        factored=True preconditions every owned layer by Algorithm 8 (NEXT-f2,
        PAPER.md:882-930) from the factored gradient Mat(g) = G A^T with G = M[Gamma factor],
        A = M[A factor] (the same per-sample matrices as the statistics); J is not used.

        profile=True (with graph=True) replays a separate graph captured with the library's
        per-stage events on (the caller enables them with ctx.bkfac_profile_enable first):
        its event nodes are re-recorded by every replay, and ``last_profile_range`` names the
        stage records of the graph just replayed (ctx.bkfac_profile_read(rng=...))."""
        torch = self.torch
        eager = (self.rsvd_every and self.k % self.rsvd_every == 0) or \
                (self.correct_every and self.k % self.correct_every == 0)
        if graph and self.k > 0 and not eager:
            key = (self.cur[0] if self.cur else 0,
                   tuple(M[g].data_ptr() for g in self.my_factors),
                   tuple(J[li].data_ptr() for li in self.my_layers) if J is not None else None,
                   factored, profile,
                   tuple(self._pend[1][li].data_ptr() for li in self.my_layers)
                   if self._pend is not None else None)
            main = stream if stream is not None else torch.cuda.current_stream(self.device)
            hit = self._graphs.get(key)
            if hit is None:
                g = torch.cuda.CUDAGraph()
                main.synchronize()
                r0 = self.ctx.bkfac_profile_count() if profile else 0
                with torch.cuda.graph(g):
                    out = self._step(M, J, torch.cuda.current_stream(self.device), factored)
                rng = (r0, self.ctx.bkfac_profile_count()) if profile else None
                self._graphs[key] = (g, out, rng)
                self.last_profile_range = rng
                with torch.cuda.stream(main):
                    g.replay()          # capture only recorded the launches: run them
                return out
            g, out, rng = hit
            self.last_profile_range = rng
            with torch.cuda.stream(main):
                g.replay()
            if self.pipe:
                self._pend = (self.k, J)
            self.k += 1
            for i in range(len(self.my_factors)):
                self.cur[i] = 1 - self.cur[i]
            return out
        return self._step(M, J, stream, factored)

    def _step(self, M, J, stream, factored=False):
        k = self.k
        torch = self.torch
        main = stream if stream is not None else torch.cuda.current_stream(self.device)
        if self.pipe and factored:
            raise ValueError("pipelined preconditioning takes J (not the factored form)")
        pipe_out = {}
        side = False     # the pending preconditioning runs beside this step's Brand update
        if self.pipe and self._pend is not None:
            rsvd_due = self.rsvd_every and k % self.rsvd_every == 0
            if rsvd_due or self.correct_every:
                # the overwrite / correction rewrites the factors the pending step needs:
                # precondition it first, on this stream
                pipe_out = self.flush(main)
            else:
                kp, Jp = self._pend
                self._pend = None
                ps = self.prec_stream
                ps.wait_stream(main)
                self.ctx.bkfac_set_option(binding.BKFAC_OPT_GEMM_CAP, self.pipe)
                self.ctx.bkfac_precondition(self._prec_items(Jp, kp), ps)
                self.ctx.bkfac_set_option(binding.BKFAC_OPT_GEMM_CAP, 148 - self.pipe)
                pipe_out = {li: self.S2[kp & 1][li] for li in self.my_layers}
                side = True
        if k == 0:
            for i in range(len(self.my_factors)):
                self._phantom(i)
            alpha, beta = 0.0, 1.0
        else:
            alpha, beta = self.rho, 1.0 - self.rho
            if self.rsvd_every and k % self.rsvd_every == 0:
                items = []
                for i, g in enumerate(self.my_factors):
                    n_g, r_g, _ = self.factors[g]
                    # sketch width l = r + r_o is capped at n (l = n is the exact EVD)
                    items.append(dict(factor=i, K=self.K[i], oversample=min(self.oversample, n_g - r_g),
                                      power_iters=self.power_iters, seed=self.rsvd_seed + g,
                                      counter=self.n_overwrites, U_out=self.U[i][self.cur[i]],
                                      D_out=self.D[i][self.cur[i]]))
                self.ctx.bkfac_rsvd_batch(items, main)
                self.n_overwrites += 1
        ups = []
        for i, g in enumerate(self.my_factors):
            c, nx = self.cur[i], 1 - self.cur[i]
            ups.append(dict(factor=i, U_in=self.U[i][c], D_in=self.D[i][c], M=M[g],
                            U_out=self.U[i][nx], D_out=self.D[i][nx], alpha=alpha, beta=beta,
                            flags=self.brand_flags))
        if self.rsvd_every:
            # the dense EA accumulate (a8) needs only M_k and must follow this step's RSVD
            # read of Mcal_{k-1}; the library overlaps it with the Brand eigensolver
            ea = [dict(factor=i, K=self.K[i], M=M[g], rho=self.rho if k > 0 else 0.0)
                  for i, g in enumerate(self.my_factors)]
            self.ctx.bkfac_brand_ea_update(ups, ea, main)
        elif ups:
            self.ctx.bkfac_brand_update(ups, main)
        if side:
            self.ctx.bkfac_set_option(binding.BKFAC_OPT_GEMM_CAP, 0)
            main.wait_stream(self.prec_stream)
        for i in range(len(self.my_factors)):
            self.cur[i] = 1 - self.cur[i]
        if self.correct_every and k > 0 and k % self.correct_every == 0:
            # Alg 7: after this step's Brand update and EA accumulate, correct the
            # representation against Mcal_k (Algorithm 6); the random modes are drawn here
            # (seeded per factor and step) and passed to the library
            gen = torch.Generator(device="cpu")
            items = []
            for i, g in enumerate(self.my_factors):
                r = self.factors[g][1]
                ncrc = max(1, min(r, int(round(self.phi_crc * r))))
                gen.manual_seed(self.correct_seed * 1000003 + g * 7919 + k)
                idx = torch.randperm(r, generator=gen)[:ncrc].to(torch.int32).to(f"cuda:{self.device}")
                U, D = self.U[i][self.cur[i]], self.D[i][self.cur[i]]
                items.append(dict(factor=i, K=self.K[i], U=U, D=D, col_idx=idx))
            self.ctx.bkfac_light_correction(items, main)
            self._crc_keep = items          # index tensors live until the stream is past them
        out = {}
        if factored and self.my_layers:
            items = []
            for lj, li in enumerate(self.my_layers):
                dG, dA, g, a = self.layers[li]
                UG, DG = self.state(g)
                UA, DA = self.state(a)
                items.append(dict(layer=lj, U_G=UG, D_G=DG, lambda_G=self.lam, U_A=UA, D_A=DA,
                                  lambda_A=self.lam, G=M[g], A=M[a], S=self.S2[k & 1][li],
                                  flags=self.precond_flags))
            self.ctx.bkfac_precondition_factored(items, main)
            out = {li: self.S2[k & 1][li] for li in self.my_layers}
        elif self.pipe:
            out = pipe_out
            if J is not None and self.my_layers:
                self._pend = (k, J)
        elif J is not None and self.my_layers:
            self.ctx.bkfac_precondition(self._prec_items(J, k), main)
            out = {li: self.S2[k & 1][li] for li in self.my_layers}
        self.k += 1
        return out

    def check(self, stream=None):
        return self.ctx.bkfac_check(stream)

    def launches(self) -> int:
        return self.ctx.bkfac_launch_count()


class SlotGather:
    """All-gather of the preconditioned gradients: slot s holds each
    rank's s-th owned layer, packed fp32 and padded to the slot maximum; one
    ``all_gather_into_tensor`` per slot (NCCL over NVLink on the GPU box, gloo in tests).

    Double-buffered by step parity so that step k's gather overlaps step k+1's compute:
    the stack preconditions straight into the send slots (``send_views`` bound with
    ``BKFACStack.bind_outputs``), ``start(b)`` issues the slot collectives asynchronously
    (NCCL orders them after the work already on the current stream, then runs them on its
    own stream beside the next step), and ``finish(b)`` makes the current stream wait for
    them and returns every layer's S -- called before buffer set b is written again."""

    def __init__(self, layers: Sequence[Tuple[int, int, int, int]], owned: List[List[int]],
                 rank: int, device, nbuf: int = 2):
        import torch
        self.torch = torch
        self.layers = layers
        self.owned = owned
        self.rank = rank
        self.world = len(owned)
        self.nslots = max((len(o) for o in owned), default=0)
        self.slot_numel = []
        for s in range(self.nslots):
            sizes = [layers[o[s]][0] * layers[o[s]][1] if s < len(o) else 0 for o in owned]
            self.slot_numel.append(max(sizes))
        self.nbuf = nbuf
        self.send = [[torch.zeros(n, dtype=torch.float32, device=device) for n in self.slot_numel]
                     for _ in range(nbuf)]
        self.recv = [[torch.zeros(n * self.world, dtype=torch.float32, device=device)
                      for n in self.slot_numel] for _ in range(nbuf)]
        self.pending = [None] * nbuf

    def bytes_per_step(self) -> int:
        return sum(4 * n * (self.world - 1) for n in self.slot_numel)

    def send_views(self, b: int = 0) -> Dict[int, "torch.Tensor"]:
        """This rank's layers as (d_G, d_A) views of buffer set b's send slots."""
        out = {}
        for s, li in enumerate(self.owned[self.rank]):
            dG, dA = self.layers[li][0], self.layers[li][1]
            out[li] = self.send[b][s][: dG * dA].view(dG, dA)
        return out

    def start(self, b: int, S_local: Optional[Dict[int, "torch.Tensor"]] = None, group=None) -> None:
        """Issue buffer set b's slot all-gathers (async).  S_local: copied into the send slots
        first unless it already lives there (send_views)."""
        import torch.distributed as dist
        if self.pending[b] is not None:
            raise RuntimeError("SlotGather.start: buffer set still in flight (call finish first)")
        mine = self.owned[self.rank]
        if S_local is not None:
            for s, li in enumerate(mine):
                t = S_local[li].reshape(-1)
                dst = self.send[b][s]
                if t.data_ptr() != dst.data_ptr():
                    dst[: t.numel()].copy_(t)
        self.pending[b] = [dist.all_gather_into_tensor(self.recv[b][s], self.send[b][s], group=group,
                                                       async_op=True) for s in range(self.nslots)]

    def finish(self, b: int) -> Dict[int, "torch.Tensor"]:
        """Wait (stream-ordered) for buffer set b's gathers; every layer's S as views."""
        if self.pending[b] is not None:
            for w in self.pending[b]:
                w.wait()
            self.pending[b] = None
        out: Dict[int, "torch.Tensor"] = {}
        for s in range(self.nslots):
            for q in range(self.world):
                if s < len(self.owned[q]):
                    li = self.owned[q][s]
                    dG, dA = self.layers[li][0], self.layers[li][1]
                    base = q * self.slot_numel[s]
                    out[li] = self.recv[b][s][base: base + dG * dA].view(dG, dA)
        return out

    def gather(self, S_local: Dict[int, "torch.Tensor"], group=None, b: int = 0) -> Dict[int, "torch.Tensor"]:
        """Synchronous form: start + finish on buffer set b."""
        self.start(b, S_local, group)
        return self.finish(b)
