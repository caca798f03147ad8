"""Expert-parallel MoE forward: one process per GPU.

Tokens are data-parallel (each rank routes its own tokens); experts are
placed per layer. The reference only *plans* residency (placement.py:125-176,
evaluate_plan :179-208) for a single device; here the plan's residents become
experts REPLICATED on every rank (always served locally, no traffic) and the
remaining experts are placed by load (``ExpertPlacement.balanced``: a hot
expert may be split over several ranks, each serving a fixed set of source
ranks), so ``evaluate_plan``'s hit rate is the fraction of activations that
never leave their home GPU.

Two transports share the routing front end (K3 router, route keys =
destination * E + expert, one counting sort over W*E keys) and the per-row
arithmetic of the single-GPU layer, so every EP forward is bit-identical to
``MoELayer.forward`` on the same tokens (tests/test_gpu_ep.py):

* ``PeerExpertParallelMoE`` (default) — fused dispatch / combine over peer
  memory with a device-side exchange plan: the routing offsets of all ranks
  are all-gathered on the device, ``moe_ep_peer_plan`` lays out every send
  base, receive block and grouped-GEMM offset, K1 writes each row straight
  into its owner's receive buffer, the owner's GEMM2 epilogue writes each
  output row straight into the home rank's buffer, the home rank combines.
  No host round trip inside a forward.
* ``ExpertParallelMoE`` — the NCCL baseline: counts all-to-all, codes /
  sidecar all_to_all_v, receiver regroup, grouped GEMMs, bf16 rows back.

The compute is behind a small backend interface (``CudaExpertBackend`` is the
product; tests plug a float64 CPU backend into the same runtime to check the
host logic and the gloo exchange at world size 2). ``ExpertParallelStack``
runs the 32-layer token path on top of either transport.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from . import ops
from .placement import PlacementPlan
from .trace import ExpertFreq


# ── placement ─────────────────────────────────────────────────────────────
@dataclass(frozen=True)
class ExpertPlacement:
    """Where each expert of one layer lives in a world of ``world`` ranks.

    replicated: experts held by every rank (served where the token is).
    owner[e]:   rank holding non-replicated expert e (its primary holder
                when the expert is split), -1 for replicated experts.
    routes:     optional [W][E] table: routes[s][e] = the rank that serves
                expert e for the tokens of source rank s. Empty = every
                source sends expert e to owner[e]. A sharded expert may be
                split over several ranks this way (``balanced``); the ranks
                appearing in its column are its holders.
    """
    world: int
    experts: int
    replicated: tuple
    owner: tuple
    routes: tuple = ()

    def __post_init__(self):
        if self.world < 1 or self.experts < 1:
            raise ValueError("world and experts must be >= 1")
        if len(self.owner) != self.experts:
            raise ValueError(f"owner has {len(self.owner)} entries for {self.experts} experts")
        rep = set(self.replicated)
        for e, o in enumerate(self.owner):
            if e in rep:
                if o != -1:
                    raise ValueError(f"replicated expert {e} must have owner -1")
            elif not 0 <= o < self.world:
                raise ValueError(f"expert {e} has owner {o} outside [0, {self.world})")
        if any(not 0 <= e < self.experts for e in rep):
            raise ValueError("replicated expert id out of range")
        if self.routes:
            if len(self.routes) != self.world or any(len(r) != self.experts for r in self.routes):
                raise ValueError("routes must be [world][experts]")
            for s_, row in enumerate(self.routes):
                for e, d in enumerate(row):
                    if e in rep and d != s_:
                        raise ValueError(f"replicated expert {e}: source {s_} must route to itself")
                    if not 0 <= d < self.world:
                        raise ValueError(f"route ({s_}, {e}) -> {d} outside the world")
            for e in range(self.experts):
                if e not in rep and self.owner[e] not in self.holders(e):
                    raise ValueError(f"expert {e}: owner {self.owner[e]} serves no source")

    @classmethod
    def sharded(cls, experts: int, world: int) -> "ExpertPlacement":
        """Contiguous blocks, no replication (expert e -> rank e * W // E)."""
        return cls(world, experts, (), tuple(e * world // experts for e in range(experts)))

    @classmethod
    def from_counts(cls, counts, world: int, replicated=()) -> "ExpertPlacement":
        """Greedy bin-packing of the non-replicated experts by routed-token
        counts: hottest first (ties -> lower id) onto the least-loaded rank
        (ties -> lower rank). Replicated experts load every rank equally
        (each serves its own tokens), so they do not enter the packing."""
        counts = np.asarray(counts, dtype=np.int64).reshape(-1)
        E = counts.size
        rep = tuple(sorted(set(int(e) for e in replicated)))
        owner = [-1] * E
        load = np.zeros(world, dtype=np.int64)
        order = np.lexsort((np.arange(E), -counts))
        for e in order:
            e = int(e)
            if e in rep:
                continue
            r = int(np.argmin(load))          # first minimum -> lowest rank on ties
            owner[e] = r
            load[r] += counts[e]
        return cls(world, E, rep, tuple(owner))

    @classmethod
    def balanced(cls, counts, world: int, replicated=(), per_source=None) -> "ExpertPlacement":
        """Load-split placement for few experts per rank (E <= W, e.g.
        Mixtral's 8 experts on 8 GPUs, where one rank per expert makes the
        hottest expert's rank the straggler). The unit of assignment is one
        source rank's rows for one expert (``per_source[s][e]``, default
        counts[e] / W). Non-replicated experts, hottest first (ties -> lower
        id), are laid end to end and cut into W consecutive runs of about
        the average load (McNaughton's wrap-around rule, quantised to whole
        units: a unit goes to the rank whose slot [r, r + 1) x average holds
        the unit's centre). So each rank's sharded load is the average within
        one unit and at most W - 1 experts are split.
        Inside a split expert every holder takes its own source's unit
        first (served locally), the remaining sources go in ascending order.
        Replicated experts serve their own tokens everywhere (equal load)."""
        counts = np.asarray(counts, dtype=np.float64).reshape(-1)
        E = counts.size
        ps = (np.tile(counts / world, (world, 1)) if per_source is None
              else np.asarray(per_source, dtype=np.float64).reshape(world, E))
        rep = tuple(sorted(set(int(e) for e in replicated)))
        nonrep = [int(e) for e in np.lexsort((np.arange(E), -counts)) if int(e) not in rep]
        target = ps[:, nonrep].sum() / world if nonrep else 0.0
        routes = [[s_ if e in rep else -1 for e in range(E)] for s_ in range(world)]
        owner = [-1] * E
        cum = 0.0
        for e in nonrep:
            n_units = {}                                   # rank -> number of e's units it serves
            for s_ in sorted(range(world), key=lambda s_: -ps[s_, e]):
                u = ps[s_, e]
                # the unit goes to the rank whose cumulative slot holds its centre
                r = min(world - 1, int((cum + 0.5 * u) // target)) if target > 0 else 0
                n_units[r] = n_units.get(r, 0) + 1
                cum += u
            # which sources each holder serves: own source first, then ascending
            free = [s_ for s_ in range(world) if s_ not in n_units]
            need = dict(n_units)
            for h in n_units:
                routes[h][e] = h
                need[h] -= 1
            for h in sorted(n_units):
                while need[h] > 0:
                    routes[free.pop(0)][e] = h
                    need[h] -= 1
            owner[e] = max(n_units, key=lambda h: (n_units[h], -h))
        split = cls(world, E, rep, tuple(owner), tuple(tuple(row) for row in routes))
        # whole experts may already balance (e.g. many experts per rank):
        # keep the unsplit packing unless splitting lowers the busiest rank
        whole = cls.from_counts(counts, world, rep)
        def peak(pl):
            return np.bincount(pl.dest_table_all().ravel(), weights=ps.ravel(), minlength=world).max()
        return split if peak(split) < peak(whole) * (1 - 1e-9) else whole

    def dest_table_all(self) -> np.ndarray:
        """[W, E]: dest_table of every source rank."""
        return np.stack([self.dest_table(r) for r in range(self.world)])

    @classmethod
    def from_plan(cls, plan: PlacementPlan, layer: int, freq: ExpertFreq, world: int,
                  balance: bool = True) -> "ExpertPlacement":
        """Residents of ``plan`` (plan_two_stage / plan_frequency / plan_path)
        at ``layer`` are replicated; the rest are placed on freq counts
        (``balanced`` load split, or ``from_counts`` one rank each)."""
        build = cls.balanced if balance else cls.from_counts
        return build(freq.counts[layer], world, plan.residents[layer])

    def dest_table(self, rank: int) -> np.ndarray:
        """dest[e] = the rank that serves expert e for tokens of ``rank``."""
        if self.routes:
            return np.asarray(self.routes[rank], dtype=np.int32)
        return np.array([rank if o == -1 else o for o in self.owner], dtype=np.int32)

    def holders(self, e: int) -> tuple:
        """Ranks holding expert e's weights (every rank if replicated)."""
        if self.owner[e] == -1:
            return tuple(range(self.world))
        if self.routes:
            return tuple(sorted({row[e] for row in self.routes}))
        return (self.owner[e],)

    def local_experts(self, rank: int) -> tuple:
        return tuple(e for e in range(self.experts) if rank in self.holders(e))

    def local_fraction(self, counts) -> float:
        """Fraction of activations served without leaving the home rank, for
        tokens spread evenly over ranks (each source holds 1/W of expert e's
        activations; they stay local when the source serves e itself)."""
        counts = np.asarray(counts, dtype=np.float64).reshape(-1)
        tot = counts.sum()
        if tot == 0:
            return 1.0
        local = sum(counts[e] / self.world for s_ in range(self.world)
                    for e, d in enumerate(self.dest_table(s_)) if d == s_)
        return float(local / tot)

    def rank_loads(self, counts) -> np.ndarray:
        """Predicted rows each rank computes per forward, for global routed
        counts ``counts`` [E] with tokens spread evenly over the ranks."""
        counts = np.asarray(counts, dtype=np.float64).reshape(-1)
        load = np.zeros(self.world)
        for s_ in range(self.world):
            for e, d in enumerate(self.dest_table(s_)):
                load[d] += counts[e] / self.world
        return load


# ── exchange ──────────────────────────────────────────────────────────────
class TorchDistExchange:
    """all_to_all over a torch.distributed process group (NCCL on GPUs, gloo
    on CPU). world == 1 without an initialised group is the identity."""

    def __init__(self, group=None):
        self.group = group
        self.dist = torch.distributed if torch.distributed.is_initialized() else None
        self.world = self.dist.get_world_size(group) if self.dist else 1
        self.rank = self.dist.get_rank(group) if self.dist else 0

    def counts(self, send: np.ndarray) -> np.ndarray:
        """send [W, E] (rows this rank sends to each rank, per expert) ->
        recv [W, E] (rows each rank sends to this one)."""
        if self.world == 1:
            return send.copy()
        dev = "cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu"
        s = torch.as_tensor(send, dtype=torch.int64, device=dev).contiguous()
        r = torch.empty_like(s)
        self.dist.all_to_all_single(r, s, group=self.group)
        return r.cpu().numpy()

    def rows(self, t: torch.Tensor, send_splits: list, recv_splits: list) -> torch.Tensor:
        if self.world == 1:
            return t
        out = t.new_empty((int(sum(recv_splits)),) + tuple(t.shape[1:]))
        self.dist.all_to_all_single(out, t.contiguous(), [int(v) for v in recv_splits],
                                    [int(v) for v in send_splits], group=self.group)
        return out


def regroup_index(recv_counts: np.ndarray, local: tuple) -> tuple[np.ndarray, np.ndarray]:
    """Received rows arrive source-major, expert-sorted within each source
    block. Returns the gather index that makes them expert-contiguous (local
    experts ascending, sources ascending within an expert) and the per-local-
    expert row counts."""
    recv_counts = np.asarray(recv_counts, dtype=np.int64)
    W, E = recv_counts.shape
    stray = np.ones(E, dtype=bool)
    stray[list(local)] = False
    if recv_counts[:, stray].any():
        raise RuntimeError("received rows for an expert this rank does not hold (placement mismatch)")
    block = np.concatenate([[0], np.cumsum(recv_counts.sum(axis=1))])
    start = block[:-1, None] + np.concatenate([np.zeros((W, 1), np.int64), np.cumsum(recv_counts, axis=1)[:, :-1]],
                                              axis=1)
    pieces = [np.arange(start[s, e], start[s, e] + recv_counts[s, e]) for e in local for s in range(W)]
    index = np.concatenate(pieces).astype(np.int32) if pieces else np.zeros(0, np.int32)
    return index, recv_counts[:, list(local)].sum(axis=0)


@dataclass
class DispatchState:
    T: int
    perm: dict
    payload: list
    send_counts: np.ndarray          # [W, E]
    send_splits: list = field(default_factory=list)


class ExpertParallelMoE:
    """One rank's view of an expert-parallel MoE layer."""

    def __init__(self, backend, placement: ExpertPlacement, exchange=None, rank: int | None = None):
        self.be = backend
        self.pl = placement
        self.ex = exchange if exchange is not None else TorchDistExchange()
        self.rank = self.ex.rank if rank is None else rank
        if getattr(self.ex, "world", placement.world) != placement.world:
            raise ValueError(f"placement is for {placement.world} ranks, the group has {self.ex.world}")
        self.local = placement.local_experts(self.rank)
        if tuple(backend.local_experts) != self.local:
            raise ValueError(f"backend holds experts {backend.local_experts}, placement gives {self.local}")
        self.dest = backend.to_index_tensor(placement.dest_table(self.rank))

    def migrate(self, placement: ExpertPlacement) -> None:
        """Re-placement step of the statistics loop: adopt a new placement
        (e.g. from fresh routing statistics). This rank uploads the weights of
        the experts it now holds from the layer spec and drops the others."""
        if placement.world != self.pl.world or placement.experts != self.pl.experts:
            raise ValueError("placement shape changed")
        self.pl = placement
        self.local = placement.local_experts(self.rank)
        self.be = self.be.with_local_experts(self.local)
        self.dest = self.be.to_index_tensor(placement.dest_table(self.rank))

    # phases (kept separate so a single process can drive several ranks: run_loopback)
    def dispatch(self, x: torch.Tensor) -> DispatchState:
        W, E = self.pl.world, self.pl.experts
        T = x.shape[0]
        idx, w = self.be.route(x)
        keys = self.be.route_keys(idx, self.dest, E)
        perm = self.be.permute(keys, w, W * E)
        payload = self.be.quantize_pack(x, perm, E)
        off = self.be.to_host(perm["offsets"]).astype(np.int64)
        send_counts = np.diff(off).reshape(W, E)
        return DispatchState(T, perm, payload, send_counts, send_counts.sum(axis=1).tolist())

    def compute(self, recv_payload: list, recv_counts: np.ndarray, mark=None) -> torch.Tensor:
        index, group_counts = regroup_index(recv_counts, self.local)
        return self.be.experts(recv_payload, index, group_counts, mark or (lambda _n: None))

    def finish(self, st: DispatchState, y_home: torch.Tensor, out=None) -> torch.Tensor:
        return self.be.combine(y_home, st.perm, st.T, out=out)

    def forward(self, x: torch.Tensor, timer=None, out: torch.Tensor | None = None) -> torch.Tensor:
        """x [T, d] on this rank's device -> [T, d]. ``timer`` (optional) gets
        ``mark(stage)`` calls between phases (CUDA events)."""
        mark = timer.mark if timer is not None else (lambda _n: None)
        mark("start")
        st = self.dispatch(x)
        mark("dispatch_prepare")
        recv_counts = self.ex.counts(st.send_counts)
        recv_splits = recv_counts.sum(axis=1).tolist()
        recv = [self.ex.rows(p, st.send_splits, recv_splits) for p in st.payload]
        mark("all_to_all_dispatch")
        y_recv = self.compute(recv, recv_counts, mark)
        y_home = self.ex.rows(y_recv, recv_splits, st.send_splits)
        mark("all_to_all_combine")
        y = self.finish(st, y_home, out)
        mark("combine")
        return y

    __call__ = forward

    def forward_host_stream(self, batches: list, depth: int = 2) -> list:
        """Serving loop over host batches (hostio.stream_batches). The NCCL
        transport's split sizes come back to the host every forward, so this
        pipelines only the copies, not the host round trips."""
        from .hostio import stream_batches
        return stream_batches(self, self.forward, self.be.d, self.be.out_dtype, batches, depth, split_ends=4)

    def forward_host(self, x_host: torch.Tensor, out_host: torch.Tensor | None = None) -> torch.Tensor:
        """Pinned host tokens in, host tokens out (the end-to-end call)."""
        x = x_host.to(self.be.device, non_blocking=True)
        y = self.forward(x)
        if out_host is None:
            out_host = torch.empty(tuple(y.shape), dtype=y.dtype, pin_memory=True)
        out_host.copy_(y, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return out_host


def _gather_offsets(ex, offsets: torch.Tensor) -> torch.Tensor:
    """Every rank's route_permute offsets [W*E+1] -> [W, W*E+1] on the
    device (one small all-gather; no host round trip)."""
    if getattr(ex, "world", 1) == 1 or ex.dist is None:
        return offsets.reshape(1, -1)
    out = torch.empty((ex.world, offsets.numel()), dtype=offsets.dtype, device=offsets.device)
    ex.dist.all_gather_into_tensor(out, offsets.contiguous(), group=ex.group)
    return out


class PeerExpertParallelMoE(ExpertParallelMoE):
    """Expert-parallel forward over peer memory (no bulk NCCL traffic and no
    host round trip): the routing offsets of all ranks are all-gathered on
    the device, one small kernel (``moe_ep_peer_plan``) derives every send
    base, receive block and grouped-GEMM offset from them, K1 writes each
    dispatched row straight into its owner's receive buffer (already
    expert-contiguous, so no regroup), the owner's GEMM2 epilogue writes
    each output row straight into the home rank's ``yhome`` slot, and the
    home rank combines locally. The receiver's row count stays on the device
    (the K1 and GEMM launches are sized for the buffer capacity and read it),
    so the host never waits inside a forward; per forward: one all-gather of
    W*E+1 ints and two device-side cross-rank barriers.

    A plan that would overflow a receive / home buffer (or route rows to a
    rank that does not hold the expert) is refused on the device by every
    rank alike: nothing is written to peer memory, and the refusal is raised
    as ``RuntimeError`` by ``check()`` — at the latest by the next forward,
    and by ``forward_host`` / ``forward_host_stream`` right away."""

    def __init__(self, backend, placement: ExpertPlacement, buffers: PeerBuffers, exchange=None,
                 rank: int | None = None):
        super().__init__(backend, placement, exchange, rank)
        if getattr(backend, "d", 0) % 16 or getattr(backend, "d", 0) < 128:
            raise ValueError("the peer transport needs d % 16 == 0 and d >= 128 (fused K1 records)")
        self.bufs = buffers
        W, E = placement.world, placement.experts
        self._rank_of = backend.to_index_tensor(np.repeat(np.arange(W, dtype=np.int32), E))
        self._local_t = backend.to_index_tensor(np.asarray(self.local, dtype=np.int32))
        self._flags = []             # (event, pinned valid flag) of forwards not checked yet
        self._flag_ring, self._flag_next = None, 0

    _RING = 64

    def migrate(self, placement: ExpertPlacement) -> None:
        super().migrate(placement)
        self._local_t = self.be.to_index_tensor(np.asarray(self.local, dtype=np.int32))

    # phases (separate so one process can drive several ranks: run_loopback_peer)
    def peer_prepare(self, x):
        W, E = self.pl.world, self.pl.experts
        idx, w = self.be.route(x)
        keys = self.be.route_keys(idx, self.dest, E)
        perm = self.be.permute(keys, w, W * E)
        return DispatchState(x.shape[0], perm, [x], None)

    def peer_plan(self, offsets_all: torch.Tensor) -> torch.Tensor:
        # the plan kernel also stores its valid flag into a pinned ring slot
        # through the host mapping (no allocation, no copy-engine transfer
        # queued behind other streams' bulk D2H copies)
        if self._flag_ring is None:
            self._flag_ring = torch.empty(self._RING, dtype=torch.int32, pin_memory=True)
        slot = self._flag_ring[self._flag_next % self._RING: self._flag_next % self._RING + 1]
        self._flag_next += 1
        if len(self._flags) >= self._RING:        # ring full: retire the oldest entry first
            self.check(wait=True)
        plan = ops.ep_peer_plan(offsets_all, self.rank, self._local_t, self.bufs.codes.shape[0],
                                self.bufs.yhome.shape[0], host_flag=slot)
        ev = torch.cuda.Event()
        ev.record()
        self._flags.append((ev, slot))
        return plan

    def check(self, wait: bool = False) -> None:
        """Raise if an earlier forward's exchange plan was refused (buffer
        overflow / placement mismatch). Non-blocking unless ``wait``."""
        keep = []
        for ev, flag in self._flags:
            if wait:
                ev.synchronize()
            if ev.query():
                if int(flag[0]) == 0:
                    self._flags = []
                    raise RuntimeError(
                        "expert-parallel exchange refused: a receive buffer (PeerBuffers cap "
                        f"{self.bufs.codes.shape[0]} rows) or home buffer ({self.bufs.yhome.shape[0]} rows) "
                        "would overflow, or rows were routed to a rank that does not hold the expert")
            else:
                keep.append((ev, flag))
        self._flags = keep

    def peer_send(self, st: DispatchState, plan: torch.Tensor):
        W, E, G = self.pl.world, self.pl.experts, len(self.local)
        v = ops.plan_views(plan, W, E, G)
        n = st.perm["src_token"].numel()
        if n == 0:
            return
        dst_rank, dst_row = ops.block_map(n, st.perm["offsets"], self._rank_of, v["send_base"], valid=v["valid"])
        self.be.dispatch_send(st.payload[0], st.perm, E, self.bufs, dst_rank, dst_row)

    def peer_compute(self, plan: torch.Tensor, mark=None):
        W, E, G = self.pl.world, self.pl.experts, len(self.local)
        if G == 0:
            return
        v = ops.plan_views(plan, W, E, G)
        cap = self.bufs.codes.shape[0]
        out_rank, out_row, row_group = ops.block_map(cap, v["starts"], v["ranks"], v["homes"], val2=v["group"],
                                                     n_dev=v["R"], nblocks=G * W)
        self.be.experts_peer_dev(self.bufs, v["R"], v["goff"], row_group, out_rank, out_row,
                                 mark or (lambda _n: None))

    def peer_finish(self, st: DispatchState, out=None):
        return self.be.combine(self.bufs.yhome[: st.perm["src_token"].numel()], st.perm, st.T, out=out)

    def forward(self, x: torch.Tensor, timer=None, out: torch.Tensor | None = None) -> torch.Tensor:
        self.check()
        mark = timer.mark if timer is not None else (lambda _n: None)
        mark("start")
        st = self.peer_prepare(x)
        plan = self.peer_plan(_gather_offsets(self.ex, st.perm["offsets"]))
        mark("dispatch_prepare")
        self.peer_send(st, plan)
        self.bufs.barrier()
        mark("dispatch_k1_peer")
        self.peer_compute(plan, mark)
        self.bufs.barrier()
        mark("gemm2_peer_barrier")
        y = self.peer_finish(st, out)
        mark("combine")
        return y

    __call__ = forward

    def forward_host(self, x_host: torch.Tensor, out_host: torch.Tensor | None = None) -> torch.Tensor:
        out = super().forward_host(x_host, out_host)
        self.check(wait=True)
        return out

    def forward_host_stream(self, batches: list, depth: int = 2) -> list:
        """Serving loop over host batches (hostio.stream_batches): the H2D of
        batch b+1 and the D2H of batch b-1 overlap batch b's EP forward."""
        from .hostio import stream_batches
        outs = stream_batches(self, self.forward, self.be.d, self.be.out_dtype, batches, depth, split_ends=4)
        self.check(wait=True)
        return outs


def run_loopback_peer(ranks: list, xs: list) -> list:
    """``run_loopback`` for the peer transport: the offsets of all ranks are
    stacked (the all-gather), every rank's plan kernel runs, every rank's K1
    writes into the other ranks' buffers, then every rank's experts write
    their outputs into the home ranks' buffers, then every rank combines."""
    sts = [m.peer_prepare(x) for m, x in zip(ranks, xs)]
    offs = torch.stack([st.perm["offsets"] for st in sts])
    plans = [m.peer_plan(offs) for m in ranks]
    for m, st, pl in zip(ranks, sts, plans):
        m.peer_send(st, pl)
    for m, pl in zip(ranks, plans):
        m.peer_compute(pl)
    outs = [m.peer_finish(st) for m, st in zip(ranks, sts)]
    for m in ranks:
        m.check(wait=True)
    return outs


def run_loopback(ranks: list, xs: list) -> list:
    """Drive W ``ExpertParallelMoE`` instances (one per simulated rank) in one
    process, performing the two all-to-all exchanges by concatenation. Used
    to exercise the multi-rank data layout (several sources per receiver,
    remote experts) on a single device; the kernels are the same, only the
    transport differs. Ranks run one after another, nothing waits on a peer."""
    W = len(ranks)
    sts = [m.dispatch(x) for m, x in zip(ranks, xs)]
    parts = [[list(torch.split(p, s.send_splits)) for p in s.payload] for s in sts]
    y_parts = []
    for r, m in enumerate(ranks):
        recv_counts = np.stack([sts[s].send_counts[r] for s in range(W)])
        recv = [torch.cat([parts[s][i][r] for s in range(W)]) for i in range(len(sts[0].payload))]
        y = m.compute(recv, recv_counts)
        y_parts.append(list(torch.split(y, recv_counts.sum(axis=1).tolist())))
    return [ranks[s].finish(sts[s], torch.cat([y_parts[r][s] for r in range(W)])) for s in range(W)]


# ── fused transport: peer memory instead of an all-to-all ────────────────
class PeerBuffers:
    """One rank's receive and return buffers, addressable by every rank of
    the EP group: ``codes`` [cap, d] u8 and ``params`` [cap, 4] int32 (the
    dispatched rows, written by the senders' K1), ``yhome`` [cap_home, d]
    bf16 (this rank's tokens' expert outputs, written by the owners' GEMM2
    epilogue), plus device tables of all ranks' base pointers.

    ``symmetric`` allocates through torch symmetric memory (NVLink peer
    mappings, one process per GPU); ``loopback`` builds W ranks' buffers in
    one process on one device (tests / single-GPU emulation: same kernels,
    the peers are just other buffers)."""

    def __init__(self, rank: int, world: int, codes, params, yhome, tabs, barrier=None):
        self.rank, self.world = rank, world
        self.codes, self.params, self.yhome = codes, params, yhome
        self.codes_tab, self.params_tab, self.y_tab = tabs
        self._barrier = barrier

    def barrier(self):
        if self._barrier is not None:
            self._barrier()

    @staticmethod
    def _tab(ptrs, device):
        return torch.tensor([int(p) for p in ptrs], dtype=torch.int64, device=device)

    @classmethod
    def symmetric(cls, d: int, cap: int, cap_home: int, group=None) -> "PeerBuffers":
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        group = group or dist.group.WORLD
        dev = torch.device("cuda", torch.cuda.current_device())
        codes = symm_mem.empty(cap, d, dtype=torch.uint8, device=dev)
        params = symm_mem.empty(cap, 4, dtype=torch.int32, device=dev)
        yhome = symm_mem.empty(cap_home, d, dtype=torch.bfloat16, device=dev)
        hs = [symm_mem.rendezvous(t, group) for t in (codes, params, yhome)]
        tabs = tuple(cls._tab(h.buffer_ptrs, dev) for h in hs)
        return cls(dist.get_rank(group), dist.get_world_size(group), codes, params, yhome, tabs,
                   barrier=lambda: hs[0].barrier(channel=0))

    @classmethod
    def loopback(cls, world: int, d: int, cap: int, cap_home: int, device="cuda") -> list:
        bufs = [(torch.empty((cap, d), dtype=torch.uint8, device=device),
                 torch.empty((cap, 4), dtype=torch.int32, device=device),
                 torch.empty((cap_home, d), dtype=torch.bfloat16, device=device)) for _ in range(world)]
        tabs = tuple(cls._tab([b[i].data_ptr() for b in bufs], device) for i in range(3))
        return [cls(r, world, *bufs[r], tabs) for r in range(world)]


def peer_send_layout(C: np.ndarray, me: int, placement: ExpertPlacement) -> tuple[np.ndarray, np.ndarray]:
    """Host restatement of the send half of ``moe_ep_peer_plan`` (the device
    plan the forward uses; tests compare the two). Sender side. C[s, r, e] =
    rows rank s sends to rank r for expert e.
    Rank r's receive buffer is expert-major (its local experts ascending),
    sender-minor. Returns per sort key (r, e) (r-major): destination rank and
    the first receive-buffer row of this sender's block."""
    W, _, E = C.shape
    rank_of = np.repeat(np.arange(W, dtype=np.int32), E)
    base = np.zeros(W * E, dtype=np.int64)
    for r in range(W):
        off = 0
        for e in placement.local_experts(r):
            base[r * E + e] = off + C[:me, r, e].sum()
            off += C[:, r, e].sum()
    return rank_of, base.astype(np.int32)


def peer_recv_layout(C: np.ndarray, me: int, local: tuple) -> tuple:
    """Host restatement of the receive half of ``moe_ep_peer_plan``.
    Receiver side: block starts of the (expert, sender) blocks in the
    receive buffer, each block's home rank and home row (the sender's sorted
    row of its first element), and the per-local-expert row counts."""
    W, _, E = C.shape
    stray = np.ones(E, dtype=bool)
    stray[list(local)] = False
    if C[:, me, stray].any():
        raise RuntimeError("received rows for an expert this rank does not hold (placement mismatch)")
    sender_off = np.concatenate([np.zeros((W, 1), np.int64), np.cumsum(C.reshape(W, W * E), axis=1)[:, :-1]], axis=1)
    starts, ranks, homes = [], [], []
    pos = 0
    for e in local:
        for s in range(W):
            starts.append(pos)
            ranks.append(s)
            homes.append(sender_off[s, me * E + e])
            pos += int(C[s, me, e])
    starts.append(pos)
    counts = np.array([C[:, me, e].sum() for e in local], dtype=np.int64)
    return (np.asarray(starts, np.int32), np.asarray(ranks, np.int32), np.asarray(homes, np.int32), counts)


# ── the B200 backend ──────────────────────────────────────────────────────
class CudaExpertBackend:
    """Expert compute of one rank on its GPU: the same kernels as
    ``MoELayer.forward`` (K3, K4, K1, K5, K6) plus the EP gather/pack
    kernels. Holds the full router and the per-expert x-side smoothing of
    all E experts (the sender quantizes for the destination expert) and the
    weights of the local experts only."""

    def __init__(self, gate_weight, experts: list[dict], local_experts, top_k: int = 2, gate_bias=None,
                 out_dtype=torch.bfloat16):
        from .moe import MoELayer

        self.local_experts = tuple(local_experts)
        self.spec = experts
        self.E = len(experts)
        self.k = top_k
        self.out_dtype = out_dtype
        self.gate_w = torch.as_tensor(gate_weight, dtype=torch.float32).cuda().contiguous()
        self.gate_b = None if gate_bias is None else torch.as_tensor(gate_bias, dtype=torch.float32).cuda()
        s13 = torch.stack([torch.as_tensor(np.asarray(_np(e["s13"])), dtype=torch.float64) for e in experts]).cuda()
        self.s13 = s13.contiguous()
        self.s13_recip, self.s13_recip32 = ops.reciprocal(self.s13, with_f32=True)
        self.bank = (MoELayer(gate_weight, [experts[e] for e in self.local_experts], top_k=1, out_dtype=out_dtype)
                     if self.local_experts else None)
        self.d = self.s13.shape[1]
        self.device = self.s13.device
        self._tiled = {}

    def with_local_experts(self, local_experts) -> "CudaExpertBackend":
        """The same layer holding a different expert subset (migration)."""
        return CudaExpertBackend(self.gate_w.cpu().numpy(), self.spec, local_experts, top_k=self.k,
                                 gate_bias=None if self.gate_b is None else self.gate_b.cpu().numpy(),
                                 out_dtype=self.out_dtype)

    @classmethod
    def from_layer_spec(cls, layer, local_experts):
        """Slice a full single-GPU ``MoELayer`` (its host expert list)."""
        return cls(layer.gate_w.cpu().numpy(), layer.host_experts, local_experts, top_k=layer.k,
                   gate_bias=None if layer.gate_b is None else layer.gate_b.cpu().numpy(), out_dtype=layer.out_dtype)

    # host <-> device helpers used by the runtime
    @staticmethod
    def to_index_tensor(a: np.ndarray) -> torch.Tensor:
        return torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32)).cuda()

    @staticmethod
    def to_host(t: torch.Tensor) -> np.ndarray:
        return t.cpu().numpy()

    def _smooth_tables(self, W: int):
        # row_group of a dispatched row is its sort key dest * E + e: tile the
        # per-expert tables W times so key indexes them directly
        if W not in self._tiled:
            self._tiled[W] = tuple(t.repeat(W, 1).contiguous() for t in (self.s13, self.s13_recip, self.s13_recip32))
        return self._tiled[W]

    def route(self, x):
        _, idx, w = ops.router_gate(x, self.gate_w, self.k, gate_bias=self.gate_b)
        return idx, w

    def route_keys(self, idx, dest, E):
        return ops.route_keys(idx, dest, E)

    def permute(self, keys, w, G):
        return ops.route_permute(keys, w, G)

    def quantize_pack(self, x, perm, E):
        W = perm["offsets"].numel() // E if E else 1
        s, sr, sr32 = self._smooth_tables(W)
        n = perm["src_token"].numel()
        a = ops.act_quant(x, smooth=s, smooth_recip=sr, smooth_recip_f32=sr32, row_group=perm["row_expert"],
                          gather=perm["src_token"], rows=n)
        return [a["codes"], ops.ep_pack_params(a, perm["row_weight"])]

    def experts(self, recv: list, index: np.ndarray, group_counts: np.ndarray, mark=lambda _n: None) -> torch.Tensor:
        codes_r, params_r = recv
        n = int(index.size)
        if n == 0:
            return torch.empty((0, self.d), dtype=torch.bfloat16, device="cuda")
        b = self.bank
        G = len(self.local_experts)
        idx = self.to_index_tensor(index)
        prm = ops.ep_unpack_params(params_r, idx)
        a1 = {"codes": ops.gather_rows(codes_r, idx), "scale_f32": prm["scale_f32"], "zp": prm["zp"],
              "rowsum": prm["rowsum"]}
        offs = self.to_index_tensor(np.concatenate([[0], np.cumsum(group_counts)]))
        row_group = self.to_index_tensor(np.repeat(np.arange(G), group_counts))
        fuse = b.d % 16 == 0 and b.d >= 128
        ext = torch.empty((n, 2), dtype=torch.int64, device="cuda") if fuse else None
        h = ops.w8a8_gemm(a1, b.w13, epilogue=L.EPI_SWIGLU, out_dtype=torch.bfloat16, group_offsets=offs,
                          num_groups=G, n_per_group=2 * b.F, next_smooth_recip_f32=b.s2_recip32 if fuse else None,
                          row_ext=ext)
        mark("gemm13_swiglu")
        a2 = ops.act_quant(h, smooth=b.s2, smooth_recip=b.s2_recip, smooth_recip_f32=b.s2_recip32,
                           row_group=row_group, row_ext=ext)
        mark("quant_h")
        y = ops.w8a8_gemm(a2, b.w2, epilogue=L.EPI_DEQUANT, out_dtype=torch.bfloat16, row_weight=prm["weight"],
                          group_offsets=offs, num_groups=G, n_per_group=b.d)
        mark("gemm2")
        inv = np.empty_like(index)
        inv[index] = np.arange(n, dtype=np.int32)
        return ops.gather_rows(y, self.to_index_tensor(inv))

    def combine(self, y_home, perm, T, out=None):
        return ops.combine(y_home, perm["token_pos"], T, self.k, out_dtype=self.out_dtype, out=out)

    # peer transport
    def dispatch_send(self, x, perm, E, bufs, dst_rank, dst_row):
        W = perm["offsets"].numel() // E
        s, sr, sr32 = self._smooth_tables(W)
        # token-major K1 (x read once per token) when x fits its registers
        tok = perm["token_pos"] if ops.act_quant_tokens_ok(x) else None
        ops.act_quant_dispatch(x, perm["src_token"], perm["row_expert"], smooth=s, smooth_recip=sr,
                               smooth_recip_f32=sr32, codes_tab=bufs.codes_tab, params_tab=bufs.params_tab,
                               dst_rank=dst_rank, dst_row=dst_row, row_weight=perm["row_weight"],
                               ldc=bufs.codes.stride(0), token_pos=tok, k=self.k)

    def experts_peer_dev(self, bufs, R_dev, goff, row_group, out_rank, out_row, mark=lambda _n: None):
        """Receiver compute with the row count on the device: kernels are
        sized for the buffer capacity and read R / the group offsets."""
        b = self.bank
        G = len(self.local_experts)
        cap = bufs.codes.shape[0]
        prm = ops.ep_unpack_params(bufs.params, None, cap, n_dev=R_dev)
        a1 = {"codes": bufs.codes, "scale_f32": prm["scale_f32"], "zp": prm["zp"], "rowsum": prm["rowsum"]}
        ext = torch.empty((cap, 2), dtype=torch.int64, device="cuda")
        h = ops.w8a8_gemm(a1, b.w13, epilogue=L.EPI_SWIGLU, out_dtype=torch.bfloat16, group_offsets=goff,
                          num_groups=G, n_per_group=2 * b.F, next_smooth_recip_f32=b.s2_recip32, row_ext=ext)
        mark("gemm13_swiglu")
        a2 = ops.act_quant_given_dev(h, R_dev, row_group, ext, smooth=b.s2, smooth_recip=b.s2_recip,
                                     smooth_recip_f32=b.s2_recip32)
        mark("quant_h")
        ops.w8a8_gemm_scatter(a2, b.w2, out_tab=bufs.y_tab, out_rank=out_rank, out_row=out_row,
                              ldo=bufs.yhome.stride(0), row_weight=prm["weight"], group_offsets=goff, num_groups=G,
                              n_per_group=b.d)
        mark("gemm2")


def plan_placement(idx: torch.Tensor, experts: int, top_k: int, world: int, top_k_per_layer: int = 1,
                   supplement_k_per_layer: int = 1, group=None) -> ExpertPlacement:
    """The paper's placement from GPU-measured routing of one layer: every
    rank records its router output (RoutingStats, one histogram kernel),
    the selections of all ranks are gathered, and plan_two_stage
    (placement.py:125-176) over the global path statistics and expert
    frequencies picks the replicated residents; the rest are bin-packed."""
    from .placement import plan_two_stage
    from .trace import RoutingStats, Trace, expert_freq, path_stats

    st = RoutingStats(1, experts, top_k)
    st.record(idx, 0)
    events = st.to_trace().events
    paths = [ev.path for ev in events]
    if torch.distributed.is_initialized() and torch.distributed.get_world_size(group) > 1:
        gathered = [None] * torch.distributed.get_world_size(group)
        torch.distributed.all_gather_object(gathered, paths, group=group)
        paths = [p for part in gathered for p in part]
    from .trace import RoutingEvent, PHASE_PREFILL
    trace = Trace(1, experts, top_k, [RoutingEvent(t, PHASE_PREFILL, p) for t, p in enumerate(paths)])
    freq = expert_freq(trace)
    plan = plan_two_stage(path_stats(trace), freq, top_k_per_layer, supplement_k_per_layer)
    return ExpertPlacement.from_plan(plan, 0, freq, world)


def plan_stack_placements(stats, world: int, top_k_per_layer: int = 1, supplement_k_per_layer: int = 1,
                          group=None) -> list:
    """Per-layer placements for an EP MoE stack from GPU-measured FULL-PATH
    statistics (``RoutingStats`` of all layers, gathered over the ranks):
    plan_two_stage (placement.py:125-176) ranks whole activation paths across
    layers, then bin-packs each layer's remaining experts."""
    from .placement import plan_two_stage
    from .trace import PHASE_PREFILL, RoutingEvent, Trace, expert_freq, path_stats

    paths = [ev.path for ev in stats.to_trace().events]
    if torch.distributed.is_initialized() and torch.distributed.get_world_size(group) > 1:
        gathered = [None] * torch.distributed.get_world_size(group)
        torch.distributed.all_gather_object(gathered, paths, group=group)
        paths = [p for part in gathered for p in part]
    trace = Trace(stats.layers, stats.experts, stats.top_k,
                  [RoutingEvent(t, PHASE_PREFILL, p) for t, p in enumerate(paths)])
    freq = expert_freq(trace)
    plan = plan_two_stage(path_stats(trace), freq, top_k_per_layer, supplement_k_per_layer)
    return [ExpertPlacement.from_plan(plan, l, freq, world) for l in range(stats.layers)]


def _np(a):
    return a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)


# ── the 32-layer token path over expert parallelism ────────
class ExpertParallelStack:
    """``moe.MoEStack``'s block structure, x_{l+1} = x_l + MoE_l(RMSNorm(x_l))
    (bf16, attention omitted), with every MoE layer expert-parallel on this
    rank. All layers of the peer transport share ONE set of PeerBuffers: a
    layer's peers write this rank's receive / home buffers only after the
    cross-rank barriers of that layer, which this rank reaches only after
    its stream has consumed the previous layer's contents."""

    def __init__(self, layers: list, attn: list | None = None, seq_len: int | None = None):
        if not layers:
            raise ValueError("empty stack")
        self.layers = layers
        self.attn, self.seq_len = attn, seq_len      # replicated attention blocks (tokens stay home)
        self.d = layers[0].be.d
        self.out_dtype = torch.bfloat16

    @classmethod
    def from_stack(cls, stack, placements: list, rank: int, buffers: PeerBuffers | None = None, exchange=None,
                   transport: str = "peer") -> "ExpertParallelStack":
        """Per-layer EP modules of ``rank`` from a full ``MoEStack`` (its host
        expert lists) and one placement per layer (``plan_stack_placements``)."""
        if len(placements) != len(stack.layers):
            raise ValueError(f"{len(placements)} placements for {len(stack.layers)} layers")
        mods = []
        for layer, pl in zip(stack.layers, placements):
            be = CudaExpertBackend.from_layer_spec(layer, pl.local_experts(rank))
            if transport == "peer":
                mods.append(PeerExpertParallelMoE(be, pl, buffers, exchange, rank))
            else:
                mods.append(ExpertParallelMoE(be, pl, exchange, rank))
        return cls(mods, stack.attn, stack.seq_len)

    def forward(self, x: torch.Tensor, timer=None, out: torch.Tensor | None = None) -> torch.Tensor:
        if timer is not None:
            timer.mark("start")
        n = ops.rmsnorm_residual(x, None)[1]
        last = len(self.layers) - 1
        for l, m in enumerate(self.layers):
            if self.attn is not None:
                x, n = ops.rmsnorm_residual(x, self.attn[l](n, self.seq_len))
            y = m.forward(n)
            if l < last:
                x, n = ops.rmsnorm_residual(x, y)
            else:
                x = ops.rmsnorm_residual(x, y, want_norm=False)[0]
        if timer is not None:
            timer.mark("stack")
        if out is not None:
            out.copy_(x)
            return out
        return x

    __call__ = forward

    def check(self, wait: bool = False) -> None:
        for m in self.layers:
            if hasattr(m, "check"):
                m.check(wait)

    def forward_host(self, x_host: torch.Tensor, out_host: torch.Tensor | None = None) -> torch.Tensor:
        x = x_host.to(self.layers[0].be.device, non_blocking=True)
        y = self.forward(x)
        if out_host is None:
            out_host = torch.empty(tuple(y.shape), dtype=y.dtype, pin_memory=True)
        out_host.copy_(y, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        self.check(wait=True)
        return out_host

    def forward_host_stream(self, batches: list, depth: int = 2) -> list:
        from .hostio import stream_batches
        outs = stream_batches(self, self.forward, self.d, self.out_dtype, batches, depth, split_ends=4,
                              quantum=self.seq_len or 1)
        self.check(wait=True)
        return outs
