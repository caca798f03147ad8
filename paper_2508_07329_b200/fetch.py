"""The paper's offload predictor (Eq. 7-8; sim.py:146-190)
re-targeted from "compute the expert on the CPU vs copy it to the GPU" to
the expert-parallel question on one NVSwitch box: **send a rank's tokens to
the rank holding the expert, or fetch the expert's weights over NVLink and
serve the tokens locally.**

Mapping (reference -> here):

  T_CPU = n * latency_CPU          (Eq. 7)  ->  T_send  = n * latency_send
  T_sum = T_e + n * latency_GPU    (Eq. 8)  ->  T_fetch = T_e + n * latency_local
  T_e = expert bytes / PCIe BW              ->  T_e = expert bytes / NVLink BW
  planned residency (plan_two_stage)        ->  the placement already serves
                                                (source, expert) on the source
  GPU expert cache (LRU)                    ->  LRU cache of fetched experts
                                                per rank (capacity in experts)

``latency_send`` is the per-row cost of remote service: the dispatched row
(d + 16 bytes) and its bf16 result (2d bytes) over NVLink plus the row's
compute at the holder scaled by the holder's load (a busy holder serves it
later); ``latency_local`` is the row's compute here at this rank's load.
Decision semantics follow the reference exactly: precedence local ->
cache (refreshing recency) -> strict comparison (ties keep the default,
sending tokens; the return hop is charged but never steers the decision);
a fetch inserts into the cache, evicting the least recently used expert.

``plan_fetches`` applies the rule to every (source rank, remote expert)
pair of one layer's placement from measured per-source routing counts and
returns the placement with the fetched pairs served locally (realised by
``ExpertParallelMoE.migrate``).
"""

from __future__ import annotations

import math
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np

UNBOUNDED = math.inf

KIND_LOCAL = "local_hit"
KIND_CACHE = "fetched_cache_hit"
KIND_SEND = "send_tokens"
KIND_FETCH = "fetch_then_local"
DECISION_KINDS = (KIND_LOCAL, KIND_CACHE, KIND_SEND, KIND_FETCH)


@dataclass
class NvlinkCostModel:
    """Per-row costs (ms per row per expert) and the expert copy.
    ``return_ms`` is charged to the send route but does not steer the
    decision (as activation_return_ms, sim.py:185-190)."""

    latency_send_ms: float
    latency_local_ms: float
    expert_bytes: float
    link_bw_bytes_per_ms: float
    return_ms: float = 0.0

    def __post_init__(self):
        for name in ("latency_send_ms", "latency_local_ms", "return_ms"):
            v = getattr(self, name)
            if math.isnan(v) or v < 0:
                raise ValueError(f"{name} must be >= 0, got {v}")
        if math.isnan(self.expert_bytes) or self.expert_bytes < 0:
            raise ValueError(f"expert_bytes must be >= 0, got {self.expert_bytes}")
        if not (self.link_bw_bytes_per_ms > 0) or math.isinf(self.link_bw_bytes_per_ms):
            raise ValueError(f"link_bw_bytes_per_ms must be positive and finite, got {self.link_bw_bytes_per_ms}")

    @property
    def transfer_ms(self) -> float:
        return self.expert_bytes / self.link_bw_bytes_per_ms

    @classmethod
    def for_layer(cls, row_ms: float, d: int, expert_bytes: float, link_gbs: float = 900.0,
                  holder_load: float = 1.0, local_load: float = 1.0) -> "NvlinkCostModel":
        """From a measured per-row layer time (e.g. bench ms_per_step /
        (T * k)), the hidden size and the NVLink bandwidth (GB/s per
        direction): a dispatched row moves d + 16 bytes out and 2d back; the
        loads are the ranks' predicted rows relative to the mean."""
        bw = link_gbs * 1e6                      # bytes per ms
        wire = (d + 16 + 2 * d) / bw
        return cls(latency_send_ms=row_ms * holder_load + wire, latency_local_ms=row_ms * local_load,
                   expert_bytes=expert_bytes, link_bw_bytes_per_ms=bw)


@dataclass(frozen=True)
class Decision:
    kind: str
    latency_ms: float


class FetchCache:
    """Per-rank LRU cache of fetched (layer, expert) keys (sim.LruCache
    semantics: capacity 0 stores nothing; insert returns the evicted key)."""

    def __init__(self, capacity: int):
        if capacity < 0:
            raise ValueError(f"capacity must be >= 0, got {capacity}")
        self.capacity = capacity
        self._order: OrderedDict = OrderedDict()

    def __contains__(self, key) -> bool:
        return key in self._order

    def __len__(self) -> int:
        return len(self._order)

    def touch(self, key) -> None:
        self._order.move_to_end(key)

    def insert(self, key):
        if self.capacity == 0:
            return None
        if key in self._order:
            self._order.move_to_end(key)
            return None
        evicted = None
        if len(self._order) >= self.capacity:
            evicted, _ = self._order.popitem(last=False)
        self._order[key] = True
        return evicted

    def residents(self) -> list:
        return list(self._order.keys())


def critical_rows(cost: NvlinkCostModel) -> float:
    """Smallest row count at which fetching strictly beats sending:
    the least integer n with n * latency_send > T_e + n * latency_local
    (sim.critical_batch); UNBOUNDED when sending is never slower per row."""
    if cost.latency_send_ms <= cost.latency_local_ms:
        return UNBOUNDED
    gap = cost.latency_send_ms - cost.latency_local_ms
    return math.floor(cost.transfer_ms / gap) + 1


def decide(expert: int, layer: int, n_rows: int, local: bool, cache: FetchCache, cost: NvlinkCostModel) -> Decision:
    """Route one (source rank, expert) group of ``n_rows`` rows (sim.decide):
    served locally by the placement, else fetched earlier (cache), else the
    strict Eq. 7-8 comparison; a fetch enters the cache."""
    if n_rows < 1:
        raise ValueError(f"n_rows must be >= 1, got {n_rows}")
    if local:
        return Decision(KIND_LOCAL, n_rows * cost.latency_local_ms)
    key = (layer, expert)
    if key in cache:
        cache.touch(key)
        return Decision(KIND_CACHE, n_rows * cost.latency_local_ms)
    t_fetch = cost.transfer_ms + n_rows * cost.latency_local_ms
    if n_rows * cost.latency_send_ms > t_fetch:
        cache.insert(key)
        return Decision(KIND_FETCH, t_fetch)
    return Decision(KIND_SEND, n_rows * cost.latency_send_ms + cost.return_ms)


def plan_fetches(placement, per_source: np.ndarray, layer: int, caches: list, row_ms: float, d: int,
                 expert_bytes: float, link_gbs: float = 900.0):
    """Apply ``decide`` to every (source rank s, expert e) pair that the
    placement serves remotely, largest row groups first, with each side's
    load taken from the placement's predicted rows (updated as pairs move).
    ``per_source[s, e]`` = rows source s routes to expert e; ``caches[s]``
    the FetchCache of rank s. Returns (new placement with the fetched and
    cached pairs served on their source, list of (s, e, Decision))."""
    from .ep import ExpertPlacement

    W, E = placement.world, placement.experts
    ps = np.asarray(per_source, dtype=np.float64).reshape(W, E)
    routes = [list(map(int, placement.dest_table(s))) for s in range(W)]
    load = np.zeros(W)
    for s in range(W):
        for e in range(E):
            load[routes[s][e]] += ps[s, e]
    mean = max(load.mean(), 1e-30)
    decisions = []
    pairs = sorted(((s, e) for s in range(W) for e in range(E) if ps[s, e] > 0),
                   key=lambda p: (-ps[p], p))
    for s, e in pairs:
        n = int(round(ps[s, e]))
        if n < 1:
            continue
        h = routes[s][e]
        cost = NvlinkCostModel.for_layer(row_ms, d, expert_bytes, link_gbs, holder_load=load[h] / mean,
                                         local_load=(load[s] + (0 if h == s else ps[s, e])) / mean)
        dec = decide(e, layer, n, h == s, caches[s], cost)
        if dec.kind in (KIND_FETCH, KIND_CACHE) and h != s:
            routes[s][e] = s
            load[h] -= ps[s, e]
            load[s] += ps[s, e]
        decisions.append((s, e, dec))
    owner = list(placement.owner)
    for e in range(E):
        if owner[e] != -1 and all(routes[s][e] != owner[e] for s in range(W)):
            owner[e] = routes[0][e]         # every source fetched e: the primary holder moves
    return ExpertPlacement(W, E, placement.replicated, tuple(owner), tuple(tuple(r) for r in routes)), decisions
