"""The Eq. 7-8 predictor re-targeted to NVLink expert parallelism
(paper_2508_07329_b200/fetch.py): the reference simulator's decision
semantics (sim.py:146-190, tests/test_sim.py) carried over — critical size,
strict comparison with ties on the default route, precedence, the return
hop not steering the decision, LRU fetch cache — plus plan_fetches on a
placement."""

import math

import numpy as np
import pytest

from paper_2508_07329_b200 import fetch as F
from paper_2508_07329_b200.ep import ExpertPlacement


def _cost(send=1.0, local=0.1, t_e=10.0, ret=0.0):
    return F.NvlinkCostModel(send, local, t_e, 1.0, ret)


def test_critical_rows_pinned_example():
    # T_e = 10, send 1, local 0.1: sending loses for the first time at n = 12
    assert F.critical_rows(_cost()) == 12


def test_critical_rows_unbounded_and_free_transfer():
    assert F.critical_rows(_cost(send=0.1, local=0.1)) == F.UNBOUNDED
    assert F.critical_rows(_cost(send=0.05, local=0.1)) == F.UNBOUNDED
    assert F.critical_rows(_cost(t_e=0.0)) == 1
    assert F.critical_rows(F.NvlinkCostModel(math.inf, 0.1, 10.0, 1.0)) == 1


def test_decide_flips_exactly_at_critical_rows():
    for n, kind in ((11, F.KIND_SEND), (12, F.KIND_FETCH), (13, F.KIND_FETCH)):
        assert F.decide(0, 0, n, False, F.FetchCache(0), _cost()).kind == kind, n


def test_decide_precedence_and_cache():
    d = F.decide(0, 0, 7, True, F.FetchCache(0), _cost())
    assert d.kind == F.KIND_LOCAL and d.latency_ms == pytest.approx(0.7)
    cache = F.FetchCache(2)
    cache.insert((0, 1))
    cache.insert((0, 2))
    d = F.decide(1, 0, 3, False, cache, _cost())
    assert d.kind == F.KIND_CACHE and d.latency_ms == pytest.approx(0.3)
    assert cache.insert((0, 3)) == (0, 2)          # (0, 1) was refreshed


def test_decide_tie_sends_and_return_hop_does_not_steer():
    d = F.decide(0, 0, 10, False, F.FetchCache(4), _cost(t_e=9.0))
    assert d.kind == F.KIND_SEND and d.latency_ms == pytest.approx(10.0)
    c = _cost(ret=100.0)
    assert F.decide(0, 0, 11, False, F.FetchCache(4), c).kind == F.KIND_SEND
    d12 = F.decide(0, 0, 12, False, F.FetchCache(4), c)
    assert d12.kind == F.KIND_FETCH and d12.latency_ms == pytest.approx(11.2)


def test_fetch_populates_cache_and_validation():
    cache = F.FetchCache(2)
    d = F.decide(5, 3, 1, False, cache, _cost(send=10.0, t_e=4.0))
    assert d.kind == F.KIND_FETCH and (3, 5) in cache
    with pytest.raises(ValueError):
        F.decide(0, 0, 0, False, cache, _cost())
    with pytest.raises(ValueError):
        F.NvlinkCostModel(-1.0, 0.1, 1.0, 1.0)
    with pytest.raises(ValueError):
        F.NvlinkCostModel(1.0, 0.1, 1.0, 0.0)
    with pytest.raises(ValueError):
        F.FetchCache(-1)


def test_for_layer_costs():
    c = F.NvlinkCostModel.for_layer(row_ms=1.4e-4, d=4096, expert_bytes=176e6, link_gbs=900.0, holder_load=1.2)
    assert c.transfer_ms == pytest.approx(176e6 / 9e8)
    assert c.latency_send_ms == pytest.approx(1.4e-4 * 1.2 + (3 * 4096 + 16) / 9e8)
    # a 20 % busier holder makes fetching pay from a few thousand rows on
    assert 3000 < F.critical_rows(c) < 6000


def test_plan_fetches_moves_big_groups_off_an_overloaded_holder():
    """8 ranks, expert 0 on rank 0 only and very hot: the big row groups of
    the other ranks fetch expert 0 (cache capacity 1 each); small groups of
    a lightly loaded expert keep being sent."""
    W, E = 8, 8
    pl = ExpertPlacement.sharded(E, W)
    ps = np.full((W, E), 500.0)
    ps[:, 0] = 12000.0
    caches = [F.FetchCache(1) for _ in range(W)]
    new, dec = F.plan_fetches(pl, ps, 0, caches, row_ms=1.4e-4, d=4096, expert_bytes=176e6)
    fetched = {(s, e) for s, e, d in dec if d.kind == F.KIND_FETCH}
    assert fetched and all(e == 0 for _, e in fetched)
    for s, e in fetched:
        assert new.dest_table(s)[e] == s and (0, 0) in caches[s]
    assert all(d.kind in (F.KIND_SEND, F.KIND_LOCAL) for s, e, d in dec if e != 0)
    before, after = pl.rank_loads(ps.sum(axis=0)), new.rank_loads(ps.sum(axis=0))
    assert after.max() < before.max()
    # a second batch: the fetched experts are now local to their sources
    _, dec2 = F.plan_fetches(new, ps, 0, caches, row_ms=1.4e-4, d=4096, expert_bytes=176e6)
    assert all(d.kind == F.KIND_LOCAL for s, e, d in dec2 if (s, e) in fetched)
