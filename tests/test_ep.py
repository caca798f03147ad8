"""Expert-parallel runtime on CPU: placement, regrouping, the loopback
driver and a real world-size-2 gloo all-to-all, with the float64 oracle
backend; every rank's output must equal moe_ref.moe_forward on its tokens
(bit-exact: the per-row arithmetic is identical and k = 2 sums commute)."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import moe_ref as M
from paper_2508_07329_b200 import placement as P
from paper_2508_07329_b200 import trace as TR
from paper_2508_07329_b200.ep import ExpertParallelMoE, ExpertPlacement, regroup_index, run_loopback

from .ep_oracle_backend import OracleBackend, random_experts

E, D, F, K = 6, 32, 48, 2


def _layer(seed=0):
    rng = np.random.default_rng(seed)
    experts = random_experts(rng, E, D, F)
    wg = rng.normal(size=(E, D)) / np.sqrt(D)
    wg[0] *= 3.0                                   # skewed routing: expert 0 hot
    return wg, experts


def _tokens(rng, T):
    x = rng.normal(size=(T, D))
    x[:, 3] *= 50.0
    return x.astype(np.float32).astype(np.float64)


# ── placement ──────────────────────────────────────────────────────────────
def test_sharded_placement_blocks():
    p = ExpertPlacement.sharded(8, 4)
    assert p.owner == (0, 0, 1, 1, 2, 2, 3, 3)
    assert p.local_experts(2) == (4, 5)
    np.testing.assert_array_equal(p.dest_table(1), [0, 0, 1, 1, 2, 2, 3, 3])


def test_bin_packing_hottest_first_least_loaded():
    counts = [50, 10, 40, 40, 5, 30]
    p = ExpertPlacement.from_counts(counts, 2)
    # hottest first onto the least-loaded rank (ties -> lower rank):
    # 0(50)->r0, 2(40)->r1, 3(40)->r1, 5(30)->r0, 1(10)->r0 (80 = 80), 4(5)->r1
    assert p.owner == (0, 0, 1, 1, 1, 0)
    loads = [sum(c for c, o in zip(counts, p.owner) if o == r) for r in range(2)]
    assert loads == [90, 85]


def test_replicated_experts_are_local_everywhere():
    p = ExpertPlacement.from_counts([9, 1, 1, 9], 2, replicated=(0, 3))
    assert p.owner[0] == -1 and p.owner[3] == -1
    for r in range(2):
        assert {0, 3} <= set(p.local_experts(r))
        assert p.dest_table(r)[0] == r and p.dest_table(r)[3] == r
    assert p.local_fraction([9, 1, 1, 9]) == pytest.approx((18 + 2 / 2) / 20)


def test_placement_from_two_stage_plan():
    cfg = TR.GenConfig(layers=2, experts_per_layer=E, top_k=2, n_prefill_tokens=60, n_decode_tokens=60,
                      zipf_s=1.2, hot_path_prob=0.3, seed=3)
    trace = TR.generate_trace(cfg)
    stats, freq = TR.path_stats(trace), TR.expert_freq(trace)
    plan = P.plan_two_stage(stats, freq, 1, 1)
    for layer in range(2):
        pl = ExpertPlacement.from_plan(plan, layer, freq, world=2)
        assert set(pl.replicated) == set(plan.residents[layer])
        rep = set(plan.residents[layer])
        assert all((o == -1) == (e in rep) for e, o in enumerate(pl.owner))
        # the local-serve fraction counts replicated activations fully
        c = freq.counts[layer]
        want = (c[list(rep)].sum() + (c.sum() - c[list(rep)].sum()) / 2) / c.sum()
        assert pl.local_fraction(c) == pytest.approx(want)


def test_placement_validation():
    with pytest.raises(ValueError):
        ExpertPlacement(2, 3, (), (0, 1))
    with pytest.raises(ValueError):
        ExpertPlacement(2, 2, (), (0, 2))
    with pytest.raises(ValueError):
        ExpertPlacement(2, 2, (0,), (0, 1))


def test_regroup_index():
    # 2 sources x 3 experts, this rank holds experts 0 and 2
    rc = np.array([[2, 0, 1], [1, 0, 3]])
    idx, g = regroup_index(rc, (0, 2))
    # source blocks: s0 rows [0,1 (e0), 2 (e2)], s1 rows [3 (e0), 4,5,6 (e2)]
    np.testing.assert_array_equal(idx, [0, 1, 3, 2, 4, 5, 6])
    np.testing.assert_array_equal(g, [3, 4])
    with pytest.raises(RuntimeError):
        regroup_index(np.array([[0, 1, 0]]), (0, 2))


# ── runtime with the oracle backend ───────────────────────────────────────
def test_ep_single_rank_matches_moe_forward():
    wg, experts = _layer(1)
    x = _tokens(np.random.default_rng(2), 40)
    pl = ExpertPlacement.sharded(E, 1)
    m = ExpertParallelMoE(OracleBackend(wg, experts, pl.local_experts(0), K), pl)
    got = m(torch.from_numpy(x)).numpy()
    want, _, _ = M.moe_forward(x, wg, experts, K)
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("W,replicated,T", [(2, (), (37, 21)), (3, (0,), (16, 1, 25)), (4, (0, 5), (8, 8, 8, 8))])
def test_ep_loopback_matches_moe_forward(W, replicated, T):
    wg, experts = _layer(3)
    rng = np.random.default_rng(4)
    xs = [_tokens(rng, t) for t in T]
    counts = np.bincount(M.router_topk(M.gate_logits(np.concatenate(xs), wg).astype(np.float32), K)[0].ravel(),
                         minlength=E)
    pl = ExpertPlacement.from_counts(counts, W, replicated)
    ranks = [ExpertParallelMoE(OracleBackend(wg, experts, pl.local_experts(r), K), pl, rank=r,
                               exchange=_NoExchange(W, r)) for r in range(W)]
    outs = run_loopback(ranks, [torch.from_numpy(x) for x in xs])
    for x, o in zip(xs, outs):
        want, _, _ = M.moe_forward(x, wg, experts, K)
        np.testing.assert_array_equal(o.numpy(), want)


class _NoExchange:
    def __init__(self, world, rank):
        self.world, self.rank = world, rank


# ── world size 2 over gloo ─────────────────────────────────────────────────
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wg, experts = _layer(5)
        rng = np.random.default_rng(100 + rank)
        x = _tokens(rng, 30 + 7 * rank)
        pl = ExpertPlacement.from_counts([40, 5, 30, 30, 10, 20], world, replicated=(2,))
        m = ExpertParallelMoE(OracleBackend(wg, experts, pl.local_experts(rank), K), pl)
        out = m(torch.from_numpy(x)).numpy()
        want, _, _ = M.moe_forward(x, wg, experts, K)
        np.save(os.path.join(outdir, f"r{rank}.npy"), np.stack([out, want]))
    finally:
        dist.destroy_process_group()


def test_ep_gloo_world2_matches_moe_forward():
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_gloo_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        for r in range(2):
            got, want = np.load(os.path.join(d, f"r{r}.npy"))
            np.testing.assert_array_equal(got, want)


# ── fused (peer memory) transport: host layout math ───────────────────────
def test_peer_layouts_agree():
    """Every sender's destination row for (receiver, expert) equals the
    receiver's block start for (expert, sender); blocks tile the receive
    buffer; home rows are the senders' sorted rows."""
    rng = np.random.default_rng(9)
    from paper_2508_07329_b200.ep import peer_recv_layout, peer_send_layout
    W, E = 3, 6
    pl = ExpertPlacement.from_counts(rng.integers(1, 100, E), W, replicated=(1,))
    C = np.zeros((W, W, E), dtype=np.int64)
    for s in range(W):
        for e in range(E):
            r = s if pl.owner[e] == -1 else pl.owner[e]
            C[s, r, e] = rng.integers(0, 7)
    for r in range(W):
        starts, ranks, homes, counts = peer_recv_layout(C, r, pl.local_experts(r))
        assert starts[-1] == C[:, r, :].sum()
        assert counts.sum() == starts[-1]
        b = 0
        for e in pl.local_experts(r):
            for s in range(W):
                rank_of, base = peer_send_layout(C, s, pl)
                assert ranks[b] == s and rank_of[r * E + e] == r
                assert base[r * E + e] == starts[b]
                assert homes[b] == C[s].reshape(-1)[: r * E + e].sum()
                b += 1


# ── load-split placement (E <= W) ─────────────────────────────────────────
def test_balanced_placement_splits_hot_experts():
    """8 experts on 8 ranks with skewed routing: one holder per expert makes
    the hottest expert's rank the straggler; the split placement keeps every
    rank within one source unit of the average and at most W - 1 experts
    are split."""
    counts = np.array([400, 90, 80, 120, 60, 100, 70, 80])
    W = 8
    whole = ExpertPlacement.from_counts(counts, W)
    pl = ExpertPlacement.balanced(counts, W)
    lw, lb = whole.rank_loads(counts), pl.rank_loads(counts)
    assert lw.max() / lw.mean() > 3.0
    unit = counts.max() / W
    assert lb.max() - lb.mean() <= unit + 1e-9
    assert sum(len(pl.holders(e)) - 1 for e in range(8)) <= W - 1
    assert lb.sum() == pytest.approx(counts.sum())
    for s in range(W):                     # every source routes each expert to one of its holders
        d = pl.dest_table(s)
        assert all(d[e] in pl.holders(e) for e in range(8))
        for e in range(8):                 # a holder serves its own tokens
            if s in pl.holders(e):
                assert d[e] == s


def test_balanced_equals_from_counts_when_whole_experts_balance():
    counts = [50, 10, 40, 40, 5, 30]
    assert ExpertPlacement.balanced(counts, 2) == ExpertPlacement.from_counts(counts, 2)


def test_balanced_keeps_replicated_local():
    counts = np.array([300, 50, 50, 200, 60, 40])
    pl = ExpertPlacement.balanced(counts, 4, replicated=(0,))
    for s in range(4):
        assert pl.dest_table(s)[0] == s
    assert pl.holders(0) == (0, 1, 2, 3)
    with pytest.raises(ValueError):
        ExpertPlacement(2, 2, (0,), (-1, 0), routes=((1, 0), (1, 0)))   # replicated routed away


@pytest.mark.parametrize("W,T", [(3, (20, 33, 7)), (4, (16, 16, 16, 16))])
def test_ep_loopback_balanced_split_matches_moe_forward(W, T):
    wg, experts = _layer(3)
    rng = np.random.default_rng(8)
    xs = [_tokens(rng, t) for t in T]
    counts = np.bincount(M.router_topk(M.gate_logits(np.concatenate(xs), wg).astype(np.float32), K)[0].ravel(),
                         minlength=E)
    pl = ExpertPlacement.balanced(counts * 4, W)
    ranks = [ExpertParallelMoE(OracleBackend(wg, experts, pl.local_experts(r), K), pl, rank=r,
                               exchange=_NoExchange(W, r)) for r in range(W)]
    for x, o in zip(xs, run_loopback(ranks, [torch.from_numpy(x) for x in xs])):
        want, _, _ = M.moe_forward(x, wg, experts, K)
        np.testing.assert_array_equal(o.numpy(), want)


def _gloo_worker_split(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wg, experts = _layer(5)
        rng = np.random.default_rng(200 + rank)
        x = _tokens(rng, 25 + 9 * rank)
        # expert 0 hot: split over both ranks (each serves its own tokens)
        pl = ExpertPlacement.balanced([400, 5, 30, 30, 10, 20], world)
        assert len(pl.holders(0)) == 2
        m = ExpertParallelMoE(OracleBackend(wg, experts, pl.local_experts(rank), K), pl)
        out = m(torch.from_numpy(x)).numpy()
        want, _, _ = M.moe_forward(x, wg, experts, K)
        np.save(os.path.join(outdir, f"r{rank}.npy"), np.stack([out, want]))
    finally:
        dist.destroy_process_group()


def test_ep_gloo_world2_split_expert():
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_gloo_worker_split, args=(2, _free_port(), d), nprocs=2, join=True)
        for r in range(2):
            got, want = np.load(os.path.join(d, f"r{r}.npy"))
            np.testing.assert_array_equal(got, want)


def test_balanced_placement_properties():
    """Randomised invariants of ExpertPlacement.balanced (hypothesis):
    every (source, expert) goes to a holder of the expert, holders serve
    their own tokens, replicated experts stay local, the busiest rank is
    never worse than one-holder packing and is within one source unit of
    the mean whenever the split placement is the one chosen."""
    from hypothesis import given, settings
    from hypothesis import strategies as st

    @settings(max_examples=120, deadline=None)
    @given(W=st.integers(1, 12), E=st.integers(1, 24), seed=st.integers(0, 10 ** 6), nrep=st.integers(0, 3))
    def check(W, E, seed, nrep):
        rng = np.random.default_rng(seed)
        counts = rng.zipf(1.5, E).astype(np.int64) * rng.integers(1, 50)
        rep = tuple(sorted(set(rng.choice(E, min(nrep, E), replace=False).tolist())))
        pl = ExpertPlacement.balanced(counts, W, rep)
        whole = ExpertPlacement.from_counts(counts, W, rep)
        for s in range(W):
            d = pl.dest_table(s)
            for e in range(E):
                assert d[e] in pl.holders(e)
                if e in rep or s in pl.holders(e):
                    assert d[e] == s
        lb, lw = pl.rank_loads(counts), whole.rank_loads(counts)
        assert lb.max() <= lw.max() + 1e-9
        assert lb.sum() == pytest.approx(counts.sum())
        if pl != whole:
            nonrep = [e for e in range(E) if e not in rep]
            unit = max(counts[e] for e in nonrep) / W
            rep_load = sum(counts[e] for e in rep) / W
            assert lb.max() <= (counts[nonrep].sum() / W + rep_load) + unit + 1e-9

    check()
