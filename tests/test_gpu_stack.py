"""GPU: a stack of W8A8 MoE layers (SURVEY.md C5 without attention) with
GPU-measured full-path routing statistics -> reference trace (write/read
round trip, expert_freq / path_stats equal the oracle's on the same
selections) -> plan_two_stage per-layer placements -> expert-parallel
execution of every layer (4 ranks emulated, peer transport) bit-identical
to the stack, before and after a re-placement (expert migration)."""

import numpy as np
import pytest
import torch

from oracle import routing_ref as RR
from paper_2508_07329_b200 import placement as P
from paper_2508_07329_b200 import trace as TR
from paper_2508_07329_b200.ep import (CudaExpertBackend, ExpertPlacement, PeerBuffers, PeerExpertParallelMoE,
                                      plan_stack_placements, run_loopback_peer)
from paper_2508_07329_b200.moe import MoEStack

from .conftest import bf16_round

pytestmark = pytest.mark.gpu

L, E, D, F, K = 3, 8, 512, 1024, 2


class _Local:
    def __init__(self, world, rank):
        self.world, self.rank = world, rank


@pytest.fixture(scope="module")
def stack(cuda):
    return MoEStack.random(L, E, D, F, top_k=K, seed=21)


def _x(T, seed):
    rng = np.random.default_rng(seed)
    x = rng.normal(size=(T, D)).astype(np.float32)
    x[:, [5, 99, 300, 411]] *= 60.0
    return torch.from_numpy(bf16_round(x)).cuda().bfloat16()


def test_stack_trace_and_placement(stack, tmp_path):
    x = _x(900, 1)
    stats = TR.RoutingStats(L, E, K)
    out = stack(x, stats=stats)
    # per-layer inputs and selections, recomputed layer by layer
    sel, h = [], x
    for layer in stack.layers:
        hn = stack.norm(h)
        sel.append(layer.route(hn)[1].cpu().numpy())
        h = (h.float() + layer.forward(hn).float()).to(h.dtype)
    assert torch.equal(h, out)
    counts = stats.counts.cpu().numpy()
    for l in range(L):
        np.testing.assert_array_equal(counts[l], np.bincount(sel[l].ravel(), minlength=E))
    tr = stats.to_trace()
    assert tr.layers == L and len(tr.events) == 900
    want_paths = [tuple(tuple(sorted(int(e) for e in sel[l][t])) for l in range(L)) for t in range(900)]
    assert [ev.path for ev in tr.events] == want_paths
    # reference statistics on the GPU-measured trace
    TR.write_trace(tmp_path / "trace.txt", tr)
    back = TR.read_trace(tmp_path / "trace.txt")
    assert [ev.path for ev in back.events] == want_paths
    freq, ps = TR.expert_freq(back), TR.path_stats(back)
    paths_np = np.array([[list(s) for s in p] for p in want_paths])
    np.testing.assert_array_equal(freq.counts, RR.expert_freq(paths_np, E))
    o_entries = RR.path_stats(paths_np)
    assert [(tuple(map(tuple, p)), c) for p, c in ps.entries] == [(tuple(map(tuple, p)), c) for p, c in o_entries]
    plan = P.plan_two_stage(ps, freq, 1, 1)
    pls = plan_stack_placements(stats, world=4)
    for l in range(L):
        assert set(pls[l].replicated) == set(plan.residents[l])


def test_stack_expert_parallel_with_migration(stack):
    W = 4
    xs = [_x(t, 10 + i) for i, t in enumerate((300, 64, 500, 200))]
    stats = TR.RoutingStats(L, E, K)
    stack(torch.cat(xs), stats=stats)
    pls = plan_stack_placements(stats, world=W)
    cap_home = 500 * K
    ranks_per_layer = []
    for l, layer in enumerate(stack.layers):
        bufs = PeerBuffers.loopback(W, D, W * cap_home, cap_home)
        ranks_per_layer.append([PeerExpertParallelMoE(CudaExpertBackend.from_layer_spec(layer, pls[l].local_experts(r)),
                                                      pls[l], bufs[r], rank=r, exchange=_Local(W, r))
                                for r in range(W)])

    def ep_stack(parts):
        hs = list(parts)
        for l in range(L):
            ys = run_loopback_peer(ranks_per_layer[l], [stack.norm(h) for h in hs])
            hs = [(h.float() + y.float()).to(h.dtype) for h, y in zip(hs, ys)]
        return hs

    want = [stack(x) for x in xs]
    for got, w in zip(ep_stack(xs), want):
        assert torch.equal(got, w)
    # re-placement: shard every layer plainly, migrate, still identical
    for l in range(L):
        for r, m in enumerate(ranks_per_layer[l]):
            m.migrate(ExpertPlacement.sharded(E, W))
    for got, w in zip(ep_stack(xs), want):
        assert torch.equal(got, w)


def test_stack_with_attention_expert_parallel(cuda):
    """Full Mixtral blocks (W8A8 attention + MoE, pre-norm residual): the
    expert-parallel stack (ExpertParallelStack, one rank, peer transport
    with the device-side plan, replicated attention) equals the
    single-GPU stack bit for bit, and the host serving loop equals both."""
    from paper_2508_07329_b200.ep import ExpertParallelStack
    st = MoEStack.random(2, E, D, F, top_k=K, seed=31, attention=True, seq_len=128, heads=8, kv_heads=2)
    assert st.attn is not None and st.attn[0].head_dim == D // 8
    x = _x(512, 40)
    want = st(x)
    assert torch.isfinite(want.float()).all()
    pls = [ExpertPlacement.sharded(E, 1) for _ in range(2)]
    bufs = PeerBuffers.loopback(1, D, 512 * K, 512 * K)[0]
    ep = ExpertParallelStack.from_stack(st, pls, 0, bufs)
    assert torch.equal(ep(x), want)
    outs = ep.forward_host_stream([(x.cpu().pin_memory(), None), (x.cpu().pin_memory(), None)])
    for o in outs:
        assert torch.equal(o, want.cpu())
    with pytest.raises(ValueError):
        st.attn[0](x[:100], 128)            # not whole sequences
