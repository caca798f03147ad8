"""GPU: the expert-parallel forward equals the single-GPU MoELayer forward
bit for bit — at world size 1 (identity exchange and a real one-rank NCCL
group) and with several simulated ranks driven in one process
(``run_loopback``: remote experts, several sources per receiver, replicated
experts, an idle rank). Also the EP plumbing kernels on their own."""

import os
import socket
import subprocess
import sys
import textwrap

import numpy as np
import pytest
import torch

from paper_2508_07329_b200 import ops
from paper_2508_07329_b200.ep import CudaExpertBackend, ExpertParallelMoE, ExpertPlacement, run_loopback
from paper_2508_07329_b200.moe import MoELayer

from .conftest import bf16_round

pytestmark = pytest.mark.gpu


def _x(rng, T, d):
    x = rng.normal(size=(T, d)).astype(np.float32)
    x[:, rng.choice(d, max(1, d // 100), replace=False)] *= 100.0
    return torch.from_numpy(bf16_round(x)).cuda().bfloat16()


@pytest.fixture(scope="module")
def layer(cuda):
    return MoELayer.random(8, 512, 1024, top_k=2, seed=3)


class _Local:
    def __init__(self, world, rank):
        self.world, self.rank = world, rank


def test_gather_rows_and_params(cuda):
    rng = np.random.default_rng(0)
    src = torch.from_numpy(rng.integers(0, 256, size=(50, 72), dtype=np.uint8)).cuda()
    idx = torch.from_numpy(rng.permutation(50)[:31].astype(np.int32)).cuda()
    assert torch.equal(ops.gather_rows(src, idx), src[idx.long()])
    odd = torch.from_numpy(rng.integers(0, 256, size=(9, 13), dtype=np.uint8)).cuda()   # byte rows
    i2 = torch.tensor([8, 0, 3], dtype=torch.int32, device=cuda)
    assert torch.equal(ops.gather_rows(odd, i2), odd[i2.long()])
    a = {"codes": src, "scale_f32": torch.rand(50, device=cuda), "zp": torch.arange(50, dtype=torch.int32,
                                                                                    device=cuda),
         "rowsum": torch.arange(50, dtype=torch.int32, device=cuda) * 7}
    w = torch.rand(50, device=cuda)
    prm = ops.ep_pack_params(a, w)
    u = ops.ep_unpack_params(prm, idx)
    li = idx.long()
    for k in ("scale_f32", "zp", "rowsum"):
        assert torch.equal(u[k], a[k][li]), k
    assert torch.equal(u["weight"], w[li])
    dest = torch.tensor([1, 1, 0, 0, 2, 2, 3, 3], dtype=torch.int32, device=cuda)
    top = torch.from_numpy(rng.integers(0, 8, size=(20, 2)).astype(np.int32)).cuda()
    assert torch.equal(ops.route_keys(top, dest, 8), dest[top.long()] * 8 + top)


def test_ep_world1_matches_layer(layer):
    x = _x(np.random.default_rng(1), 777, layer.d)
    pl = ExpertPlacement.sharded(layer.E, 1)
    ep = ExpertParallelMoE(CudaExpertBackend.from_layer_spec(layer, pl.local_experts(0)), pl)
    assert torch.equal(ep(x), layer.forward(x))


@pytest.mark.parametrize("W,replicated,T", [(2, (), (600, 333)), (4, (0, 5), (256, 1, 700, 90)),
                                            (3, (0, 1, 2, 3, 4, 5, 6), (100, 200, 50))])
def test_ep_loopback_matches_layer(layer, W, replicated, T):
    rng = np.random.default_rng(2)
    xs = [_x(rng, t, layer.d) for t in T]
    counts = np.bincount(layer.route(torch.cat(xs))[1].cpu().numpy().ravel(), minlength=layer.E)
    pl = ExpertPlacement.from_counts(counts, W, replicated)
    ranks = [ExpertParallelMoE(CudaExpertBackend.from_layer_spec(layer, pl.local_experts(r)), pl, rank=r,
                               exchange=_Local(W, r)) for r in range(W)]
    for x, out in zip(xs, run_loopback(ranks, xs)):
        assert torch.equal(out, layer.forward(x))


def test_ep_nccl_single_rank_group(tmp_path):
    """A real NCCL process group (world 1): counts and rows go through
    all_to_all_single; result equals the plain layer forward."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    script = textwrap.dedent(f"""
        import os, sys, torch, numpy as np
        sys.path.insert(0, {repr(os.getcwd())})
        import torch.distributed as dist
        from paper_2508_07329_b200.moe import MoELayer
        from paper_2508_07329_b200.ep import CudaExpertBackend, ExpertParallelMoE, ExpertPlacement
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="{port}")
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1)
        layer = MoELayer.random(8, 256, 512, top_k=2, seed=4)
        x = (torch.randn(300, 256, device="cuda") * 3).bfloat16()
        pl = ExpertPlacement.sharded(8, 1)
        ep = ExpertParallelMoE(CudaExpertBackend.from_layer_spec(layer, pl.local_experts(0)), pl)
        ok = torch.equal(ep(x), layer.forward(x))
        dist.destroy_process_group()
        print("EQUAL" if ok else "DIFFERENT")
    """)
    r = subprocess.run([sys.executable, "-c", script], capture_output=True, text=True, timeout=300)
    assert "EQUAL" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("W,replicated,T", [(1, (), (500,)), (2, (), (600, 333)), (4, (0, 5), (256, 1, 700, 90)),
                                            (3, (0, 1, 2, 3, 4, 5, 6), (100, 200, 50))])
def test_ep_peer_loopback_matches_layer(layer, W, replicated, T):
    """Fused peer-memory transport (K1 writes into the owners' receive
    buffers, GEMM2 writes into the home ranks' buffers), W ranks emulated in
    one process: bit-identical to the single-GPU forward."""
    from paper_2508_07329_b200.ep import PeerBuffers, PeerExpertParallelMoE, run_loopback_peer
    rng = np.random.default_rng(3)
    xs = [_x(rng, t, layer.d) for t in T]
    counts = np.bincount(layer.route(torch.cat(xs))[1].cpu().numpy().ravel(), minlength=layer.E)
    pl = ExpertPlacement.from_counts(counts, W, replicated)
    cap_home = max(T) * layer.k
    bufs = PeerBuffers.loopback(W, layer.d, W * cap_home, cap_home)
    ranks = [PeerExpertParallelMoE(CudaExpertBackend.from_layer_spec(layer, pl.local_experts(r)), pl, bufs[r],
                                   rank=r, exchange=_Local(W, r)) for r in range(W)]
    for x, out in zip(xs, run_loopback_peer(ranks, xs)):
        assert torch.equal(out, layer.forward(x))


def test_ep_peer_symmetric_memory_single_rank(tmp_path):
    """The peer transport over torch symmetric memory (NCCL world of 1):
    buffers rendezvoused, device barrier, result equals the plain forward."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    script = textwrap.dedent(f"""
        import os, sys, torch
        sys.path.insert(0, {repr(os.getcwd())})
        import torch.distributed as dist
        from paper_2508_07329_b200.moe import MoELayer
        from paper_2508_07329_b200.ep import (CudaExpertBackend, ExpertPlacement, PeerBuffers,
                                              PeerExpertParallelMoE)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="{port}")
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        layer = MoELayer.random(8, 256, 512, top_k=2, seed=4)
        x = (torch.randn(300, 256, device="cuda") * 3).bfloat16()
        pl = ExpertPlacement.sharded(8, 1)
        bufs = PeerBuffers.symmetric(256, 600, 600)
        ep = PeerExpertParallelMoE(CudaExpertBackend.from_layer_spec(layer, pl.local_experts(0)), pl, bufs)
        ok = torch.equal(ep(x), layer.forward(x))
        dist.destroy_process_group()
        print("EQUAL" if ok else "DIFFERENT")
    """)
    r = subprocess.run([sys.executable, "-c", script], capture_output=True, text=True, timeout=300)
    assert "EQUAL" in r.stdout, r.stdout + r.stderr[-3000:]


def _offsets_from_counts(C):
    """Per sender s: route_permute offsets over its W*E keys from C[s, r, e]."""
    W, _, E = C.shape
    return np.stack([np.concatenate([[0], np.cumsum(C[s].reshape(-1))]) for s in range(W)]).astype(np.int32)


@pytest.mark.parametrize("W,E,seed", [(1, 8, 0), (3, 6, 1), (8, 8, 2), (4, 16, 3)])
def test_ep_peer_plan_matches_host_layout(cuda, W, E, seed):
    """The device exchange plan (moe_ep_peer_plan) equals the host layout
    functions for every rank, with split (multi-holder) placements; an
    overflowing capacity is refused on the device (valid 0, nothing received)."""
    from paper_2508_07329_b200.ep import peer_recv_layout, peer_send_layout
    rng = np.random.default_rng(seed)
    counts = rng.integers(50, 400, E)
    pl = ExpertPlacement.balanced(counts, W, replicated=(1,) if E > 2 else ())
    C = np.zeros((W, W, E), dtype=np.int64)
    for s in range(W):
        dest = pl.dest_table(s)
        for e in range(E):
            C[s, dest[e], e] = rng.integers(0, 40)
    offs = torch.from_numpy(_offsets_from_counts(C)).cuda()
    cap = int(C.sum(axis=(0, 2)).max()) + 3
    cap_home = int(C.sum(axis=(1, 2)).max())
    for me in range(W):
        local = pl.local_experts(me)
        G = len(local)
        plan = ops.ep_peer_plan(offs, me, torch.tensor(local, dtype=torch.int32, device=cuda), cap, cap_home)
        v = {k: t.cpu().numpy() for k, t in ops.plan_views(plan, W, E, G).items()}
        assert v["valid"][0] == 1
        _, base = peer_send_layout(C, me, pl)
        live = C[me].reshape(-1) > 0
        np.testing.assert_array_equal(v["send_base"][live], base[live])
        starts, ranks, homes, gc = peer_recv_layout(C, me, local)
        np.testing.assert_array_equal(v["starts"], starts)
        np.testing.assert_array_equal(v["ranks"], ranks)
        np.testing.assert_array_equal(v["homes"], homes)
        np.testing.assert_array_equal(v["goff"], np.concatenate([[0], np.cumsum(gc)]))
        np.testing.assert_array_equal(v["group"], np.repeat(np.arange(G), W))
        assert v["R"][0] == starts[-1]
        bad = ops.ep_peer_plan(offs, me, torch.tensor(local, dtype=torch.int32, device=cuda), cap - 4, cap_home)
        assert bad[0].item() == 0 and bad[1].item() == 0


@pytest.mark.parametrize("W,T", [(2, (600, 333)), (4, (256, 1, 700, 90)), (8, (64,) * 8)])
def test_ep_peer_loopback_balanced_split(layer, W, T):
    """Split experts (ExpertPlacement.balanced: one hot expert served by
    several ranks, each for a fixed set of sources) over the fused peer
    transport and over the NCCL-style transport: bit-identical to the
    single-GPU forward."""
    from paper_2508_07329_b200.ep import PeerBuffers, PeerExpertParallelMoE, run_loopback_peer
    rng = np.random.default_rng(W)
    xs = [_x(rng, t, layer.d) for t in T]
    skew = np.full(layer.E, 100)
    skew[3] = 1000                          # a hot expert: split over several ranks
    pl = ExpertPlacement.balanced(skew, W)
    assert W < 4 or any(len(pl.holders(e)) > 1 for e in range(layer.E))
    cap_home = max(T) * layer.k
    bufs = PeerBuffers.loopback(W, layer.d, W * cap_home, cap_home)
    ranks = [PeerExpertParallelMoE(CudaExpertBackend.from_layer_spec(layer, pl.local_experts(r)), pl, bufs[r],
                                   rank=r, exchange=_Local(W, r)) for r in range(W)]
    for x, out in zip(xs, run_loopback_peer(ranks, xs)):
        assert torch.equal(out, layer.forward(x))
    ranks = [ExpertParallelMoE(CudaExpertBackend.from_layer_spec(layer, pl.local_experts(r)), pl, rank=r,
                               exchange=_Local(W, r)) for r in range(W)]
    for x, out in zip(xs, run_loopback(ranks, xs)):
        assert torch.equal(out, layer.forward(x))


def test_ep_peer_overflow_refused(layer):
    """Receive buffers too small for the routed rows: no rank writes peer
    memory and the refusal is raised (not a silent overflow)."""
    from paper_2508_07329_b200.ep import PeerBuffers, PeerExpertParallelMoE, run_loopback_peer
    rng = np.random.default_rng(5)
    W, T = 2, (500, 500)
    xs = [_x(rng, t, layer.d) for t in T]
    pl = ExpertPlacement.sharded(layer.E, W)
    bufs = PeerBuffers.loopback(W, layer.d, 64, max(T) * layer.k)
    ranks = [PeerExpertParallelMoE(CudaExpertBackend.from_layer_spec(layer, pl.local_experts(r)), pl, bufs[r],
                                   rank=r, exchange=_Local(W, r)) for r in range(W)]
    sentinel = [b.codes.clone() for b in bufs]
    with pytest.raises(RuntimeError, match="exchange refused"):
        run_loopback_peer(ranks, xs)
    for b, s in zip(bufs, sentinel):
        assert torch.equal(b.codes, s)


def test_ep_forward_host_stream(layer):
    """EP serving loop from pinned host batches equals the device forward."""
    from paper_2508_07329_b200.ep import PeerBuffers, PeerExpertParallelMoE
    rng = np.random.default_rng(6)
    pl = ExpertPlacement.sharded(layer.E, 1)
    bufs = PeerBuffers.loopback(1, layer.d, 2 * 700 * layer.k, 700 * layer.k)[0]
    ep = PeerExpertParallelMoE(CudaExpertBackend.from_layer_spec(layer, pl.local_experts(0)), pl, bufs)
    xs = [_x(rng, t, layer.d) for t in (700, 300, 512)]
    batches = [(x.cpu().pin_memory(), None) for x in xs]
    outs = ep.forward_host_stream(batches)
    for x, o in zip(xs, outs):
        assert torch.equal(o, layer.forward(x).cpu())


def test_ep_fetch_decisions_then_migrate(layer):
    """The Eq. 7-8 predictor re-targeted to NVLink (fetch.plan_fetches) on
    measured per-source routing: the returned placement (fetched experts
    served on their sources) is realised by migrate on every rank and the
    forward stays bit-identical to the single-GPU layer."""
    from paper_2508_07329_b200 import fetch as F
    from paper_2508_07329_b200.ep import PeerBuffers, PeerExpertParallelMoE, run_loopback_peer
    rng = np.random.default_rng(12)
    W, T = 4, 600
    xs = [_x(rng, T, layer.d) for _ in range(W)]
    per_source = np.stack([np.bincount(layer.route(x)[1].cpu().numpy().ravel(), minlength=layer.E) for x in xs])
    pl = ExpertPlacement.sharded(layer.E, W)
    caches = [F.FetchCache(2) for _ in range(W)]
    # a tiny "expert" makes fetching cheap, so the rule fires for the larger row groups
    new, dec = F.plan_fetches(pl, per_source, 0, caches, row_ms=1.4e-4, d=layer.d, expert_bytes=2e5)
    assert any(d.kind == F.KIND_FETCH for _, _, d in dec)
    cap_home = T * layer.k
    bufs = PeerBuffers.loopback(W, layer.d, W * cap_home, cap_home)
    ranks = [PeerExpertParallelMoE(CudaExpertBackend.from_layer_spec(layer, pl.local_experts(r)), pl, bufs[r],
                                   rank=r, exchange=_Local(W, r)) for r in range(W)]
    for m in ranks:
        m.migrate(new)
    for x, out in zip(xs, run_loopback_peer(ranks, xs)):
        assert torch.equal(out, layer.forward(x))
