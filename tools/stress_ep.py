"""Randomised sweep of the expert-parallel transports in one process (W
ranks emulated, tests/test_gpu_ep.py style): random world sizes, replicated
sets, balanced / frequency placements and per-rank token counts; every rank's
output must equal the single-GPU layer forward bit for bit, for the fused
peer-memory transport and the all-to-all one.

    python tools/stress_ep.py [seconds] [seed]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2508_07329_b200.ep import (CudaExpertBackend, ExpertParallelMoE, ExpertPlacement, PeerBuffers,  # noqa: E402
                                      PeerExpertParallelMoE, run_loopback, run_loopback_peer)
from paper_2508_07329_b200.moe import MoELayer  # noqa: E402
from tests.conftest import bf16_round  # noqa: E402


class _Local:
    def __init__(self, world, rank):
        self.world, self.rank = world, rank


budget = float(sys.argv[1]) if len(sys.argv) > 1 else 180.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
layers = {E: MoELayer.random(E, 512, 1024, top_k=2, seed=E) for E in (4, 8)}
t_end = time.time() + budget
n = fails = 0
while time.time() < t_end:
    E = int(rng.choice([4, 8]))
    layer = layers[E]
    W = int(rng.integers(1, 5))
    T = [int(v) for v in rng.integers(1, 900, size=W)]
    xs = []
    for t in T:
        x = rng.normal(size=(t, 512)).astype(np.float32)
        x[:, rng.choice(512, 5, replace=False)] *= 100.0
        xs.append(torch.from_numpy(bf16_round(x)).cuda().bfloat16())
    counts = np.bincount(layer.route(torch.cat(xs))[1].cpu().numpy().ravel(), minlength=E)
    nrep = int(rng.integers(0, E))
    replicated = tuple(sorted(rng.choice(E, nrep, replace=False).tolist()))
    pl = (ExpertPlacement.balanced(counts, W, replicated) if rng.random() < 0.5
          else ExpertPlacement.from_counts(counts, W, replicated))
    want = [layer.forward(x) for x in xs]
    ok = True
    try:
        cap_home = max(T) * layer.k
        bufs = PeerBuffers.loopback(W, layer.d, W * cap_home, cap_home)
        ranks = [PeerExpertParallelMoE(CudaExpertBackend.from_layer_spec(layer, pl.local_experts(r)), pl, bufs[r],
                                       rank=r, exchange=_Local(W, r)) for r in range(W)]
        ok &= all(torch.equal(o, w) for o, w in zip(run_loopback_peer(ranks, xs), want))
        ranks = [ExpertParallelMoE(CudaExpertBackend.from_layer_spec(layer, pl.local_experts(r)), pl, rank=r,
                                   exchange=_Local(W, r)) for r in range(W)]
        ok &= all(torch.equal(o, w) for o, w in zip(run_loopback(ranks, xs), want))
    except Exception as e:   # noqa: BLE001
        ok = False
        print("error:", repr(e)[:200], flush=True)
    n += 1
    fails += not ok
    print(f"E={E} W={W} T={T} replicated={replicated} routes={len(pl.routes) if pl.routes else 0}: "
          f"{'ok' if ok else 'FAIL'}", flush=True)
print(f"{n} configurations, {fails} failures", flush=True)
