"""Expert-parallel MoE at the Mixtral shape, W ranks emulated on ONE GPU
(same kernels; the "peers" are other buffers, ranks run phase by phase):
plan_two_stage placement over the routing of all ranks' tokens, peer-memory
dispatch / combine, result compared bit for bit with the single-GPU layer.

    python tools/ep_emulate.py [W] [tokens_per_rank]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2508_07329_b200.ep import (CudaExpertBackend, ExpertParallelMoE, PeerBuffers, PeerExpertParallelMoE,
                                      plan_placement, run_loopback, run_loopback_peer)
from paper_2508_07329_b200.moe import MoELayer


class _Local:
    def __init__(self, world, rank):
        self.world, self.rank = world, rank


W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
T = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
layer = MoELayer.random(8, 4096, 14336, top_k=2, seed=1)
xs = [torch.from_numpy(bench.synth_tokens(T, 4096, 100 + r)).to(torch.bfloat16).cuda() for r in range(W)]
pl = plan_placement(layer.route(torch.cat(xs))[1], 8, 2, W)
print("placement: replicated", pl.replicated, "owner", pl.owner, flush=True)
cap_home = T * 2
bufs = PeerBuffers.loopback(W, 4096, W * cap_home, cap_home)
peer = [PeerExpertParallelMoE(CudaExpertBackend.from_layer_spec(layer, pl.local_experts(r)), pl, bufs[r], rank=r,
                              exchange=_Local(W, r)) for r in range(W)]
t0 = time.perf_counter()
outs = run_loopback_peer(peer, xs)
torch.cuda.synchronize()
print(f"peer transport: {W} ranks x {T} tokens in {time.perf_counter() - t0:.2f} s (emulated, serial)", flush=True)
ok = all(torch.equal(o, layer.forward(x)) for o, x in zip(outs, xs))
a2a = [ExpertParallelMoE(CudaExpertBackend.from_layer_spec(layer, pl.local_experts(r)), pl, rank=r,
                         exchange=_Local(W, r)) for r in range(W)]
ok2 = all(torch.equal(o, layer.forward(x)) for o, x in zip(run_loopback(a2a, xs), xs))
counts = np.bincount(layer.route(torch.cat(xs))[1].cpu().numpy().ravel(), minlength=8)
print(f"bit-identical to the single-GPU layer: peer={ok} all-to-all={ok2}; "
      f"local fraction {pl.local_fraction(counts):.3f}", flush=True)
