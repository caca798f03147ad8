"""Sub-phase times of the EP send phase for one emulated rank (W = 8,
T tokens per rank, balanced placement): router, route keys + permutation
over W*E keys, device plan, row map, K1 dispatch into the peer buffers."""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_07329_b200 import ops  # noqa: E402
from paper_2508_07329_b200.ep import CudaExpertBackend, PeerBuffers, PeerExpertParallelMoE, plan_placement  # noqa: E402
from paper_2508_07329_b200.moe import MoELayer  # noqa: E402


class _Local:
    def __init__(self, world, rank):
        self.world, self.rank = world, rank


W, T = 8, int(sys.argv[1]) if len(sys.argv) > 1 else 8192
layer = MoELayer.random(8, 4096, 14336, top_k=2, seed=1)
xs = [torch.from_numpy(bench.synth_tokens(T, 4096, 100 + r)).to(torch.bfloat16).cuda() for r in range(W)]
pl = plan_placement(layer.route(torch.cat(xs))[1], 8, 2, W)
bufs = PeerBuffers.loopback(W, 4096, 4 * T * 2, T * 2)
m = PeerExpertParallelMoE(CudaExpertBackend.from_layer_spec(layer, pl.local_experts(0)), pl, bufs[0], rank=0,
                          exchange=_Local(W, 0))
ms = [PeerExpertParallelMoE(CudaExpertBackend.from_layer_spec(layer, pl.local_experts(r)), pl, bufs[r], rank=r,
                            exchange=_Local(W, r)) for r in range(W)]


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


acc = {}
for rep in range(6):
    sts = [mm.peer_prepare(x) for mm, x in zip(ms, xs)]
    offs = torch.stack([st.perm["offsets"] for st in sts])
    x = xs[0]
    e0 = ev()
    idx, w = m.be.route(x)
    e1 = ev()
    keys = m.be.route_keys(idx, m.dest, 8)
    perm = m.be.permute(keys, w, W * 8)
    e2 = ev()
    plan = m.peer_plan(offs)
    e3 = ev()
    v = ops.plan_views(plan, W, 8, len(m.local))
    dst_rank, dst_row = ops.block_map(perm["src_token"].numel(), perm["offsets"], m._rank_of, v["send_base"],
                                      valid=v["valid"])
    e4 = ev()
    m.be.dispatch_send(x, perm, 8, m.bufs, dst_rank, dst_row)
    e5 = ev()
    torch.cuda.synchronize()
    if rep >= 2:
        for k, (a, b) in {"router": (e0, e1), "keys_permute": (e1, e2), "plan": (e2, e3), "block_map": (e3, e4),
                          "k1_dispatch": (e4, e5)}.items():
            acc[k] = acc.get(k, 0.0) + a.elapsed_time(b) / 4
m.check(wait=True)
print(json.dumps({k: round(v, 4) for k, v in acc.items()}))
