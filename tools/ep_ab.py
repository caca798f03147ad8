"""In-process A/B at the bench shape: the plain single-GPU layer forward vs
the expert-parallel (peer transport, world 1, device-side plan) forward,
alternating blocks of `steps` steps (thermal drift hits both alike)."""
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_07329_b200.ep import CudaExpertBackend, ExpertPlacement, PeerBuffers, PeerExpertParallelMoE  # noqa: E402
from paper_2508_07329_b200.moe import MoELayer  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
T = 16384
layer = MoELayer.random(8, 4096, 14336, top_k=2, seed=1)
x = torch.from_numpy(bench.synth_tokens(T, 4096, 100)).to(torch.bfloat16).cuda()
pl = ExpertPlacement.sharded(8, 1)
ep = PeerExpertParallelMoE(CudaExpertBackend.from_layer_spec(layer, pl.local_experts(0)), pl,
                           PeerBuffers.loopback(1, 4096, T * 2, T * 2)[0])
assert torch.equal(ep(x), layer.forward(x))
res = {"plain": [], "ep": []}
stage = {"plain": {}, "ep": {}}
for rnd in range(3):
    for name, m in (("plain", layer), ("ep", ep)):
        for _ in range(3):
            m.forward(x)
        torch.cuda.synchronize()
        tm = bench.StageTimer()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(steps):
            m.forward(x, timer=tm)
        b.record()
        torch.cuda.synchronize()
        res[name].append(a.elapsed_time(b) / steps)
        for k, v in tm.stage_ms().items():
            stage[name][k] = stage[name].get(k, 0.0) + v / steps / 3
print(json.dumps({"ms": res, "stages": {n: {k: round(v, 4) for k, v in s.items()} for n, s in stage.items()}}))
