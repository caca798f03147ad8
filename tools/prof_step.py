"""One MoE-layer step at the bench shape, for ncu (launch list / per-kernel capture)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2508_07329_b200.moe import MoELayer
import bench
T = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
layer = MoELayer.random(8, 4096, 14336, top_k=2, seed=1)
x = torch.from_numpy(bench.synth_tokens(T, 4096, 100)).to(torch.bfloat16).cuda()
for _ in range(steps):
    layer.forward(x)
torch.cuda.synchronize()
print("ok")
