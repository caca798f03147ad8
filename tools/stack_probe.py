"""Per-layer timing through a Mixtral-shape MoE stack (stage events), to see
whether deeper layers' activations change kernel costs."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import bench
from paper_2508_07329_b200.moe import MoEStack

L_ = int(sys.argv[1]) if len(sys.argv) > 1 else 8
stack = MoEStack.random(L_, 8, 4096, 14336, top_k=2, seed=7)
for lay in stack.layers:
    lay.host_experts = None
x = torch.from_numpy(bench.synth_tokens(4096, 4096, 100)).to(torch.bfloat16).cuda()
h = x
for l, layer in enumerate(stack.layers):
    t = bench.StageTimer()
    hn = stack.norm(h)
    for _ in range(3):
        layer.forward(hn)
    torch.cuda.synchronize()
    t = bench.StageTimer()
    y = layer.forward(hn, timer=t)
    torch.cuda.synchronize()
    st = t.stage_ms()
    print(l, f"amax {h.float().abs().max().item():9.1f}", " ".join(f"{k}={v:.3f}" for k, v in st.items()),
          f"total={sum(st.values()):.3f}")
    h = (h.float() + y.float()).to(h.dtype)
