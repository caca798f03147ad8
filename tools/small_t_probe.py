"""Run the Mixtral-shape MoE layer forward at a given token count a few times
(for an ncu launch list at small, latency/HBM-bound batch sizes).

    python tools/small_t_probe.py T [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from bench import D, E, F, TOPK, synth_tokens
from paper_2508_07329_b200.moe import MoELayer

T = int(sys.argv[1]) if len(sys.argv) > 1 else 16
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
layer = MoELayer.random(E, D, F, top_k=TOPK, seed=1)
x = torch.from_numpy(synth_tokens(T, D, seed=100)).to(torch.bfloat16).cuda()
for _ in range(reps):
    layer.forward(x)
torch.cuda.synchronize()
print("ok")
