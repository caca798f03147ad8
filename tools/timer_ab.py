"""Layer forward timed back to back with and without the per-stage CUDA
events (which sit between the PDL-chained kernels), CUDA-event time per step;
run once per library build (MOE_B200_LIB=...) to compare.

    python tools/timer_ab.py [steps] [tokens]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_07329_b200.moe import MoELayer  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
T = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
layer = MoELayer.random(8, 4096, 14336, top_k=2, seed=1)
x = torch.from_numpy(bench.synth_tokens(T, 4096, 100)).to(torch.bfloat16).cuda()
for _ in range(5):
    layer.forward(x)
torch.cuda.synchronize()
res = {}
for rep in range(3):
    for use_timer in (False, True):
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tm = bench.StageTimer()
        t0.record()
        for _ in range(steps):
            layer.forward(x, timer=tm if use_timer else None)
        t1.record()
        torch.cuda.synchronize()
        res.setdefault("timer" if use_timer else "plain", []).append(round(t0.elapsed_time(t1) / steps, 4))
print(os.environ.get("MOE_B200_LIB", "default").split("/")[-1], T, res, flush=True)
