"""GEMM raster band sweep at the bench shape (C4, 16384 tokens): per band
budget (MOE_TUNE_BAND_MB) the per-stage CUDA-event times of the layer
forward, averaged over `steps` steps after warm-up.

    python tools/band_sweep.py [steps] [mb,mb,...]
With MOE_B200_BAND_ONE=<mb> it runs a single setting (for ncu)."""
import json
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_07329_b200 import _lib as L  # noqa: E402
from paper_2508_07329_b200.moe import MoELayer  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
mbs = [int(v) for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else "6,12,24,48,96,100000".split(","))]
if os.environ.get("MOE_B200_BAND_ONE"):
    mbs = [int(os.environ["MOE_B200_BAND_ONE"])]
layer = MoELayer.random(8, 4096, 14336, top_k=2, seed=1)
x = torch.from_numpy(bench.synth_tokens(16384, 4096, 100)).to(torch.bfloat16).cuda()
out = {}
for mb in mbs:
    with L.tuned(L.TUNE_BAND_MB, mb):
        for _ in range(3):
            layer.forward(x)
        torch.cuda.synchronize()
        tm = bench.StageTimer()
        for _ in range(steps):
            layer.forward(x, timer=tm)
        torch.cuda.synchronize()
        st = {k: round(v / steps, 4) for k, v in tm.stage_ms().items()}
    out[mb] = st
    print(mb, st, flush=True)
print(json.dumps(out))
