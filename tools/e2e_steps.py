"""End-to-end serving loop (MoELayer.forward_host_stream) vs the number of
batches K at the bench shape: separates the pipeline fill / drain (paid
once per call) from a steady-state cost of overlapping the copies."""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_07329_b200.moe import MoELayer  # noqa: E402

T = 16384
layer = MoELayer.random(8, 4096, 14336, top_k=2, seed=1)
xh = torch.from_numpy(bench.synth_tokens(T, 4096, 100)).to(torch.bfloat16).pin_memory()
oh = torch.empty((T, 4096), dtype=torch.bfloat16, pin_memory=True)
xd = xh.cuda()
res = {}
for rnd in range(2):
    for K in (5, 20, 60):
        layer.forward_host_stream([(xh, oh)] * 3)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        layer.forward_host_stream([(xh, oh)] * K)
        torch.cuda.synchronize()
        e2e = (time.perf_counter() - t0) * 1000 / K
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(K):
            layer.forward(xd)
        b.record()
        torch.cuda.synchronize()
        res.setdefault(K, []).append({"e2e_ms": round(e2e, 3), "device_ms": round(a.elapsed_time(b) / K, 3)})
print(json.dumps(res))
