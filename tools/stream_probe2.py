"""Reproduce bench.py's e2e sequence: device loop (stage timer), single calls, then the stream."""
import sys, time
sys.path.insert(0, ".")
import torch
import bench
from paper_2508_07329_b200.moe import MoELayer
T, D = 16384, 4096
layer = MoELayer.random(8, D, 14336, top_k=2, seed=1)
xh = torch.from_numpy(bench.synth_tokens(T, D, 100)).to(torch.bfloat16).pin_memory()
oh = torch.empty((T, D), dtype=torch.bfloat16, pin_memory=True)
xd = xh.cuda()
K = 30
def wall(fn, n=1):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t) * 1e3
for stage in sys.argv[1:]:
    if stage == "dev":
        t = bench.StageTimer()
        print("device+timer ms", wall(lambda: layer.forward(xd, timer=t), K) / K)
    elif stage == "single":
        print("single ms", wall(lambda: layer.forward_host(xh, oh), K + 5) / (K + 5))
    elif stage == "stream":
        layer.forward_host_stream([(xh, oh)] * 5)
        print("stream ms", wall(lambda: layer.forward_host_stream([(xh, oh)] * K)) / K)
