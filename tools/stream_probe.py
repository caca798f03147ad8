"""e2e serving-loop probe: forward_host_stream vs forward_host vs device forward."""
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
layer.forward_host_stream([(xh, oh)] * 3)
for depth in (2, 3):
    print("stream depth", depth, "ms/step", wall(lambda: layer.forward_host_stream([(xh, oh)] * K, depth=depth)) / K)
print("single call ms", wall(lambda: layer.forward_host(xh, oh), K) / K)
print("device ms", wall(lambda: layer.forward(xd), K) / K)
