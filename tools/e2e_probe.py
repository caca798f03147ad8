"""Probe the host-buffer pipeline of MoELayer.forward_host: chunk plans."""
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

def wall(fn, n=10):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e3

print("forward dev ms", wall(lambda: layer.forward(xd)))
print("h2d ms", wall(lambda: xd.copy_(xh, non_blocking=True)))
print("d2h ms", wall(lambda: oh.copy_(xd, non_blocking=True)))
plans = {"4x4096": [4096] * 4, "8x2048": [2048] * 8, "default": None,
         "ramp512": MoELayer.chunk_plan(T, 4096, 512), "ramp1024_8192": MoELayer.chunk_plan(T, 8192, 1024),
         "ramp512_8192": MoELayer.chunk_plan(T, 8192, 512), "ramp2048": MoELayer.chunk_plan(T, 4096, 2048)}
for name, pl in plans.items():
    print(f"forward_host {name:14s} {str(pl if pl else MoELayer.chunk_plan(T)):60s} ms",
          wall(lambda: layer.forward_host(xh, oh, chunks=pl)))
for t in (1024, 2048, 4096, 8192, 16384):
    print(f"forward dev T={t:6d} ms", wall(lambda: layer.forward(xd[:t])))
