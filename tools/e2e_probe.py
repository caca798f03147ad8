"""Probe the host-buffer pipeline: copy/compute overlap of MoELayer.forward_host."""
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
for ch in (16384, 8192, 4096, 2048):
    print("forward_host chunk", ch, "ms", wall(lambda: layer.forward_host(xh, oh, chunk_tokens=ch)))
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for ch in (4096, 2048):
        print("forward_host on side stream chunk", ch, "ms", wall(lambda: layer.forward_host(xh, oh, chunk_tokens=ch)))
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def both():
    with torch.cuda.stream(s1):
        xd.copy_(xh, non_blocking=True)
    with torch.cuda.stream(s2):
        layer.forward(xd[:8192])
print("h2d || forward(8192) ms", wall(both))
print("forward(8192) ms", wall(lambda: layer.forward(xd[:8192])))
