"""Diagnose slow host pipelines after device loops: per-call times + allocator stats."""
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
def st():
    s = torch.cuda.memory_stats()
    return {k: s.get(k) for k in ("num_alloc_retries", "num_device_alloc", "num_device_free", "reserved_bytes.all.current")}
print("start", st())
t = bench.StageTimer()
for _ in range(30):
    layer.forward(xd, timer=t)
torch.cuda.synchronize()
print("after dev", st())
for i in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    layer.forward_host(xh, oh)
    torch.cuda.synchronize(); print("single", i, round((time.perf_counter() - t0) * 1e3, 2), st())
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    layer.forward_host_stream([(xh, oh)] * 10)
    torch.cuda.synchronize(); print("stream10", i, round((time.perf_counter() - t0) * 1e3 / 10, 2), st())
