import os, sys, subprocess, time
sys.path.insert(0, ".")
import torch
import bench
from paper_2508_07329_b200.moe import MoELayer
layer = MoELayer.random(8, 4096, 14336, top_k=2, seed=1)
x = torch.from_numpy(bench.synth_tokens(16384, 4096, 100)).to(torch.bfloat16).cuda()
for _ in range(5): layer.forward(x)
torch.cuda.synchronize()
def plain(n):
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(n): layer.forward(x)
    t1.record(); torch.cuda.synchronize()
    return round(t0.elapsed_time(t1) / n, 3)
def staged(n):
    tm = bench.StageTimer()
    for _ in range(n): layer.forward(x, timer=tm)
    torch.cuda.synchronize()
    return round(sum(tm.stage_ms().values()) / n, 3)
for smi in (False, True, False, True):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader", "-lms", "100"], stdout=subprocess.DEVNULL) if smi else None
    time.sleep(0.5)
    print("smi" if smi else "nosmi", "plain60", plain(60), "staged10", staged(10), "plain10", plain(10), "staged60", staged(60), flush=True)
    if p: p.terminate(); p.wait()
    time.sleep(1.0)
