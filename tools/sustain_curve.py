"""Per-step time of the C4 layer over a long back-to-back run (from an idle
GPU), with the SM clock and board power sampled by nvidia-smi: shows the
burst-to-sustained transition under the board's power cap.

    python tools/sustain_curve.py [steps] > profiles/sustain_r02.json"""
import json
import os
import subprocess
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_07329_b200.moe import MoELayer  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
layer = MoELayer.random(8, 4096, 14336, top_k=2, seed=1)
x = torch.from_numpy(bench.synth_tokens(16384, 4096, 100)).to(torch.bfloat16).cuda()
for _ in range(3):
    layer.forward(x)
torch.cuda.synchronize()
time.sleep(3.0)                                   # idle: let the clocks recover
f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
p = subprocess.Popen(["nvidia-smi", "--query-gpu=timestamp,clocks.sm,power.draw", "--format=csv,noheader,nounits",
                      "-lms", "20"], stdout=f, stderr=subprocess.DEVNULL)
time.sleep(0.3)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
t0 = time.time()
ev[0].record()
for i in range(steps):
    layer.forward(x)
    ev[i + 1].record()
torch.cuda.synchronize()
t1 = time.time()
time.sleep(0.2)
p.terminate()
p.wait()
ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
rows = [r.split(", ") for r in open(f.name).read().splitlines() if r.count(",") == 2]
os.unlink(f.name)
clk = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
pw = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
win = 10
out = {"steps": steps, "wall_s": round(t1 - t0, 3),
       "ms_per_step_by_window": [round(sum(ms[i:i + win]) / len(ms[i:i + win]), 4) for i in range(0, steps, win)],
       "first_10_ms": round(sum(ms[:10]) / 10, 4), "last_100_ms": round(sum(ms[-100:]) / 100, 4),
       "sm_mhz_samples": clk[:: max(1, len(clk) // 40)], "power_w_samples": pw[:: max(1, len(pw) // 40)]}
print(json.dumps(out))
