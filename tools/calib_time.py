"""HAQ calibration time at the Mixtral expert shapes on one B200 (SURVEY.md
a12-a17 at C4 scale): quantize_layer (21-point smoothing search, Hessian,
inverse factor, fp64 GPTQ column loop) for one expert's stacked W1||W3
[28672, 4096] and its W2 [4096, 14336], with T routed calibration tokens.
The CPU oracle is timed on a row slice and extrapolated (rows are
independent in the column loop).

    python tools/calib_time.py [T] [out.json]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2508_07329_b200 import quant

T = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 1024
rng = np.random.default_rng(0)
res = {"tokens": T}
for name, (R, n) in {"w13": (28672, 4096), "w2": (4096, 14336)}.items():
    w = torch.from_numpy(rng.normal(size=(R, n)) * 0.02).cuda()
    x = rng.normal(size=(n, T))
    x[rng.choice(n, n // 100, replace=False)] *= 50.0
    xd = torch.from_numpy(x).cuda()
    quant.quantize_layer(w[:256].contiguous(), xd)          # warm-up (module loading, solver handles)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = quant.quantize_layer(w, xd)
    torch.cuda.synchronize()
    res[name] = {"rows": R, "cols": n, "gpu_s": time.perf_counter() - t0,
                 "smoothing_exponent": float(out.smoothing.exponent)}
    print(name, res[name], flush=True)
path = next((a for a in sys.argv[1:] if a.endswith(".json")), None)
if path:
    json.dump(res, open(path, "w"), indent=1)
