"""K8 (GPTQ column loop) at the Mixtral shapes per lanes-per-row setting
(MOE_TUNE_GPTQ_LANES 8 / 16 / 32), CUDA events; codes compared across
settings (they must be identical)."""
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2508_07329_b200 import _lib as L  # noqa: E402
from paper_2508_07329_b200 import ops, quant  # noqa: E402

out = {}
torch.manual_seed(0)
for R, n in ((28672, 4096), (4096, 14336)):
    x = torch.randn((n, n + 64), dtype=torch.float64, device="cuda")
    H = 2.0 * x @ x.T
    H += 0.01 * H.diagonal().mean() * torch.eye(n, device="cuda", dtype=torch.float64)
    U = quant._inverse_upper_factor_device(H)
    w = torch.randn((R, n), dtype=torch.float64, device="cuda") * 0.02
    sc = (w.amax(1) - w.amin(1)) / 255.0
    zp = torch.clamp(torch.round(-w.amin(1) / sc), 0, 255).to(torch.int32)
    ref = None
    for lanes in (8, 16, 32):
        best = None
        with L.tuned(L.TUNE_GPTQ_LANES, lanes):
            c = ops.gptq_columns(w, U, sc, zp, 8)
            torch.cuda.synchronize()
            for _ in range(3):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                c = ops.gptq_columns(w, U, sc, zp, 8)
                b.record()
                torch.cuda.synchronize()
                best = a.elapsed_time(b) if best is None else min(best, a.elapsed_time(b))
        ref = c if ref is None else ref
        ms = best
        out[f"R{R}_n{n}_lanes{lanes}"] = {"ms": ms, "tflops": R * n * (n - 1) / ms / 1e9, "equal": bool(torch.equal(c, ref))}
        print(f"R{R}_n{n}_lanes{lanes}", out[f"R{R}_n{n}_lanes{lanes}"], flush=True)
print(json.dumps(out))
