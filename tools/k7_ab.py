"""K7 (Hessian accumulation) throughput at the Mixtral expert shapes: DMMA
kernel vs the SIMT kernel (MOE_B200_K7_SIMT=1 in a second process)."""
import json
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2508_07329_b200 import ops  # noqa: E402

out = {"kernel": "simt" if os.environ.get("MOE_B200_K7_SIMT") else "dmma"}
for n, T in ((4096, 1024), (14336, 1024)):
    x = torch.randn((T, n), dtype=torch.float64, device="cuda")
    for _ in range(2):
        ops.hessian(x)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        ops.hessian(x, finalize=False)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    out[f"n{n}"] = {"ms": ms, "tflops": 2.0 * n * n * T / ms / 1e9}
print(json.dumps(out))
