"""One K7 (Hessian accumulation) and one K8 (GPTQ column loop) launch at the
Mixtral W2 shape (n = 14336, T = 1024 calibration tokens, R = 4096 rows), for
ncu:  ncu --set full -k regex:"hessian_accum|gptq_columns" python tools/calib_ncu.py"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2508_07329_b200 import ops, quant  # noqa: E402

n, T, R = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (14336, 1024, 4096)))
rng = np.random.default_rng(0)
x = torch.from_numpy(rng.normal(size=(T, n))).cuda()
H = ops.hessian(x)
U = quant._inverse_upper_factor_device(H)
w = torch.from_numpy(rng.normal(size=(R, n)) * 0.02).cuda()
sc = (w.amax(1) - w.amin(1)) / 255.0
zp = torch.clamp(torch.round(-w.amin(1) / sc), 0, 255).to(torch.int32)
ops.gptq_columns(w, U, sc, zp, 8)
torch.cuda.synchronize()
print("ok")
