"""Step-by-step device check of the MoE forward (debug aid; run with
MOE_B200_SYNC=1 CUDA_LAUNCH_BLOCKING=1)."""
import sys, traceback
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2508_07329_b200 import ops, _lib as L
torch.cuda.set_device(0)
L.load()
def step(name, fn):
    try:
        r = fn(); torch.cuda.synchronize(); print("OK  ", name, flush=True); return r
    except Exception as e:
        print("FAIL", name, repr(e)[:300], flush=True); traceback.print_exc(); sys.exit(1)
x = torch.randn(256, 256, device="cuda")
s = torch.ones(1, 256, dtype=torch.float64, device="cuda")
step("recip", lambda: ops.reciprocal(s))
step("act_quant f32 plain", lambda: ops.act_quant(x))
step("act_quant f32 mult", lambda: ops.act_quant(x, smooth=s, smooth_mode=L.SMOOTH_MULTIPLY, granularity="per_output_row", rowsum=False))
step("act_quant bf16 div", lambda: ops.act_quant(x.bfloat16(), smooth=s))
step("act_quant per_tensor", lambda: ops.act_quant(x, granularity="per_tensor"))
gw = torch.randn(8, 256, device="cuda")
lg, idx, w = step("router", lambda: ops.router_gate(x.bfloat16(), gw, 2))
print(idx[:4].tolist(), w[:4].tolist())
p = step("permute", lambda: ops.route_permute(idx, w, 8))
print(p["offsets"].tolist())
a1 = step("act_quant gather", lambda: ops.act_quant(x.bfloat16(), smooth=s.expand(8, 256).contiguous(), row_group=p["row_expert"], gather=p["src_token"], rows=512))
a = ops.act_quant(x)
wq = ops.act_quant(torch.randn(256, 256, device="cuda"), granularity="per_output_row")
step("gemm simt small K", lambda: ops.w8a8_gemm(ops.act_quant(x[:, :48].contiguous()), ops.act_quant(torch.randn(64, 48, device="cuda")), epilogue=L.EPI_ACC_I32))
step("gemm tc acc", lambda: ops.w8a8_gemm(a, wq, epilogue=L.EPI_ACC_I32))
step("gemm tc dequant", lambda: ops.w8a8_gemm(a, wq))
print("all steps ok")
