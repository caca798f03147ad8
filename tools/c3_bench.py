"""C3 (BASELINE.json configs[2]): OPT-6.7B-shape W8A8 FFN (fc1 4096->16384,
ReLU, fc2 16384->4096) prefill of 8192 tokens on one B200. CUDA-event
timing per stage (K1 x, GEMM fc1, ReLU, K1 h, GEMM fc2), int8 TOPS of the
GEMMs against the measured cuBLASLt int8 peak."""
import json
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2508_07329_b200 import _lib as L
from paper_2508_07329_b200 import ops
from paper_2508_07329_b200.linear import W8A8Linear

T, D, F = 8192, 4096, 16384
rng = np.random.default_rng(0)
x = torch.from_numpy(rng.normal(size=(T, D)).astype(np.float32)).cuda()
x[:, torch.from_numpy(rng.choice(D, D // 100, replace=False)).cuda()] *= 100.0
x = x.bfloat16()
s1 = np.exp(rng.normal(size=D) * 0.5)
s2 = np.exp(rng.normal(size=F) * 0.5)
fc1 = W8A8Linear.from_rtn(torch.randn(F, D, device="cuda") * 0.02, smooth=s1,
                          bias=rng.normal(size=F).astype(np.float32) * 0.1)
fc2 = W8A8Linear.from_rtn(torch.randn(D, F, device="cuda") * 0.02, smooth=s2,
                          bias=rng.normal(size=D).astype(np.float32) * 0.1)


def step(ev=None):
    marks = []
    def mark():
        if ev is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            marks.append(e)
    mark()
    xq = fc1.quantize_input(x); mark()
    h = ops.w8a8_gemm(xq, fc1.w, epilogue=L.EPI_DEQUANT, out_dtype=torch.bfloat16, bias=fc1.bias); mark()
    h = torch.relu_(h); mark()
    hq = fc2.quantize_input(h); mark()
    y = ops.w8a8_gemm(hq, fc2.w, epilogue=L.EPI_DEQUANT, out_dtype=torch.bfloat16, bias=fc2.bias); mark()
    return y, marks


for _ in range(3):
    step()
torch.cuda.synchronize()
names = ["k1_x", "gemm_fc1", "relu(torch)", "k1_h", "gemm_fc2"]
acc = np.zeros(len(names))
n = 20
for _ in range(n):
    _, m = step(True)
    torch.cuda.synchronize()
    acc += [m[i].elapsed_time(m[i + 1]) for i in range(len(names))]
ms = acc / n
peak = json.load(open("profiles/int8_peak.json"))["cublaslt_int8_burst"]
ops1 = 2 * T * D * F
res = {"config": "C3 OPT-6.7B FFN W8A8, 8192 tokens", "stages_ms": dict(zip(names, ms.round(4).tolist())),
       "gemm_fc1_tops": ops1 / (ms[1] / 1e3) / 1e12, "gemm_fc2_tops": ops1 / (ms[4] / 1e3) / 1e12,
       "int8_peak_measured": peak, "tokens_per_s": T / (ms.sum() / 1e3)}
res["gemm_frac_of_measured_peak"] = 2 * ops1 / ((ms[1] + ms[4]) / 1e3) / 1e12 / peak
print(json.dumps(res))
