"""Measured int8 tensor-core peak on this B200 (SURVEY.md §8d asks for one:
MEASURED_PEAKS.json has bf16 only). cuBLASLt int8 GEMM via torch._int_mm
(s8 x s8 -> s32) at 8192^3, burst (best of 10) and sustained (back to back
for ~4 s), next to this repo's tcgen05 kind::i8 GEMM on the same shape
(ACC_I32 epilogue, exact int32 out). Writes profiles/int8_peak.json."""
import json
import sys
import time

sys.path.insert(0, ".")
import torch

from paper_2508_07329_b200 import _lib as L
from paper_2508_07329_b200 import ops

N = 8192
ops_per = 2 * N ** 3


def timed(fn, reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def measure(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    burst = min(timed(fn, 1) for _ in range(10))
    t_end = time.time() + 4.0
    ms = []
    while time.time() < t_end:
        ms.append(timed(fn, 10))
    sustained = sorted(ms)[len(ms) // 2]
    return ops_per / burst / 1e9, ops_per / sustained / 1e9


a = torch.randint(-128, 127, (N, N), dtype=torch.int8, device="cuda")
b = torch.randint(-128, 127, (N, N), dtype=torch.int8, device="cuda")
bt = b.t()
res = {"shape": [N, N, N], "unit": "TOPS"}
try:
    res["cublaslt_int8_burst"], res["cublaslt_int8_sustained"] = measure(lambda: torch._int_mm(a, bt))
except Exception as ex:  # noqa: BLE001
    res["cublaslt_error"] = repr(ex)

au = torch.randint(0, 256, (N, N), dtype=torch.uint8, device="cuda")
wu = torch.randint(0, 256, (N, N), dtype=torch.uint8, device="cuda")
A = {"codes": au, "zp": torch.zeros(N, dtype=torch.int32, device="cuda"),
     "rowsum": au.sum(1, dtype=torch.int32), "scale_f32": torch.ones(N, device="cuda")}
W = {"codes": wu, "zp": torch.zeros(N, dtype=torch.int32, device="cuda"),
     "rowsum": wu.sum(1, dtype=torch.int32), "scale_f32": torch.ones(N, device="cuda")}
acc = torch.empty((N, N), dtype=torch.int32, device="cuda")
res["ours_u8_acc_burst"], res["ours_u8_acc_sustained"] = measure(
    lambda: ops.w8a8_gemm(A, W, epilogue=L.EPI_ACC_I32, out=acc))
ybf = torch.empty((N, N), dtype=torch.bfloat16, device="cuda")
res["ours_w8a8_bf16_burst"], res["ours_w8a8_bf16_sustained"] = measure(
    lambda: ops.w8a8_gemm(A, W, epilogue=L.EPI_DEQUANT, out=ybf))
bf = torch.randn(N, N, dtype=torch.bfloat16, device="cuda")
res["cublas_bf16_burst_tflops"], res["cublas_bf16_sustained_tflops"] = measure(lambda: bf @ bf)
res["when"] = time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())
res["gpu"] = torch.cuda.get_device_name()
print(json.dumps(res))
with open("profiles/int8_peak.json", "w") as f:
    json.dump(res, f, indent=1)
