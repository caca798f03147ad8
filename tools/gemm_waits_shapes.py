"""MMA operand-wait share of the tcgen05 GEMM (profile variant, see
tools/gemm_waits.py) for dense DEQUANT GEMMs of growing footprint: if the
waits vanish when A and W fit in L2, the MoE GEMMs' waits are HBM latency /
L2 capacity, not the L2 -> SM fabric or the TMA engine."""
import ctypes
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2508_07329_b200 import _lib as L  # noqa: E402
from paper_2508_07329_b200 import ops  # noqa: E402

lib = L.load()
lib.moe_debug_gemm_waits.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros((1024, 6), dtype=np.uint64)
out = {}
for (M, N, K) in [(4096, 2048, 4096), (8192, 4096, 4096), (16384, 8192, 4096), (32768, 16384, 4096),
                  (32768, 4096, 14336)]:
    g = torch.Generator(device="cuda").manual_seed(0)
    a = {"codes": torch.randint(0, 256, (M, K), dtype=torch.uint8, device="cuda", generator=g),
         "scale_f32": torch.full((M,), 1e-3, device="cuda"), "zp": torch.full((M,), 128, dtype=torch.int32, device="cuda")}
    a["rowsum"] = a["codes"].sum(1, dtype=torch.int32)
    w = {"codes": torch.randint(0, 256, (N, K), dtype=torch.uint8, device="cuda", generator=g),
         "scale_f32": torch.full((N,), 1e-3, device="cuda"), "zp": torch.full((N,), 128, dtype=torch.int32, device="cuda")}
    w["rowsum"] = w["codes"].sum(1, dtype=torch.int32)
    for _ in range(3):
        ops.w8a8_gemm(a, w, epilogue=L.EPI_DEQUANT, out_dtype=torch.bfloat16)
    lib.moe_debug_gemm_waits(buf.ctypes.data, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ops.w8a8_gemm(a, w, epilogue=L.EPI_DEQUANT, out_dtype=torch.bfloat16)
    e1.record()
    lib.moe_debug_gemm_waits(buf.ctypes.data, 1)
    ms = e0.elapsed_time(e1)
    lead = buf[0:148:2].astype(np.float64)
    tot = lead[:, 3].sum()
    out[f"{M}x{N}x{K}"] = {"footprint_MB": (M + N) * K / 2 ** 20, "ms": ms, "tops": 2 * M * N * K / ms / 1e9,
                           "mma_wait_operands": (lead[:, 1].sum() + lead[:, 4].sum()) / tot,
                           "mma_wait_accumulator": lead[:, 0].sum() / tot}
    print(json.dumps({k: round(v, 4) for k, v in out[f"{M}x{N}x{K}"].items()}), M, N, K, flush=True)
