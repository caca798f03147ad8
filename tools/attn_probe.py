"""Attention half of a C5 block at the bench shape (16384 tokens = 4 x 4096):
time of the fused W8A8 QKV projection (K1 + GEMM), RoPE, SDPA and the W8A8
output projection, CUDA events, and the SDPA backend torch picks."""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_07329_b200.attention import W8A8Attention  # noqa: E402

att = W8A8Attention.random(4096, 32, 8, 128, seed=3, max_pos=4096)
x = torch.from_numpy(bench.synth_tokens(16384, 4096, 100)).to(torch.bfloat16).cuda()
S = 4096


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


for _ in range(3):
    att(x, S)
torch.cuda.synchronize()
acc = {"qkv_ms": 0.0, "rope_ms": 0.0, "sdpa_ms": 0.0, "o_ms": 0.0}
n = 10
for _ in range(n):
    e0 = ev()
    qkv = att.qkv(x, out_dtype=torch.bfloat16)
    e1 = ev()
    from paper_2508_07329_b200 import ops
    pos = att.positions(x.shape[0], S)
    ops.rope_(qkv, 32, 128, att.cos, att.sin, pos)
    ops.rope_(qkv[:, 32 * 128:], 8, 128, att.cos, att.sin, pos)
    e2 = ev()
    a = att.attend(qkv, S)
    e3 = ev()
    att.o(a, out_dtype=torch.bfloat16)
    e4 = ev()
    torch.cuda.synchronize()
    for k, (p, q) in zip(acc, ((e0, e1), (e1, e2), (e2, e3), (e3, e4))):
        acc[k] += p.elapsed_time(q) / n
flops = 2 * 2 * 4 * 32 * S * S * 128 / 2
acc["sdpa_tflops"] = flops / (acc["sdpa_ms"] / 1e3) / 1e12
acc["qkv_tops"] = 2 * 16384 * 6144 * 4096 / (acc["qkv_ms"] / 1e3) / 1e12
acc["o_tops"] = 2 * 16384 * 4096 * 4096 / (acc["o_ms"] / 1e3) / 1e12
try:
    from torch.nn.attention import SDPBackend, sdpa_kernel
    res = {}
    q = torch.randn(1, 32, 4096, 128, device="cuda", dtype=torch.bfloat16)
    k = torch.randn(1, 8, 4096, 128, device="cuda", dtype=torch.bfloat16)
    for b in (SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION, SDPBackend.EFFICIENT_ATTENTION):
        try:
            with sdpa_kernel([b]):
                torch.nn.functional.scaled_dot_product_attention(q, k, k, is_causal=True, enable_gqa=True)
            res[str(b)] = "ok"
        except Exception as exc:  # noqa: BLE001
            res[str(b)] = repr(exc)[:80]
    acc["backends"] = res
except Exception as exc:  # noqa: BLE001
    acc["backends"] = repr(exc)[:200]
print(json.dumps(acc))
