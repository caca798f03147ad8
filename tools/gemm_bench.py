"""Grouped GEMM variants at the bench shape (CUDA events, L2 flushed between
runs): GEMM13 with SwiGLU + extreme records (as in the step), SwiGLU only,
plain dequant epilogue, and GEMM2 — to see how much the epilogue costs."""
import sys

sys.path.insert(0, ".")
import torch

import bench
from paper_2508_07329_b200 import _lib as L
from paper_2508_07329_b200 import ops
from paper_2508_07329_b200.moe import MoELayer

T = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
layer = MoELayer.random(8, 4096, 14336, top_k=2, seed=1)
x = torch.from_numpy(bench.synth_tokens(T, 4096, 100)).to(torch.bfloat16).cuda()
_, idx, w = layer.route(x)
perm = ops.route_permute(idx, w, layer.E)
R = T * layer.k
a1 = ops.act_quant(x, smooth=layer.s13, smooth_recip=layer.s13_recip, smooth_recip_f32=layer.s13_recip32,
                   row_group=perm["row_expert"], gather=perm["src_token"], rows=R)
ext = torch.empty((R, 2), dtype=torch.int64, device="cuda")
h = torch.empty((R, layer.F), dtype=torch.bfloat16, device="cuda")
ybig = torch.empty((R, 2 * layer.F), dtype=torch.bfloat16, device="cuda")
G = dict(group_offsets=perm["offsets"], num_groups=layer.E)
variants = {
    "gemm13_swiglu_ext": lambda: ops.w8a8_gemm(a1, layer.w13, epilogue=L.EPI_SWIGLU, out=h, n_per_group=2 * layer.F,
                                               next_smooth_recip_f32=layer.s2_recip32, row_ext=ext, **G),
    "gemm13_swiglu": lambda: ops.w8a8_gemm(a1, layer.w13, epilogue=L.EPI_SWIGLU, out=h, n_per_group=2 * layer.F, **G),
    "gemm13_dequant_bf16": lambda: ops.w8a8_gemm(a1, layer.w13, epilogue=L.EPI_DEQUANT, out=ybig,
                                                 n_per_group=2 * layer.F, **G),
}
a2 = ops.act_quant(h, smooth=layer.s2, smooth_recip=layer.s2_recip, smooth_recip_f32=layer.s2_recip32,
                   row_group=perm["row_expert"])
y = torch.empty((R, layer.d), dtype=torch.bfloat16, device="cuda")
variants["gemm2"] = lambda: ops.w8a8_gemm(a2, layer.w2, epilogue=L.EPI_DEQUANT, out=y, row_weight=perm["row_weight"],
                                          n_per_group=layer.d, **G)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ops13 = 2 * R * 2 * layer.F * layer.d
for name, fn in variants.items():
    for _ in range(3):
        fn()
    ts = []
    for _ in range(15):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    ms = ts[len(ts) // 2]
    nops = ops13 if name != "gemm2" else 2 * R * layer.d * layer.F
    print(f"{name:22s} {ms:7.3f} ms  {nops / ms / 1e9:7.0f} TOPS")
