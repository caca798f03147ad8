"""Where the grouped GEMMs' tensor pipe waits (debug library variant built
with -DMOE_GEMM_PROFILE=1: tools/build_variant.sh gemm_i8 prof
-DMOE_GEMM_PROFILE=1): per leader CTA, cycles the MMA issuer spends waiting
for a free accumulator (epilogue behind), for a full smem stage (operands
late), and the producer waiting for a free stage, over the issuer's whole
loop. Bench shape, one step, GEMM13 and GEMM2 separately.

    MOE_B200_LIB=paper_2508_07329_b200/lib/variants/libmoe_b200_prof.so python tools/gemm_waits.py"""
import ctypes
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_07329_b200 import _lib as L  # noqa: E402
from paper_2508_07329_b200 import ops  # noqa: E402
from paper_2508_07329_b200.moe import MoELayer  # noqa: E402

lib = L.load()
lib.moe_debug_gemm_waits.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros((1024, 6), dtype=np.uint64)


def read(reset=True):
    lib.moe_debug_gemm_waits(buf.ctypes.data, 1 if reset else 0)
    return buf.copy()


layer = MoELayer.random(8, 4096, 14336, top_k=2, seed=1)
x = torch.from_numpy(bench.synth_tokens(16384, 4096, 100)).to(torch.bfloat16).cuda()
for _ in range(3):
    layer.forward(x)
torch.cuda.synchronize()
_, idx, w = layer.route(x)
perm = ops.route_permute(idx, w, layer.E)
a1 = ops.act_quant_tokens(x, perm["token_pos"], perm["row_expert"], smooth=layer.s13, smooth_recip=layer.s13_recip,
                          smooth_recip_f32=layer.s13_recip32)
ext = torch.empty((idx.numel(), 2), dtype=torch.int64, device="cuda")
out = {}
read()
for rep in range(3):
    h = ops.w8a8_gemm(a1, layer.w13, epilogue=L.EPI_SWIGLU, out_dtype=torch.bfloat16, group_offsets=perm["offsets"],
                      num_groups=layer.E, n_per_group=2 * layer.F, next_smooth_recip_f32=layer.s2_recip32, row_ext=ext)
    g13 = read()
    a2 = ops.act_quant(h, smooth=layer.s2, smooth_recip=layer.s2_recip, smooth_recip_f32=layer.s2_recip32,
                       row_group=perm["row_expert"], row_ext=ext)
    read()
    y = ops.w8a8_gemm(a2, layer.w2, epilogue=L.EPI_DEQUANT, out_dtype=torch.bfloat16, row_weight=perm["row_weight"],
                      group_offsets=perm["offsets"], num_groups=layer.E, n_per_group=layer.d)
    g2 = read()
    for name, g in (("gemm13", g13), ("gemm2", g2)):
        lead = g[0:148:2].astype(np.float64)              # leader CTAs of the 74 pairs
        tot = lead[:, 3].sum()
        out.setdefault(name, []).append({"mma_wait_accumulator": lead[:, 0].sum() / tot,
                                         "mma_wait_operands_steady": lead[:, 1].sum() / tot,
                                         "mma_wait_operands_tile_start": lead[:, 4].sum() / tot,
                                         "producer_wait_stage": g[:148, 2].astype(np.float64).sum() / (2 * tot),
                                         "issuer_loop_mcycles_per_cta": tot / 74 / 1e6})
print(json.dumps(out, indent=1))
