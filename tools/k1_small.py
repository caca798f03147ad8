"""K1 at small row counts (decode-size batches): the CTA-per-row kernel vs
the per-warp / bulk kernels, on the Mixtral-shape layer's x (gathered) and h
(with epilogue records), and the whole layer forward (CUDA graph) with
each choice — picks MOE_TUNE_K1_SMALL_ROWS.

    python tools/k1_small.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2508_07329_b200 import _lib as L
from paper_2508_07329_b200 import ops
from paper_2508_07329_b200.moe import MoELayer

layer = MoELayer.random(8, 4096, 14336, top_k=2, seed=1)
xall = torch.from_numpy(bench.synth_tokens(4096, 4096, 100)).to(torch.bfloat16).cuda()


def timeit(fn, n=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


for T in (1, 8, 16, 64, 128, 256, 512, 1024):
    x = xall[:T].contiguous()
    _, idx, w = layer.route(x)
    perm = ops.route_permute(idx, w, layer.E)
    R = T * layer.k

    def qx():
        return ops.act_quant(x, smooth=layer.s13, smooth_recip=layer.s13_recip, smooth_recip_f32=layer.s13_recip32,
                             row_group=perm["row_expert"], gather=perm["src_token"], rows=R)
    a1 = qx()
    ext = torch.empty((R, 2), dtype=torch.int64, device="cuda")
    h = ops.w8a8_gemm(a1, layer.w13, epilogue=L.EPI_SWIGLU, out_dtype=torch.bfloat16,
                      group_offsets=perm["offsets"], num_groups=layer.E, n_per_group=2 * layer.F,
                      next_smooth_recip_f32=layer.s2_recip32, row_ext=ext)

    def qh():
        return ops.act_quant(h, smooth=layer.s2, smooth_recip=layer.s2_recip, smooth_recip_f32=layer.s2_recip32,
                             row_group=perm["row_expert"], row_ext=ext)
    res = {}
    outs = {}
    for name, v in (("warp", 0), ("cta", 1 << 40)):
        with L.tuned(L.TUNE_K1_SMALL_ROWS, v):
            outs[name] = (qx(), qh())
            g = layer.graphed(T)
            res[name] = (timeit(qx), timeit(qh), timeit(lambda: g(x)))
            del g
    same = all(torch.equal(outs["warp"][i][k], outs["cta"][i][k]) for i in range(2)
               for k in ("codes", "scale", "zp", "rowsum"))
    f, r = res["warp"], res["cta"]
    print(f"T={T:5d} rows={R:5d}  quant_x warp {f[0]:6.1f} cta {r[0]:6.1f} us | quant_h warp {f[1]:6.1f} "
          f"cta {r[1]:6.1f} us | layer(graph) warp {f[2]:6.1f} cta {r[2]:6.1f} us  identical={same}", flush=True)
