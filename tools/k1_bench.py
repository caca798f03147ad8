"""K1 micro-benchmark at the bench shape: quant_x (gathered x, pass A) and
quant_h (h with epilogue records), per launch configuration
(MOE_B200_K1_CFG), CUDA-event timed, plus HBM GB/s of the algorithmic bytes."""
import os
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


def qx():
    return ops.act_quant(x, smooth=layer.s13, smooth_recip=layer.s13_recip, smooth_recip_f32=layer.s13_recip32,
                         row_group=perm["row_expert"], gather=perm["src_token"], rows=R)


a1 = qx()
ext = torch.empty((R, 2), dtype=torch.int64, device="cuda")
h = ops.w8a8_gemm(a1, layer.w13, epilogue=L.EPI_SWIGLU, out_dtype=torch.bfloat16, group_offsets=perm["offsets"],
                  num_groups=layer.E, n_per_group=2 * layer.F, next_smooth_recip_f32=layer.s2_recip32, row_ext=ext)


def qh():
    return ops.act_quant(h, smooth=layer.s2, smooth_recip=layer.s2_recip, smooth_recip_f32=layer.s2_recip32,
                         row_group=perm["row_expert"], row_ext=ext)


def qh_plain():
    return ops.act_quant(h, smooth=layer.s2, smooth_recip=layer.s2_recip, smooth_recip_f32=layer.s2_recip32,
                         row_group=perm["row_expert"])


flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(n):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


if os.environ.get("K1_PROF"):
    for _ in range(2):
        qx()
        qh()
    torch.cuda.synchronize()
    print("ok")
    sys.exit(0)
ref_x, ref_h = qx(), qh_plain()
bytes_x = R * 4096 * 2 + R * 4096       # gathered bf16 rows read + codes written
bytes_h = R * 14336 * 2 + R * 14336
for cfg in sys.argv[2].split(",") if len(sys.argv) > 2 else ("-1", "0", "7"):
    os.environ["MOE_B200_K1_CFG"] = cfg
    gx, gh = qx(), qh()
    ok = all(torch.equal(gx[k], ref_x[k]) for k in ("codes", "scale", "zp", "rowsum")) and \
        all(torch.equal(gh[k], ref_h[k]) for k in ("codes", "scale", "zp", "rowsum"))
    tx, th, tp = timeit(qx), timeit(qh), timeit(qh_plain)
    print(f"cfg {cfg}: quant_x {tx*1e3:7.1f} us ({bytes_x/tx/1e6:6.0f} GB/s)  quant_h {th*1e3:7.1f} us "
          f"({bytes_h/th/1e6:6.0f} GB/s)  quant_h(no records) {tp*1e3:7.1f} us  match={ok}")
