"""A/B of the token-major K1 on x (and K1 on h) at the bench shape: CUDA-event
time per launch over `reps` launches; run once per library variant
(MOE_B200_LIB=...) and compare. Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_07329_b200 import _lib as L  # noqa: E402
from paper_2508_07329_b200 import ops  # noqa: E402
from paper_2508_07329_b200.moe import MoELayer  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
layer = MoELayer.random(8, 4096, 14336, top_k=2, seed=1)
x = torch.from_numpy(bench.synth_tokens(16384, 4096, 100)).to(torch.bfloat16).cuda()
_, idx, w = layer.route(x)
perm = ops.route_permute(idx, w, layer.E)
R = idx.numel()


def qx():
    return ops.act_quant_tokens(x, perm["token_pos"], perm["row_expert"], smooth=layer.s13,
                                smooth_recip=layer.s13_recip, smooth_recip_f32=layer.s13_recip32)


a1 = qx()
ext = torch.empty((R, 2), dtype=torch.int64, device="cuda")
h = ops.w8a8_gemm(a1, layer.w13, epilogue=L.EPI_SWIGLU, out_dtype=torch.bfloat16, group_offsets=perm["offsets"],
                  num_groups=layer.E, n_per_group=2 * layer.F, next_smooth_recip_f32=layer.s2_recip32, row_ext=ext)


def qh():
    return ops.act_quant(h, smooth=layer.s2, smooth_recip=layer.s2_recip, smooth_recip_f32=layer.s2_recip32,
                         row_group=perm["row_expert"], row_ext=ext)


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in evs:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) * 1000 for a, b in evs)
    return {"median_us": ts[len(ts) // 2], "min_us": ts[0]}


out = {"lib": os.environ.get("MOE_B200_LIB", "default"), "quant_h": timed(qh)}
for rnd in range(2):
    for mode in (1, 2):      # MOE_TUNE_K1_TOKENS: 1 token kernel, 2 token-major walk of the row kernel
        with L.tuned(L.TUNE_K1_TOKENS, mode):
            ref = qx()
            out.setdefault(f"quant_x_mode{mode}", []).append(timed(qx)["median_us"])
            out[f"codes_sum_mode{mode}"] = int(ref["codes"].sum(dtype=torch.int64))
            out[f"codes_eq_mode{mode}"] = bool(torch.equal(ref["codes"], a1["codes"]) and torch.equal(ref["scale"], a1["scale"]))
print(json.dumps(out), flush=True)
