"""Quick check of the CTA-pair (cta_group::2) GEMM path vs an exact float64 product."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2508_07329_b200 import ops, _lib as L
torch.manual_seed(0)
def operand(rows, K):
    c = torch.randint(0, 256, (rows, K), dtype=torch.uint8, device="cuda")
    zp = torch.randint(0, 256, (rows,), dtype=torch.int32, device="cuda")
    sc = torch.rand(rows, dtype=torch.float64, device="cuda") * 1e-3 + 1e-4
    return {"codes": c, "zp": zp, "scale": sc, "scale_f32": sc.float(), "rowsum": c.sum(1, dtype=torch.int32)}
for (M, N, K, G) in [(4096, 512, 1024, 1), (2500, 768, 4096, 1), (5000, 256, 512, 4)]:
    a, w = operand(M, K), operand(N * G, K)
    offs = None
    if G > 1:
        cuts = torch.tensor([0, 1100, 1101, 3000, M], dtype=torch.int32, device="cuda")
        offs = cuts
    acc = ops.w8a8_gemm(a, w, epilogue=L.EPI_ACC_I32, group_offsets=offs, num_groups=G, n_per_group=N)
    torch.cuda.synchronize()
    A = a["codes"].double() - a["zp"].double()[:, None]
    W = w["codes"].double() - w["zp"].double()[:, None]
    ok = True
    for g in range(G):
        lo, hi = (0, M) if offs is None else (int(offs[g]), int(offs[g + 1]))
        if hi == lo:
            continue
        ref = A[lo:hi] @ W[g * N:(g + 1) * N].T
        bad = (acc[lo:hi].double() != ref).sum().item()
        ok &= bad == 0
        print(M, N, K, G, "group", g, "mismatches", bad)
print("PAIR_OK" if ok else "PAIR_FAIL")
