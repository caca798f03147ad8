"""Randomised sweep of the grouped W8A8 GEMM (moe_w8a8_gemm) against the
oracle's exact integer accumulators: random group counts and (possibly
empty, ragged) group sizes — crossing the single-CTA / CTA-pair threshold of
2048 rows —, N off the 256-wide tile, K off the 128-byte k-block (and K not
a multiple of 16: the SIMT path), random zero points; the ACC_I32 epilogue
must be bit-exact, DEQUANT within rtol 1e-5 of the float64 oracle on the
same accumulators.

    python tools/stress_gemm.py [seconds] [seed]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import moe_ref as M  # noqa: E402
from paper_2508_07329_b200 import _lib as L  # noqa: E402
from paper_2508_07329_b200 import ops  # noqa: E402
from tests.test_gpu_kernels import _dev_operand, _rand_operand  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 180.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 3)
t_end = time.time() + budget
n = fails = 0
while time.time() < t_end:
    G = int(rng.integers(1, 9))
    sizes = rng.integers(0, 1200, size=G)
    sizes[rng.random(G) < 0.2] = 0
    if sizes.sum() == 0:
        sizes[0] = int(rng.integers(1, 300))
    Mt = int(sizes.sum())
    N = int(rng.choice([int(rng.integers(1, 65)) * 8, 256, 512, 768]))
    K = int(rng.choice([int(rng.integers(1, 40)) * 16, int(rng.integers(8, 1200)), 4096, 1040]))
    cuda = torch.device("cuda:0")
    a = _rand_operand(rng, Mt, K)
    w = _rand_operand(rng, G * N, K)
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
    ad, wd = _dev_operand(cuda, *a), _dev_operand(cuda, *w)
    od = torch.from_numpy(offs).to(cuda)
    ok = True
    try:
        acc = ops.w8a8_gemm(ad, wd, epilogue=L.EPI_ACC_I32, group_offsets=od, num_groups=G, n_per_group=N)
        y = ops.w8a8_gemm(ad, wd, epilogue=L.EPI_DEQUANT, out_dtype=torch.float32, group_offsets=od, num_groups=G,
                          n_per_group=N)
        acc, y = acc.cpu().numpy(), y.cpu().numpy()
        for g in range(G):
            lo, hi = offs[g], offs[g + 1]
            if hi == lo:
                continue
            wc, wz, ws = (v[g * N:(g + 1) * N] for v in w)
            yr, accr = M.w8a8_linear(a[0][lo:hi], a[2][lo:hi], a[1][lo:hi], wc, ws, wz)
            ok &= np.array_equal(acc[lo:hi], accr)
            ok &= np.allclose(y[lo:hi], yr, rtol=1e-5, atol=1e-6 * max(1e-30, np.abs(yr).max()))
    except Exception as e:   # noqa: BLE001
        ok = False
        print("error", repr(e)[:160], flush=True)
    n += 1
    fails += not ok
    print(f"G={G} rows={Mt} sizes={sizes.tolist()} N={N} K={K}: {'ok' if ok else 'FAIL'}", flush=True)
print(f"{n} configurations, {fails} failures", flush=True)
