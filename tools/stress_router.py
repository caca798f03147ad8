"""Randomised sweep of the router (tensor-core cluster / persistent kernels
and the SIMT kernels) and the permutation against the oracle: random token
counts, widths, expert counts, top-k and gate biases. Logits within rtol
1e-5 of the float64 product (float32 accumulation), expert ids and
permutation bit-exact against the oracle's top-k on the GPU's own logits,
weights within float32 rounding; the tensor-core and SIMT logits agree.

    python tools/stress_router.py [seconds] [seed]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import moe_ref as M  # noqa: E402
from paper_2508_07329_b200 import ops  # noqa: E402
from tests.conftest import bf16_round  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 9)
t_end = time.time() + budget
n = fails = 0
while time.time() < t_end:
    T = int(rng.choice([int(rng.integers(1, 300)), int(rng.integers(300, 20000))]))
    d = int(rng.choice([int(rng.integers(1, 65)) * 64, int(rng.integers(8, 3000))]))
    E = int(rng.choice([2, 4, 8, 16, 32]))
    k = int(rng.integers(1, min(E, 8) + 1))
    x = bf16_round(rng.normal(size=(T, d)).astype(np.float32))
    wg = (rng.normal(size=(E, d)) / np.sqrt(d)).astype(np.float32)
    gb = rng.normal(size=E).astype(np.float32) if rng.random() < 0.5 else None
    xd = torch.from_numpy(x).cuda().bfloat16()
    gwd = torch.from_numpy(wg).cuda()
    gbd = torch.from_numpy(gb).cuda() if gb is not None else None
    ok = True
    try:
        lg, idx, w = ops.router_gate(xd, gwd, k, gate_bias=gbd)
        lg = lg.cpu().numpy()
        ref = M.gate_logits(x, wg) + (gb.astype(np.float64) if gb is not None else 0.0)
        ok &= np.allclose(lg, ref, rtol=1e-5, atol=1e-5 * max(1.0, np.abs(ref).max()))
        oidx, ow, _ = M.router_topk(lg, k)
        ok &= np.array_equal(idx.cpu().numpy(), oidx)
        ok &= np.allclose(w.cpu().numpy(), ow, rtol=1e-5, atol=1e-7)
        if d % 64 == 0 and E <= 16:          # both router families on the same rows
            lg2, idx2, _ = ops.router_gate(xd, gwd, k, gate_bias=gbd, tensor_cores=False)
            ok &= np.allclose(lg2.cpu().numpy(), lg, rtol=1e-5, atol=1e-5 * max(1.0, np.abs(ref).max()))
        perm = ops.route_permute(idx, w, E)
        offs, tok, slot, pos = M.permute(oidx, E)
        ok &= np.array_equal(perm["offsets"].cpu().numpy(), offs)
        ok &= np.array_equal(perm["src_token"].cpu().numpy(), tok)
        ok &= np.array_equal(perm["token_pos"].cpu().numpy().reshape(T, k), pos)
    except Exception as e:   # noqa: BLE001
        ok = False
        print("error", repr(e)[:160], flush=True)
    n += 1
    fails += not ok
    print(f"T={T} d={d} E={E} k={k} bias={gb is not None}: {'ok' if ok else 'FAIL'}", flush=True)
print(f"{n} configurations, {fails} failures", flush=True)
