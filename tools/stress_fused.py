"""Randomised sweep of the layer's fused paths against their unfused
equivalents (same library, knobs flipped): the top-2 combine fused into
GEMM2, the token-major K1 on x, the producer-record K1 on h and the fused-K1
GEMM2 against GEMM2 + combine, the gathered K1 and the exact-extreme K1 —
the layer output must be bit-identical (raw bf16 bits) every way.

    python tools/stress_fused.py [seconds] [seed]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2508_07329_b200 import _lib as L  # noqa: E402
from paper_2508_07329_b200.moe import MoELayer  # noqa: E402
from tests.conftest import bf16_round  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 150.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 13)
layers = {}
t_end = time.time() + budget
n = fails = 0
while time.time() < t_end:
    d = int(rng.choice([256, 512, 1024]))
    F = int(rng.choice([256, 512, 768]))
    E = int(rng.choice([4, 8]))
    key = (d, F, E)
    if key not in layers:
        layers[key] = MoELayer.random(E, d, F, top_k=2, seed=len(layers) + 1)
    layer = layers[key]
    T = int(rng.integers(1, 4000))
    x = rng.normal(size=(T, d)).astype(np.float32)
    x[:, rng.choice(d, max(1, d // 100), replace=False)] *= 100.0
    xd = torch.from_numpy(bf16_round(x)).cuda().bfloat16()
    outs = []
    try:
        outs.append(layer.forward(xd))                                  # defaults
        with L.tuned(L.TUNE_FUSED_COMBINE, 0), L.tuned(L.TUNE_K1_TOKENS, 0):
            outs.append(layer.forward(xd))                              # unfused combine, gathered K1 on x
        with L.tuned(L.TUNE_K1_TOKENS, 1):
            outs.append(layer.forward(xd))                              # register token kernel
        with L.tuned(L.TUNE_FUSED_QUANT, 1):
            outs.append(layer.forward(xd))                              # K1 of h inside GEMM2
        with L.tuned(L.TUNE_K1_SMALL_ROWS, 1 << 40):
            outs.append(layer.forward(xd))                              # CTA-per-row K1 everywhere (no records)
        ok = all(torch.equal(o.view(torch.int16), outs[0].view(torch.int16)) for o in outs[1:])
    except Exception as e:   # noqa: BLE001
        ok = False
        print("error", repr(e)[:160], flush=True)
    n += 1
    fails += not ok
    print(f"T={T} d={d} F={F} E={E}: {'ok' if ok else 'FAIL'}", flush=True)
print(f"{n} configurations, {fails} failures", flush=True)
