"""Randomised stage-by-stage parity sweep of the MoE layer against the oracle
(the checks of tests/test_gpu_moe.py::_stagewise: routing, permutation, K1 on
x and on h bit-exact, GEMMs vs exact integer accumulators, combine) over
random shapes / expert counts / top-k / token counts, for a time budget.

    python tools/stress_parity.py [seconds] [seed]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from tests.test_gpu_moe import _stagewise  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 240.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 2024)
t_end = time.time() + budget
n = fails = 0
while time.time() < t_end:
    d = int(rng.choice([256, 384, 512, 1024, 1536]))
    F = int(rng.choice([256, 512, 640, 1024]))
    E = int(rng.choice([2, 4, 8, 16]))
    k = int(rng.choice([k for k in (1, 2, 4) if k <= E]))
    T = int(rng.integers(1, 5000))
    seed = int(rng.integers(0, 1 << 30))
    try:
        _stagewise(torch.device("cuda:0"), T, d, F, E=E, k=k, seed=seed)
        status = "ok"
    except AssertionError as e:
        fails += 1
        status = "FAIL " + str(e).splitlines()[0][:120]
    n += 1
    print(f"T={T} d={d} F={F} E={E} k={k} seed={seed}: {status}", flush=True)
print(f"{n} configurations, {fails} failures", flush=True)
