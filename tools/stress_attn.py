"""Randomised sweep of the C5 attention half (W8A8 QKV, RoPE, causal GQA
SDPA, W8A8 output projection) against the float64 oracle, stage by stage
(tests/test_gpu_moe.py::_attention_stagewise) over random widths, head
counts, GQA ratios, head dims and packed sequence lengths.

    python tools/stress_attn.py [seconds] [seed]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from tests.test_gpu_moe import _attention_stagewise  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 23)
t_end = time.time() + budget
n = fails = 0
while time.time() < t_end:
    hd = int(rng.choice([32, 64, 128]))
    Hk = int(rng.choice([1, 2, 4]))
    H = Hk * int(rng.choice([1, 2, 4]))
    d = int(rng.choice([256, 512, 768]))
    S = int(rng.choice([16, 64, 128, 256]))
    B = int(rng.integers(1, 5))
    seed = int(rng.integers(0, 1 << 20))
    try:
        _attention_stagewise(d, H, Hk, hd, S, B, seed=seed)
        status = "ok"
    except AssertionError as e:
        fails += 1
        status = "FAIL " + str(e).splitlines()[0][:120]
    n += 1
    print(f"d={d} H={H} Hk={Hk} hd={hd} S={S} B={B} seed={seed}: {status}", flush=True)
print(f"{n} configurations, {fails} failures", flush=True)
