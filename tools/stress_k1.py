"""Randomised sweep of K1 (moe_act_quant through ops.act_quant) against the
oracle's float64 restatement of rtn_quantize / apply_smoothing: random row
and column counts (ragged), input dtypes, bit widths, symmetric / asymmetric,
per-tensor / per-token, smoothing by division (grouped tables, optional
gather) or multiplication, producer records for bf16 rows, and the CTA-per-row
/ per-warp / bulk kernels; codes, scales, zero points and row sums must be
bit-identical.

    python tools/stress_k1.py [seconds] [seed]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import quant_ref as Q  # noqa: E402
from paper_2508_07329_b200 import _lib as L  # noqa: E402
from paper_2508_07329_b200 import ops  # noqa: E402
from tests.conftest import bf16_round  # noqa: E402
from tests.test_gpu_kernels import _true_records  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 180.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 5)
t_end = time.time() + budget
n = fails = 0
DT = {"bf16": torch.bfloat16, "f32": torch.float32, "f64": torch.float64, "f16": torch.float16}
while time.time() < t_end:
    rows = int(rng.integers(1, 2500))
    cols = int(rng.choice([int(rng.integers(1, 300)), int(rng.integers(1, 600)) * 8, 4096, 14336]))
    dt = str(rng.choice(list(DT)))
    bits = int(rng.integers(2, 9))
    sym = bool(rng.random() < 0.25)
    gran = "per_tensor" if rng.random() < 0.15 else "per_token"
    mode = str(rng.choice(["none", "divide", "multiply"]))
    small = bool(rng.random() < 0.3)
    x = rng.normal(size=(rows, cols)) * np.exp(rng.normal(size=(rows, 1)))
    x[:, rng.choice(cols, max(1, cols // 100), replace=False)] *= 100.0
    if rng.random() < 0.1:
        x = np.maximum(x, 0.0)                          # one-sided rows
    if dt == "bf16":
        x = bf16_round(x.astype(np.float32)).astype(np.float64)
    elif dt == "f16":
        x = x.astype(np.float16).astype(np.float64)
    elif dt == "f32":
        x = x.astype(np.float32).astype(np.float64)
    G = int(rng.integers(1, 6))
    s = np.exp(rng.normal(size=(G, cols)) * 0.7)
    group = rng.integers(0, G, size=rows).astype(np.int32)
    gather = rng.integers(0, rows, size=rows).astype(np.int32) if (mode == "divide" and rng.random() < 0.3) else None
    xd = torch.from_numpy(x).cuda().to(DT[dt])
    kw = {"bits": bits, "symmetric": sym, "granularity": gran}
    xin = x[gather] if gather is not None else x
    if mode == "none":
        xs = xin
    elif mode == "divide":
        xs = xin / s[group]
        kw.update(smooth=torch.from_numpy(s).cuda(), row_group=torch.from_numpy(group).cuda(),
                  gather=torch.from_numpy(gather).cuda() if gather is not None else None)
    else:
        xs = xin * s[0]
        kw.update(smooth=torch.from_numpy(s[:1]).cuda(), smooth_mode=L.SMOOTH_MULTIPLY)
    if gran == "per_tensor" and mode == "divide":
        kw.pop("row_group"); xs = xin / s[0]; kw["smooth"] = torch.from_numpy(s[:1]).cuda()
    use_rec = (dt == "bf16" and mode == "divide" and gran == "per_token" and gather is None and bits == 8
               and not sym and cols % 8 == 0 and rng.random() < 0.5)
    if use_rec:
        kw["row_ext"] = torch.from_numpy(_true_records(x.astype(np.float32),
                                                       (1.0 / s).astype(np.float32)[group])).cuda()
    codes, sc, zp = Q.rtn(xs, Q.cfg(bits, sym, gran))
    try:
        with L.tuned(L.TUNE_K1_SMALL_ROWS, 1 << 40 if small else 256):
            r = ops.act_quant(xd, **kw)
        ok = (np.array_equal(r["codes"].cpu().numpy(), codes) and np.array_equal(r["scale"].cpu().numpy(), sc)
              and np.array_equal(r["zp"].cpu().numpy(), zp))
        if ok and r["rowsum"] is not None and gran == "per_token":
            ok = np.array_equal(r["rowsum"].cpu().numpy(), codes.astype(np.int64).sum(1))
    except Exception as e:   # noqa: BLE001
        ok = False
        print("error", repr(e)[:160], flush=True)
    n += 1
    fails += not ok
    print(f"rows={rows} cols={cols} {dt} bits={bits} sym={sym} {gran} {mode} gather={gather is not None} "
          f"rec={use_rec} cta={small}: {'ok' if ok else 'FAIL'}", flush=True)
print(f"{n} configurations, {fails} failures", flush=True)
