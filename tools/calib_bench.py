"""Calibration path on the B200 next to the reference functions on the box's
host cores, at the Mixtral expert
shapes: stacked W1||W3 [28672, 4096] and W2 [4096, 14336], T routed
calibration tokens.

Per stage, GPU (CUDA events, after a warm-up) and CPU (the oracle's
restatement of the reference function, oracle/quant_ref.py, numpy/OpenBLAS
on all host threads, best of `reps`):
  rtn_quantize      per-token RTN of the activations       (quant.py:214-231)
  quant_loss        one smoothing grid point               (quant.py:267-283)
  search_smoothing  21 quant_loss evaluations            (quant.py:286-311)
  build_hessian     K7, 2 n^2 T flops (full product)      (quant.py:327-343)
  inverse factor    damped inverse + Cholesky              (quant.py:366-385)
  column loop       K8, R n (n-1) flops                   (quant.py:415-434)
CPU timings of shapes that take minutes-hours in the oracle are taken on a
slice and scaled (labelled): search_smoothing and the column loop on a row
slice (linear in R: rows are independent), build_hessian on a token slice
(linear in T), the inverse factor at a smaller n (cubic in n).

    python tools/calib_bench.py [T] [out.json]   (on gpurun: write the json under gpurun_out/)
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import quant_ref as Q  # noqa: E402
from paper_2508_07329_b200 import ops, quant  # noqa: E402
from paper_2508_07329_b200.quant import QuantConfig  # noqa: E402

FP64_SPEC_TFLOPS = 40.0       # B200 FP64 (spec; no measured FP64 peak in MEASURED_PEAKS.json)


def gpu_time(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        t = a.elapsed_time(b) / 1000.0
        best = t if best is None else min(best, t)
    return best


def cpu_time(fn, reps=3, budget=60.0):
    best, t_all = None, time.perf_counter()
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        t = time.perf_counter() - t0
        best = t if best is None else min(best, t)
        if time.perf_counter() - t_all > budget:
            break
    return best


def main():
    T = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 1024
    out_path = next((a for a in sys.argv[1:] if a.endswith(".json")), None)
    rng = np.random.default_rng(0)
    cfg = QuantConfig(bits=8, symmetric=False, granularity="per_token")
    c = Q.cfg(8, False, Q.PER_TOKEN)
    res = {"tokens": T, "host": {"cpu_count": os.cpu_count(), "numpy": np.__version__},
           "fp64_peak_tflops": FP64_SPEC_TFLOPS, "fp64_peak_source": "B200 spec (not measured)", "shapes": {}}
    try:
        import subprocess
        res["host"]["lscpu_model"] = next((ln.split(":", 1)[1].strip() for ln in subprocess.run(
            ["lscpu"], capture_output=True, text=True).stdout.splitlines() if ln.startswith("Model name")), None)
    except Exception:
        pass
    for name, (R, n) in {"w13": (28672, 4096), "w2": (4096, 14336)}.items():
        w = rng.normal(size=(R, n)) * 0.02
        x = rng.normal(size=(n, T))
        x[rng.choice(n, n // 100, replace=False)] *= 50.0
        wd, xd = torch.from_numpy(w).cuda(), torch.from_numpy(x).cuda()
        r = {"rows": R, "cols": n}
        # -- GPU stages --------------------------------------------------
        r["gpu_search_smoothing_s"] = gpu_time(lambda: quant.search_smoothing(wd, xd, cfg))
        sm = quant.search_smoothing(wd, xd, cfg)
        f = torch.from_numpy(np.asarray(sm.factors)).cuda()
        ws, xs = ops.apply_smoothing(wd, xd, f)
        xt = xs.T.contiguous()
        r["gpu_build_hessian_s"] = gpu_time(lambda: ops.hessian(xt))
        H = ops.hessian(xt)
        r["k7_tflops"] = 2.0 * n * n * T / r["gpu_build_hessian_s"] / 1e12
        r["k7_frac_fp64_spec"] = r["k7_tflops"] / FP64_SPEC_TFLOPS
        r["gpu_inverse_factor_s"] = gpu_time(lambda: quant._inverse_upper_factor_device(H))
        U = quant._inverse_upper_factor_device(H)
        prm = quant._k1(ws, cfg, quant.PER_OUTPUT_ROW)
        r["gpu_column_loop_s"] = gpu_time(lambda: ops.gptq_columns(ws, U, prm["scale"], prm["zp"], 8))
        r["k8_tflops"] = R * n * (n - 1) / r["gpu_column_loop_s"] / 1e12
        r["k8_frac_fp64_spec"] = r["k8_tflops"] / FP64_SPEC_TFLOPS
        r["gpu_quantize_layer_s"] = gpu_time(lambda: quant.quantize_layer(wd, xd, cfg), reps=1)
        # -- CPU (oracle port of the reference functions) ----------------
        rs = 256                                           # row slice
        t = cpu_time(lambda: Q.search_smoothing(w[:rs], x, c, 21), reps=1)
        r["cpu_search_smoothing_s"] = t * R / rs
        r["cpu_search_smoothing_note"] = f"{rs}-row slice x {R / rs:.0f} (linear in R)"
        ts = 256                                           # token slice
        t = cpu_time(lambda: Q.build_hessian(x[:, :ts]))
        r["cpu_build_hessian_s"] = t * T / ts
        r["cpu_build_hessian_note"] = f"{ts}-token slice x {T / ts:.0f} (linear in T)"
        n_small = 1024
        hs = Q.build_hessian(x[:n_small])
        t = cpu_time(lambda: Q.inverse_upper_factor(hs), reps=1)
        r["cpu_inverse_factor_s"] = t * (n / n_small) ** 3
        r["cpu_inverse_factor_note"] = f"measured at n={n_small} ({t:.2f} s), x (n/{n_small})^3"
        rr = 32
        Uh = U.cpu().numpy()
        wsh = ws[:rr].cpu().numpy()
        sc, zp = prm["scale"][:rr].cpu().numpy(), prm["zp"][:rr].cpu().numpy()
        t = cpu_time(lambda: Q.gptq_columns(wsh, Uh, sc, zp, 255), reps=1)
        r["cpu_column_loop_s"] = t * R / rr
        r["cpu_column_loop_note"] = f"{rr}-row slice x {R / rr:.0f} (rows independent)"
        # a6 rtn_quantize of the calibration activations (per token, X channels x tokens) and
        # a11 quant_loss at exponent 0.5 (one grid point of the search)
        xtok = torch.from_numpy(x.T.copy()).cuda()
        r["gpu_rtn_quantize_s"] = gpu_time(lambda: quant.rtn_quantize(xd, cfg))
        t = cpu_time(lambda: Q.rtn(x, c))
        r["cpu_rtn_quantize_s"] = t
        f05 = np.maximum(np.abs(x).max(axis=1), 1e-8) ** 0.5
        r["gpu_quant_loss_s"] = gpu_time(lambda: quant.quant_loss(wd, xd, f05, cfg))
        t = cpu_time(lambda: Q.quant_loss(w[:rs], x, f05, c), reps=1)
        r["cpu_quant_loss_s"] = t * R / rs
        r["cpu_quant_loss_note"] = f"{rs}-row slice x {R / rs:.0f} (linear in R)"
        del xtok
        for k in ("search_smoothing", "build_hessian", "inverse_factor", "column_loop", "rtn_quantize", "quant_loss"):
            r[f"speedup_{k}"] = r[f"cpu_{k}_s"] / r[f"gpu_{k}_s"]
        res["shapes"][name] = r
        print(name, json.dumps(r), flush=True)
    if out_path:
        json.dump(res, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main()
