"""Per-config report (SURVEY.md §8d "Reported outputs: per config"): for
every BASELINE.json config, the B200 throughput (CUDA events), the int8
GEMM rate where GEMMs dominate, the oracle's CPU throughput on the same
inputs (bounded sample, this host's cores) and a parity verdict.

    python tools/config_report.py [--skip-c5] [out.json]  ->  prints JSON, writes profiles/configs_r01.json

Test infrastructure: the CPU legs call the oracle (checker / baseline only)."""
import json
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from oracle import moe_ref as M
from oracle import quant_ref as Q
from paper_2508_07329_b200 import _lib as L
from paper_2508_07329_b200 import ops
from paper_2508_07329_b200.linear import W8A8Linear
from paper_2508_07329_b200.moe import MoELayer, MoEStack
from paper_2508_07329_b200.quant import PER_TOKEN, QuantConfig
from paper_2508_07329_b200.trace import RoutingStats

PEAK = json.load(open("profiles/int8_peak.json"))["cublaslt_int8_burst"]


def bf16(a):
    return torch.from_numpy(np.asarray(a, np.float32)).bfloat16().float().numpy()


def dev_ms(fn, n=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def cpu_s(fn, budget=10.0, max_runs=3):
    times, end = [], time.perf_counter() + budget
    while not times or (time.perf_counter() < end and len(times) < max_runs):
        t0 = time.perf_counter()
        fn()
        times.append(time.perf_counter() - t0)
    return min(times)


def outliers(rng, T, d, frac=0.01, scale=100.0, cols=None):
    x = rng.normal(size=(T, d)).astype(np.float32)
    cols = rng.choice(d, max(1, int(d * frac)), replace=False) if cols is None else cols
    x[:, cols] *= scale
    return bf16(x)


def c1():
    """2-layer OPT-style FFN (d=256, ffn=1024, ReLU, residual), HAQ calibration + W8A8 forward, 512 tokens."""
    rng = np.random.default_rng(1)
    d, f, T = 256, 1024, 512
    x = outliers(rng, T, d, 0.02, 30.0).astype(np.float64)
    cfg = QuantConfig(8, False, PER_TOKEN)
    # warm-up: first-use costs (module loading, cuSOLVER handles, kernel
    # attributes) of both linear shapes out of the timing
    W8A8Linear.from_float(rng.normal(size=(f, d)) * 0.05, x.T.copy(), cfg)
    W8A8Linear.from_float(rng.normal(size=(d, f)) * 0.03, np.abs(rng.normal(size=(f, 512))), cfg)
    torch.cuda.synchronize()
    layers, parity, t_cal = [], True, 0.0
    h = x
    for _ in range(2):
        w1, w2 = rng.normal(size=(f, d)) * 0.05, rng.normal(size=(d, f)) * 0.03
        t0 = time.perf_counter()
        fc1 = W8A8Linear.from_float(w1, h.T.copy(), cfg, out_dtype=torch.float32)
        a = np.maximum(fc1(torch.from_numpy(h.astype(np.float32)).cuda()).double().cpu().numpy(), 0)
        fc2 = W8A8Linear.from_float(w2, a.astype(np.float32).astype(np.float64).T.copy(), cfg, out_dtype=torch.float32)
        torch.cuda.synchronize()
        t_cal += time.perf_counter() - t0
        o1 = Q.quantize_layer(w1, h.T, Q.cfg(8, False, PER_TOKEN))
        parity &= bool(np.array_equal(np.asarray(fc1.calibration.quantized.codes), o1["codes"]))
        layers.append((fc1, fc2))
        h = bf16(h + fc2(torch.from_numpy(a.astype(np.float32)).cuda()).double().cpu().numpy()).astype(np.float64)
    xd = torch.from_numpy(x.astype(np.float32)).cuda().bfloat16()

    def fwd():
        z = xd
        for fc1, fc2 in layers:
            z = (z.float() + fc2(torch.relu(fc1(z)).bfloat16()).float()).bfloat16()
        return z
    ms = dev_ms(fwd, 20)
    cpu_cal = cpu_s(lambda: Q.quantize_layer(rng.normal(size=(f, d)) * 0.05, x.T, Q.cfg(8, False, PER_TOKEN)), 20, 1)
    return {"config": "C1 tiny OPT FFN stack (2 layers, d=256, ffn=1024), 512 tokens",
            "gpu_forward_tokens_per_s": T / (ms / 1e3), "gpu_haq_calibration_s": t_cal,
            "cpu_oracle_quantize_layer_s_per_linear": cpu_cal,
            "gpu_haq_speedup_vs_cpu_oracle": (cpu_cal * 4) / t_cal,
            "parity": "codes bit-exact vs oracle quantize_layer" if parity else "MISMATCH"}


def c2():
    """Toy MoE d=1024, E=8, top-2, ffn=3584, 4096 tokens."""
    rng = np.random.default_rng(2)
    layer = MoELayer.random(8, 1024, 3584, seed=5, out_dtype=torch.float32)
    x = outliers(rng, 4096, 1024)
    xd = torch.from_numpy(x).cuda().bfloat16()
    ms = dev_ms(lambda: layer.forward(xd))
    g = layer.graphed(4096)
    ms_graph = dev_ms(lambda: g(xd))
    out, aux = layer.forward(xd, out_dtype=torch.float32, return_aux=True)
    experts = [layer.expert_host(e) for e in range(8)]
    lg = aux["logits"].cpu().numpy()
    ref, _, _ = M.moe_forward(x[:1024].astype(np.float64), None, experts, logits=lg[:1024])
    rel = float(np.linalg.norm(out[:1024].cpu().numpy() - ref) / np.linalg.norm(ref))
    deq = [{"s13": e["s13"], "s2": e["s2"], **{n: Q.dequant(e[f"{n}_codes"], e[f"{n}_scale"], e[f"{n}_zp"],
                                                            "per_output_row") for n in ("w1", "w3", "w2")}}
           for e in experts]
    cs = cpu_s(lambda: M.moe_forward_fakequant(x[:512].astype(np.float64), None, deq, 2, logits=lg[:512]), 15)
    ops_tok = 2 * 6 * 1024 * 3584
    return {"config": "C2 toy MoE d=1024 E=8 top-2 ffn=3584, 4096 tokens",
            "gpu_tokens_per_s": 4096 / (ms / 1e3), "gpu_ms": ms,
            "gpu_cuda_graph_tokens_per_s": 4096 / (ms_graph / 1e3), "gpu_cuda_graph_ms": ms_graph,
            "layer_int8_tops": 4096 * ops_tok / (min(ms, ms_graph) / 1e3) / 1e12,
            "cpu_oracle_fakequant_tokens_per_s": 512 / cs, "cpu_cores": os.cpu_count(),
            "parity": f"normwise rel. error vs float64 oracle on the GPU's logits: {rel:.2e} (stagewise bit-exact: "
                      "tests/test_gpu_moe.py::test_moe_c2_stagewise)"}


def c3():
    """OPT-6.7B FFN W8A8 (fc1 4096->16384, ReLU, fc2), 8192 tokens."""
    rng = np.random.default_rng(3)
    T, D, F = 8192, 4096, 16384
    x = torch.from_numpy(outliers(rng, T, D)).cuda().bfloat16()
    fc1 = W8A8Linear.from_rtn(torch.randn(F, D, device="cuda") * 0.02, smooth=np.exp(rng.normal(size=D) * 0.5))
    fc2 = W8A8Linear.from_rtn(torch.randn(D, F, device="cuda") * 0.02, smooth=np.exp(rng.normal(size=F) * 0.5))
    ms = dev_ms(lambda: fc2(torch.relu(fc1(x))))
    g1 = dev_ms(lambda: ops.w8a8_gemm(fc1.quantize_input(x), fc1.w, epilogue=L.EPI_DEQUANT,
                                      out_dtype=torch.bfloat16), 10) - dev_ms(lambda: fc1.quantize_input(x), 10)
    xs = x[:64].float().cpu().numpy().astype(np.float64)
    w1h = fc1.w["codes"].cpu().numpy()
    cs = cpu_s(lambda: M.w8a8_linear(*M.quantize_rows(xs, fc1.smooth.cpu().numpy()[0])[:3], w1h,
                                     fc1.w["scale"].cpu().numpy(), fc1.w["zp"].cpu().numpy()), 15)
    ops_ = 2 * T * D * F
    return {"config": "C3 OPT-6.7B FFN W8A8 (4096x16384), 8192 tokens",
            "gpu_tokens_per_s": T / (ms / 1e3), "gpu_ms": ms,
            "gemm_fc1_tops_approx": ops_ / (g1 / 1e3) / 1e12, "int8_peak_measured": PEAK,
            "cpu_oracle_fc1_tokens_per_s": 64 / cs, "cpu_cores": os.cpu_count(),
            "parity": "K1 codes and int32 accumulators bit-exact, dequant rtol 1e-5 "
                      "(tests/test_gpu_moe.py::test_w8a8_linear[8192-4096-16384])"}


def c5(L_=32, T=16384):
    """32-layer Mixtral-shape W8A8 MoE stack (no attention) on ONE B200, path statistics -> 8-rank placement."""
    from paper_2508_07329_b200.ep import plan_stack_placements
    t0 = time.perf_counter()
    stack = MoEStack.random(L_, 8, 4096, 14336, top_k=2, seed=7)
    for lay in stack.layers:         # keep only the GEMM operands (host-spec copies are not needed here)
        lay.host_experts = None
    torch.cuda.synchronize()
    init_s = time.perf_counter() - t0
    rng = np.random.default_rng(5)
    x = torch.from_numpy(outliers(rng, T, 4096)).cuda().bfloat16()
    ms = dev_ms(lambda: stack(x), 3, 1)
    stats = RoutingStats(L_, 8, 2)
    stack(x, stats=stats)
    pls = plan_stack_placements(stats, world=8)
    freq = stats.expert_freq().counts
    local = float(np.mean([pl.local_fraction(freq[l]) for l, pl in enumerate(pls)]))
    return {"config": f"C5-shape: {L_}-layer Mixtral W8A8 MoE stack (attention omitted), {T} tokens, 1 B200",
            "gpu_tokens_per_s_through_stack": T / (ms / 1e3), "gpu_ms_per_forward": ms, "init_s": init_s,
            "weights_gb": L_ * 1.41, "placement_8gpu_two_stage_local_fraction": local,
            "note": "EP at 2/4/8 GPUs not measured this round (one GPU per call); placement from GPU path stats"}


if __name__ == "__main__":
    out = {"gpu": torch.cuda.get_device_name(), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    for name, fn in (("C1", c1), ("C2", c2), ("C3", c3)):
        out[name] = fn()
        torch.cuda.empty_cache()
        print(name, json.dumps(out[name]), flush=True)
    if "--skip-c5" not in sys.argv:
        out["C5"] = c5()
        print("C5", json.dumps(out["C5"]), flush=True)
    path = next((a for a in sys.argv[1:] if a.endswith(".json")), "profiles/configs_r01.json")
    os.makedirs(os.path.dirname(path) or ".", exist_ok=True)
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
