"""Generate the golden vectors that pin the oracle to the UNMODIFIED reference.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``moekit`` from /root/reference/pkg/src, runs the reference's own
functions on seeded inputs and writes tests/golden/golden_*.npz. The GPU box
has no /root/reference, so the committed .npz files are what the tests read
there. Nothing here is imported by the product package.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def _bf16_round(a: np.ndarray) -> np.ndarray:
    """Round float32 values to bfloat16 (RNE) and return them as float64 -
    the exact values a bf16 GPU tensor holds."""
    f = np.asarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def main() -> None:
    sys.path.insert(0, str(REF))
    from moekit import placement, quant, trace  # noqa: E402  (reference, unmodified)
    from moekit.quant import QuantConfig

    g: dict[str, np.ndarray] = {}

    # 1. rounding known-answer test (test_quant.py:32-38 plus the fp64 edge)
    kat = np.array([0.5, -0.5, 1.5, 2.5, -2.5, 0.49, -0.49, 3.0,
                    0.49999999999999994, -0.49999999999999994, 254.5, -0.0, 1e-300])
    g["rha_in"] = kat
    g["rha_out"] = quant._round_half_away(kat)

    # 2. rtn_quantize across bits / symmetry / granularity
    rng = np.random.default_rng(1234)
    cases = []
    for bits in (2, 4, 8):
        for sym in (False, True):
            for gran in ("per_tensor", "per_token", "per_output_row"):
                cases.append((bits, sym, gran))
    for i, (bits, sym, gran) in enumerate(cases):
        x = rng.normal(size=(7, 33)) * rng.choice([1e-3, 1.0, 30.0], size=(7, 1))
        x[2] = 0.75                       # constant row -> scale floor path
        x[5, 3] = 500.0                   # outlier
        q = quant.rtn_quantize(x, QuantConfig(bits=bits, symmetric=sym, granularity=gran))
        g[f"rtn{i}_x"] = x
        g[f"rtn{i}_cfg"] = np.array([bits, int(sym), ("per_tensor", "per_token", "per_output_row").index(gran)])
        g[f"rtn{i}_codes"] = q.codes.astype(np.int32)
        g[f"rtn{i}_scales"] = q.scales
        g[f"rtn{i}_zps"] = q.zero_points
    g["rtn_ncases"] = np.array(len(cases))

    # 3. K1 semantics on bf16-representable activations: per-token RTN of
    #    x / s via the reference's own apply_smoothing + rtn_quantize
    tokens, chans = 64, 96
    xb = _bf16_round(rng.normal(size=(tokens, chans)) * np.where(rng.random(chans) < 0.05, 60.0, 1.0))
    s = np.maximum(np.abs(xb).max(axis=0), 1e-8) ** 0.55
    w_dummy = np.ones((1, chans))
    _, xs = quant.apply_smoothing(w_dummy, xb.T, s)          # channels x tokens
    qk = quant.rtn_quantize(xs.T, QuantConfig(bits=8, granularity="per_token"))
    g["k1_x_bf16"] = xb
    g["k1_smooth"] = s
    g["k1_codes"] = qk.codes.astype(np.int32)
    g["k1_scales"] = qk.scales
    g["k1_zps"] = qk.zero_points

    # 4-5. quant_loss and search_smoothing
    for i in range(4):
        w = rng.normal(size=(6, 12))
        x = rng.normal(size=(12, 40))
        x[int(rng.integers(0, 12))] *= 80.0
        f = np.exp(rng.normal(size=12))
        c = QuantConfig(bits=8, granularity=("per_tensor", "per_token")[i % 2])
        g[f"ql{i}_w"], g[f"ql{i}_x"], g[f"ql{i}_f"] = w, x, f
        g[f"ql{i}_gran"] = np.array(i % 2)
        g[f"ql{i}_loss"] = np.array(quant.quant_loss(w, x, f, c))
        sm = quant.search_smoothing(w, x, c)
        g[f"ss{i}_exp"] = np.array(sm.exponent)
        g[f"ss{i}_loss"] = np.array(sm.loss)
        g[f"ss{i}_factors"] = sm.factors

    # 6-8. Hessian, inverse factor, compensated quantization
    x = rng.normal(size=(24, 80))
    x[3] *= 40.0
    h = quant.build_hessian(x)
    g["hs_x"], g["hs_h"] = x, h
    g["hs_u"] = quant._inverse_upper_factor(h)
    w = rng.normal(size=(10, 24))
    for bits in (3, 4, 8):
        q = quant.hessian_quantize(w, h, QuantConfig(bits=bits))
        g[f"hq{bits}_codes"] = q.codes.astype(np.int32)
        g[f"hq{bits}_scales"] = q.scales
        g[f"hq{bits}_zps"] = q.zero_points
    order = rng.permutation(24)
    qo = quant.hessian_quantize(w, h, QuantConfig(bits=4), order=order)
    g["hs_w"], g["hq_order"], g["hqo_codes"] = w, order, qo.codes.astype(np.int32)

    # 9. full layer pipeline (a C1-like slice: 32 x 64 weight, 128 tokens)
    wl = rng.normal(size=(32, 64)) * 0.02
    xl = rng.normal(size=(64, 128))
    xl[[5, 40]] *= 100.0
    for j, ordering in enumerate(("none", "max_abs")):
        res = quant.quantize_layer(wl, xl, QuantConfig(bits=8, granularity="per_token"),
                                   ordering=ordering)
        g[f"ly{j}_codes"] = res.quantized.codes.astype(np.int32)
        g[f"ly{j}_scales"] = res.quantized.scales
        g[f"ly{j}_zps"] = res.quantized.zero_points
        g[f"ly{j}_exp"] = np.array(res.smoothing.exponent)
        g[f"ly{j}_loss"] = np.array(res.smoothing.loss)
        g[f"ly{j}_mse"] = np.array(res.output_mse)
        g[f"ly{j}_rtn_mse"] = np.array(res.rtn_baseline_mse)
    g["ly_w"], g["ly_x"] = wl, xl

    # 10. routing statistics and placement on reference-generated traces
    for j, seed in enumerate((0, 7)):
        tr = trace.generate_trace(trace.GenConfig(layers=32, experts_per_layer=8, top_k=2,
                                                  n_prefill_tokens=300, hot_path_prob=0.3,
                                                  zipf_s=1.2, seed=seed))
        paths = np.array([ev.path for ev in tr.events], dtype=np.int32)
        st = trace.path_stats(tr)
        fq = trace.expert_freq(tr)
        g[f"tr{j}_paths"] = paths
        g[f"tr{j}_freq"] = fq.counts
        g[f"tr{j}_stat_paths"] = np.array([p for p, _ in st.entries[:50]], dtype=np.int32)
        g[f"tr{j}_stat_counts"] = np.array([c for _, c in st.entries[:50]], dtype=np.int64)
        g[f"tr{j}_stat_n"] = np.array(len(st.entries))
        for name, plan in (("two", placement.plan_two_stage(st, fq, 2, 2)),
                           ("two23", placement.plan_two_stage(st, fq, 2, 3)),
                           ("freq", placement.plan_frequency(fq, 128)),
                           ("path", placement.plan_path(st, 128))):
            mask = np.zeros((32, 8), dtype=np.int8)
            for layer, r in enumerate(plan.residents):
                mask[layer, sorted(r)] = 1
            rep = placement.evaluate_plan(plan, tr)
            g[f"tr{j}_{name}_mask"] = mask
            g[f"tr{j}_{name}_eval"] = np.array([rep.mean, rep.std, rep.gap])

    # 11. MOEP packing (8-bit and 3-bit)
    for bits in (3, 8):
        wq = quant.rtn_quantize(rng.normal(size=(5, 11)), QuantConfig(bits=bits, granularity="per_output_row"))
        blob = quant.precision_pack(wq, quant.TARGET_GPU_INT).blob
        g[f"pk{bits}_codes"] = wq.codes.astype(np.int32)
        g[f"pk{bits}_scales"] = wq.scales
        g[f"pk{bits}_zps"] = wq.zero_points
        g[f"pk{bits}_blob"] = np.frombuffer(blob, dtype=np.uint8)

    np.savez_compressed(OUT / "golden_moekit.npz", **g)
    print(f"wrote {len(g)} arrays to {OUT / 'golden_moekit.npz'}")


if __name__ == "__main__":
    main()
