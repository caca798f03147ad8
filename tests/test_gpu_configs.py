"""GPU: BASELINE.json configs not covered elsewhere.

C1 — tiny OPT-style decoder FFN stack (2 layers, d=256, ffn=1024, ReLU,
residual), HAQ-calibrated layer by layer on its own activations and run
W8A8 on 512 synthetic tokens: every linear's codes, scales, zero points and
smoothing factors equal the oracle's quantize_layer on identical inputs, and
each layer's output matches the float64 fake-quant forward."""

import numpy as np
import pytest
import torch

from oracle import quant_ref as Q
from paper_2508_07329_b200.linear import W8A8Linear
from paper_2508_07329_b200.quant import PER_TOKEN, QuantConfig

from .conftest import bf16_round

pytestmark = pytest.mark.gpu


def _fake_quant_linear(x_rows, codes, scales, zps, factors, bias):
    """Oracle forward of one W8A8 linear: dequant(Q(W f)) @ fake_quant(X / f) + b."""
    c = Q.cfg(8, False, PER_TOKEN)
    xs = (np.asarray(x_rows, np.float64) / factors).T               # channels x tokens
    y = Q.dequant(codes, scales, zps, Q.PER_OUTPUT_ROW) @ Q.fake_quant_acts(xs, c)
    return y.T + bias[None, :]


def test_c1_tiny_opt_ffn_stack(cuda):
    rng = np.random.default_rng(7)
    d, ffn, T, steps = 256, 1024, 512, 21
    x = rng.normal(size=(T, d)).astype(np.float32)
    x[:, rng.choice(d, 4, replace=False)] *= 30.0
    x = bf16_round(x).astype(np.float64)
    cfg = QuantConfig(bits=8, symmetric=False, granularity=PER_TOKEN)
    for layer in range(2):
        w1, b1 = rng.normal(size=(ffn, d)) * 0.05, (rng.normal(size=ffn) * 0.1).astype(np.float32)
        w2, b2 = rng.normal(size=(d, ffn)) * 0.03, (rng.normal(size=d) * 0.1).astype(np.float32)
        fc1 = W8A8Linear.from_float(w1, x.T.copy(), cfg, steps, bias=b1, out_dtype=torch.float32)
        o1 = Q.quantize_layer(w1, x.T, Q.cfg(8, False, PER_TOKEN), steps)
        q1 = fc1.calibration.quantized
        np.testing.assert_array_equal(np.asarray(q1.codes), o1["codes"])
        np.testing.assert_array_equal(np.asarray(q1.scales), o1["scales"])
        np.testing.assert_array_equal(np.asarray(q1.zero_points), o1["zero_points"])
        np.testing.assert_array_equal(fc1.calibration.smoothing.factors, o1["factors"])
        h_gpu = fc1(torch.from_numpy(x.astype(np.float32)).to(cuda)).double().cpu().numpy()
        h_ref = _fake_quant_linear(x, o1["codes"], o1["scales"], o1["zero_points"], o1["factors"], b1)
        np.testing.assert_allclose(h_gpu, h_ref, rtol=1e-4, atol=1e-4 * np.abs(h_ref).max())
        a = np.maximum(h_gpu, 0.0).astype(np.float32).astype(np.float64)   # ReLU, the GPU's own values
        fc2 = W8A8Linear.from_float(w2, a.T.copy(), cfg, steps, bias=b2, out_dtype=torch.float32)
        o2 = Q.quantize_layer(w2, a.T, Q.cfg(8, False, PER_TOKEN), steps)
        q2 = fc2.calibration.quantized
        np.testing.assert_array_equal(np.asarray(q2.codes), o2["codes"])
        np.testing.assert_array_equal(fc2.calibration.smoothing.factors, o2["factors"])
        y_gpu = fc2(torch.from_numpy(a.astype(np.float32)).to(cuda)).double().cpu().numpy()
        y_ref = _fake_quant_linear(a, o2["codes"], o2["scales"], o2["zero_points"], o2["factors"], b2)
        np.testing.assert_allclose(y_gpu, y_ref, rtol=1e-4, atol=1e-4 * np.abs(y_ref).max())
        assert fc1.calibration.output_mse == pytest.approx(o1["output_mse"], rel=1e-6)
        x = bf16_round((x + y_gpu).astype(np.float32)).astype(np.float64)   # residual, next layer's input
