"""GPU: HAQ calibration of a whole MoE layer — per-expert
routing of the calibration set, stacked W1/W3 with one smoothing vector,
W2 on the expert's SwiGLU activations — and the paper's quality claim on
held-out tokens: the HAQ-calibrated W8A8 layer is closer to the float layer
than plain per-row RTN weights without smoothing."""

import numpy as np
import pytest
import torch

from paper_2508_07329_b200 import ops, quant
from paper_2508_07329_b200.calib_moe import calibrate_moe_layer, float_moe_forward
from paper_2508_07329_b200.moe import MoELayer

pytestmark = pytest.mark.gpu

E, D, F, K = 4, 256, 256, 2


def _tokens(rng, T):
    x = rng.normal(size=(T, D))
    x[:, [3, 77, 190]] *= 40.0                      # outlier channels (the smoothing target)
    return torch.from_numpy(x.astype(np.float32)).cuda().bfloat16().float()


def _layer(rng):
    experts = [{"w1": rng.normal(size=(F, D)) * 0.05, "w3": rng.normal(size=(F, D)) * 0.05,
                "w2": rng.normal(size=(D, F)) * 0.05} for _ in range(E)]
    wg = rng.normal(size=(E, D)) / np.sqrt(D)
    return wg.astype(np.float32), experts


def test_calibrate_moe_layer_quality(cuda):
    rng = np.random.default_rng(0)
    wg, experts = _layer(rng)
    x_cal, x_test = _tokens(rng, 1024), _tokens(rng, 512)
    layer, rep = calibrate_moe_layer(wg, experts, x_cal, top_k=K, grid_steps=11, out_dtype=torch.float32)
    # routing of the calibration set
    _, idx, _ = ops.router_gate(x_cal.bfloat16().contiguous(), torch.from_numpy(wg).cuda(), K)
    counts = [(idx == e).any(dim=1).sum().item() for e in range(E)]
    assert [r.tokens for r in rep] == counts
    assert sum(counts) == 1024 * K
    # expert 0's stacked W1/W3 is exactly the per-layer operator on its tokens
    tok = torch.nonzero((idx.long() == 0).any(dim=1)).flatten()
    xe = x_cal.double()[tok]
    w13 = np.concatenate([experts[0]["w1"], experts[0]["w3"]])
    r = quant.quantize_layer(w13, xe.T.contiguous(), quant.QuantConfig(granularity="per_token"), 11)
    np.testing.assert_array_equal(np.asarray(r.quantized.codes[:F]), layer.host_experts[0]["w1"].codes)
    np.testing.assert_array_equal(r.smoothing.factors, layer.host_experts[0]["s13"])
    # every expert beats (or matches) its RTN baseline on its own calibration set
    for rp in rep:
        assert rp.mse13 <= rp.rtn_mse13 * 1.0001 and rp.mse2 <= rp.rtn_mse2 * 1.0001
    # held-out quality vs float, and vs RTN weights without smoothing
    ref = float_moe_forward(wg, experts, x_test, K)
    haq = layer.forward(x_test.bfloat16()).double()
    rtn_experts = []
    for ex in experts:
        d = {k: quant.rtn_quantize(np.asarray(ex[k]), quant.QuantConfig(granularity="per_output_row"))
             for k in ("w1", "w3", "w2")}
        d.update(s13=np.ones(D), s2=np.ones(F))
        rtn_experts.append(d)
    rtn = MoELayer(wg, rtn_experts, top_k=K, out_dtype=torch.float32).forward(x_test.bfloat16()).double()
    err = lambda y: (torch.linalg.norm(y - ref) / torch.linalg.norm(ref)).item()   # noqa: E731
    e_haq, e_rtn = err(haq), err(rtn)
    assert e_haq < 0.05, e_haq
    assert e_haq < e_rtn, (e_haq, e_rtn)
