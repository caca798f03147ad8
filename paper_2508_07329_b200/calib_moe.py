"""HAQ calibration of a whole MoE layer on the GPU.

The reference quantizes one linear layer at a time (``quantize_layer``,
quant.py:437-490: smoothing search, smoothed Hessian, compensated column
loop). For a MoE layer the paper applies it per expert on the activations
that expert actually sees (§III-B). This module composes the
per-layer operator into that calibration:

  1. route the calibration tokens with the layer's own router (K3);
  2. per expert e, gather the tokens routed to it;
  3. W1 and W3 share their input, so they are calibrated as one stacked
     matrix ``[W1; W3]`` with ONE smoothing vector s13 (the forward divides
     x by s13 once for both, fused into K1);
  4. the expert's float SwiGLU activation h = silu(x W1^T) * (x W3^T) of the
     same tokens calibrates W2 (smoothing s2, Hessian of h / s2);
  5. the quantized experts, their smoothing vectors and the router form a
     ``MoELayer`` (the W8A8 forward).

An expert that receives fewer than ``min_tokens`` calibration tokens is
calibrated on all tokens instead (its Hessian would be degenerate), and the
report says so. Everything runs through the device implementations of the
reference operators (K1/K2 losses, K7 Hessian, K8 column loop).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .moe import MoELayer
from .quant import DEFAULT_GRID_STEPS, ORDER_NONE, QuantConfig, QuantizedMatrix, quantize_layer


@dataclass
class ExpertCalibReport:
    expert: int
    tokens: int                 # calibration tokens routed to the expert
    used_all_tokens: bool       # fewer than min_tokens were routed: calibrated on all
    exponent13: float           # chosen smoothing exponents (search_smoothing)
    exponent2: float
    mse13: float                # output MSE of the quantized stacked W1/W3 (quantize_layer)
    rtn_mse13: float            # the RTN baseline of the same layer
    mse2: float
    rtn_mse2: float


def _silu(g: torch.Tensor) -> torch.Tensor:
    return g / (1.0 + torch.exp(-g))


def calibrate_moe_layer(gate_weight, experts_fp: list, x_calib: torch.Tensor, top_k: int = 2,
                        cfg: QuantConfig | None = None, grid_steps: int = DEFAULT_GRID_STEPS,
                        ordering: str = ORDER_NONE, gate_bias=None, min_tokens: int = 16,
                        out_dtype=torch.bfloat16) -> tuple[MoELayer, list]:
    """experts_fp[e] = {"w1": [F, d], "w3": [F, d], "w2": [d, F]} float weights
    (numpy or torch); x_calib [T, d] calibration tokens (CUDA tensor).
    Returns the W8A8 ``MoELayer`` and one ``ExpertCalibReport`` per expert."""
    cfg = cfg or QuantConfig(bits=8, symmetric=False, granularity="per_token")
    x = x_calib.cuda()
    if x.dim() != 2:
        raise ValueError("x_calib must be [T, d]")
    E = len(experts_fp)
    gw = torch.as_tensor(np.asarray(gate_weight, dtype=np.float32)).cuda().contiguous()
    gb = None if gate_bias is None else torch.as_tensor(np.asarray(gate_bias, dtype=np.float32)).cuda()
    if gw.shape != (E, x.shape[1]):
        raise ValueError(f"gate weight must be [{E}, {x.shape[1]}], got {tuple(gw.shape)}")
    _, idx, _ = ops.router_gate(x.to(torch.bfloat16).contiguous(), gw, top_k, gate_bias=gb)
    idx = idx.long()
    xf = x.to(torch.float64)
    experts, reports = [], []
    for e in range(E):
        ex = experts_fp[e]
        w1 = torch.as_tensor(np.asarray(ex["w1"]) if not isinstance(ex["w1"], torch.Tensor) else ex["w1"])
        w3 = torch.as_tensor(np.asarray(ex["w3"]) if not isinstance(ex["w3"], torch.Tensor) else ex["w3"])
        w2 = torch.as_tensor(np.asarray(ex["w2"]) if not isinstance(ex["w2"], torch.Tensor) else ex["w2"])
        w1, w3, w2 = (t.to(device="cuda", dtype=torch.float64) for t in (w1, w3, w2))
        F = w1.shape[0]
        tok = torch.nonzero((idx == e).any(dim=1)).flatten()
        used_all = tok.numel() < min_tokens
        xe = xf if used_all else xf[tok]
        # stacked [W1; W3] with one smoothing vector (shared input)
        r13 = quantize_layer(torch.cat([w1, w3], 0), xe.T.contiguous(), cfg, grid_steps, ordering)
        # W2 sees the expert's float SwiGLU activation of the same tokens
        h = _silu(xe @ w1.T) * (xe @ w3.T)
        r2 = quantize_layer(w2, h.T.contiguous(), cfg, grid_steps, ordering)
        q13 = r13.quantized
        codes13, sc13, zp13 = (np.asarray(q13.codes), np.asarray(q13.scales), np.asarray(q13.zero_points))
        experts.append({
            "w1": QuantizedMatrix(codes13[:F], sc13[:F], zp13[:F], cfg.bits, "per_output_row"),
            "w3": QuantizedMatrix(codes13[F:], sc13[F:], zp13[F:], cfg.bits, "per_output_row"),
            "w2": r2.quantized,
            "s13": np.asarray(r13.smoothing.factors, dtype=np.float64),
            "s2": np.asarray(r2.smoothing.factors, dtype=np.float64),
        })
        reports.append(ExpertCalibReport(e, int(tok.numel()), bool(used_all), r13.smoothing.exponent,
                                         r2.smoothing.exponent, r13.output_mse, r13.rtn_baseline_mse,
                                         r2.output_mse, r2.rtn_baseline_mse))
    layer = MoELayer(gw.cpu().numpy(), experts, top_k=top_k, out_dtype=out_dtype,
                     gate_bias=None if gb is None else gb.cpu().numpy())
    return layer, reports


def float_moe_forward(gate_weight, experts_fp: list, x: torch.Tensor, top_k: int = 2, gate_bias=None,
                      idx: torch.Tensor | None = None, w: torch.Tensor | None = None) -> torch.Tensor:
    """Float64 reference forward of the unquantized layer (quality checks):
    routing from the same K3 router unless (idx, w) are given."""
    xd = x.cuda()
    if idx is None:
        gw = torch.as_tensor(np.asarray(gate_weight, dtype=np.float32)).cuda().contiguous()
        gb = None if gate_bias is None else torch.as_tensor(np.asarray(gate_bias, dtype=np.float32)).cuda()
        _, idx, w = ops.router_gate(xd.to(torch.bfloat16).contiguous(), gw, top_k, gate_bias=gb)
    xf = xd.to(torch.float64)
    out = torch.zeros_like(xf)
    idx, w = idx.long(), w.to(torch.float64)
    for e, ex in enumerate(experts_fp):
        tok, slot = torch.nonzero(idx == e, as_tuple=True)
        if tok.numel() == 0:
            continue
        w1, w3, w2 = (torch.as_tensor(np.asarray(ex[k]) if not isinstance(ex[k], torch.Tensor) else ex[k]).to(
            device="cuda", dtype=torch.float64) for k in ("w1", "w3", "w2"))
        xe = xf[tok]
        y = (_silu(xe @ w1.T) * (xe @ w3.T)) @ w2.T
        out.index_add_(0, tok, w[tok, slot][:, None] * y)
    return out
