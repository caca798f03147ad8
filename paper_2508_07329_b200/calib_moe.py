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


def swiglu_calib_acts(xe: torch.Tensor, w1: torch.Tensor, w3: torch.Tensor) -> torch.Tensor:
    """The float64 SwiGLU activation h = silu(x W1^T) * (x W3^T) [tokens, F]
    that calibrates W2 (oracle/calib_moe_ref.swiglu_acts)."""
    return _silu(xe @ w1.T) * (xe @ w3.T)


def _route_calib(gate_weight, x_calib, top_k, gate_bias, E):
    x = x_calib.cuda()
    if x.dim() != 2:
        raise ValueError("x_calib must be [T, d]")
    gw = torch.as_tensor(np.asarray(gate_weight, dtype=np.float32)).cuda().contiguous()
    gb = None if gate_bias is None else torch.as_tensor(np.asarray(gate_bias, dtype=np.float32)).cuda()
    if gw.shape != (E, x.shape[1]):
        raise ValueError(f"gate weight must be [{E}, {x.shape[1]}], got {tuple(gw.shape)}")
    _, idx, _ = ops.router_gate(x.to(torch.bfloat16).contiguous(), gw, top_k, gate_bias=gb)
    return gw, gb, idx.long(), x.to(torch.float64)


def _calibrate_expert(e: int, ex: dict, xf: torch.Tensor, idx: torch.Tensor, cfg: QuantConfig, grid_steps: int,
                      ordering: str, min_tokens: int) -> tuple[dict, "ExpertCalibReport"]:
    """HAQ for one expert from the calibration tokens routed to it."""
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
    h = swiglu_calib_acts(xe, w1, w3)
    r2 = quantize_layer(w2, h.T.contiguous(), cfg, grid_steps, ordering)
    q13 = r13.quantized
    codes13, sc13, zp13 = (np.asarray(q13.codes), np.asarray(q13.scales), np.asarray(q13.zero_points))
    out = {
        "w1": QuantizedMatrix(codes13[:F], sc13[:F], zp13[:F], cfg.bits, "per_output_row"),
        "w3": QuantizedMatrix(codes13[F:], sc13[F:], zp13[F:], cfg.bits, "per_output_row"),
        "w2": r2.quantized,
        "s13": np.asarray(r13.smoothing.factors, dtype=np.float64),
        "s2": np.asarray(r2.smoothing.factors, dtype=np.float64),
    }
    rep = ExpertCalibReport(e, int(tok.numel()), bool(used_all), r13.smoothing.exponent, r2.smoothing.exponent,
                            r13.output_mse, r13.rtn_baseline_mse, r2.output_mse, r2.rtn_baseline_mse)
    return out, rep


def calibrate_moe_layer(gate_weight, experts_fp: list, x_calib: torch.Tensor, top_k: int = 2,
                        cfg: QuantConfig | None = None, grid_steps: int = DEFAULT_GRID_STEPS,
                        ordering: str = ORDER_NONE, gate_bias=None, min_tokens: int = 16,
                        out_dtype=torch.bfloat16) -> tuple[MoELayer, list]:
    """experts_fp[e] = {"w1": [F, d], "w3": [F, d], "w2": [d, F]} float weights
    (numpy or torch); x_calib [T, d] calibration tokens (CUDA tensor).
    Returns the W8A8 ``MoELayer`` and one ``ExpertCalibReport`` per expert."""
    cfg = cfg or QuantConfig(bits=8, symmetric=False, granularity="per_token")
    E = len(experts_fp)
    gw, gb, idx, xf = _route_calib(gate_weight, x_calib, top_k, gate_bias, E)
    experts, reports = [], []
    for e in range(E):
        ex, rep = _calibrate_expert(e, experts_fp[e], xf, idx, cfg, grid_steps, ordering, min_tokens)
        experts.append(ex)
        reports.append(rep)
    layer = MoELayer(gw.cpu().numpy(), experts, top_k=top_k, out_dtype=out_dtype,
                     gate_bias=None if gb is None else gb.cpu().numpy())
    return layer, reports


def calibrate_moe_layer_distributed(gate_weight, experts_fp: list, x_calib: torch.Tensor, top_k: int = 2,
                                    cfg: QuantConfig | None = None, grid_steps: int = DEFAULT_GRID_STEPS,
                                    ordering: str = ORDER_NONE, gate_bias=None, min_tokens: int = 16,
                                    out_dtype=torch.bfloat16, group=None) -> tuple[MoELayer, list]:
    """calibrate_moe_layer with the experts spread over the ranks (expert e
    on rank e % world; every rank holds the same calibration tokens), the
    quantized experts broadcast from their owners: every rank returns the
    same layer, bit-identical to the single-GPU calibration (each expert's
    computation is the same)."""
    import torch.distributed as dist
    cfg = cfg or QuantConfig(bits=8, symmetric=False, granularity="per_token")
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    E = len(experts_fp)
    gw, gb, idx, xf = _route_calib(gate_weight, x_calib, top_k, gate_bias, E)
    mine = {e: _calibrate_expert(e, experts_fp[e], xf, idx, cfg, grid_steps, ordering, min_tokens)
            for e in range(E) if e % world == rank}
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"     # gloo: host tensors
    experts, reports = [], []
    for e in range(E):
        owner = e % world
        ex = experts_fp[e]
        F, d = np.asarray(ex["w1"]).shape if not isinstance(ex["w1"], torch.Tensor) else tuple(ex["w1"].shape)
        if owner == rank:
            out, rep = mine[e]
            t = {"c13": torch.from_numpy(np.concatenate([np.asarray(out["w1"].codes), np.asarray(out["w3"].codes)])
                                         .astype(np.uint8)),
                 "c2": torch.from_numpy(np.asarray(out["w2"].codes).astype(np.uint8)),
                 "p13": torch.from_numpy(np.concatenate([np.asarray(out["w1"].scales), np.asarray(out["w3"].scales),
                                                         np.asarray(out["w1"].zero_points),
                                                         np.asarray(out["w3"].zero_points)]).astype(np.float64)),
                 "p2": torch.from_numpy(np.concatenate([np.asarray(out["w2"].scales),
                                                        np.asarray(out["w2"].zero_points)]).astype(np.float64)),
                 "s": torch.from_numpy(np.concatenate([out["s13"], out["s2"]])),
                 "rep": torch.tensor([rep.tokens, int(rep.used_all_tokens), rep.exponent13, rep.exponent2,
                                      rep.mse13, rep.rtn_mse13, rep.mse2, rep.rtn_mse2], dtype=torch.float64)}
            t = {k: v.to(dev) for k, v in t.items()}
        else:
            t = {"c13": torch.empty((2 * F, d), dtype=torch.uint8, device=dev),
                 "c2": torch.empty((d, F), dtype=torch.uint8, device=dev),
                 "p13": torch.empty(4 * F, dtype=torch.float64, device=dev),
                 "p2": torch.empty(2 * d, dtype=torch.float64, device=dev),
                 "s": torch.empty(d + F, dtype=torch.float64, device=dev),
                 "rep": torch.empty(8, dtype=torch.float64, device=dev)}
        for k in ("c13", "c2", "p13", "p2", "s", "rep"):
            dist.broadcast(t[k], src=dist.get_global_rank(group, owner) if group is not None else owner,
                           group=group)
        c13, c2 = t["c13"].cpu().numpy().astype(np.int32), t["c2"].cpu().numpy().astype(np.int32)
        p13, p2, sv, r = (t[k].cpu().numpy() for k in ("p13", "p2", "s", "rep"))
        experts.append({
            "w1": QuantizedMatrix(c13[:F], p13[:F], p13[2 * F:3 * F].astype(np.int32), cfg.bits, "per_output_row"),
            "w3": QuantizedMatrix(c13[F:], p13[F:2 * F], p13[3 * F:].astype(np.int32), cfg.bits, "per_output_row"),
            "w2": QuantizedMatrix(c2, p2[:d], p2[d:].astype(np.int32), cfg.bits, "per_output_row"),
            "s13": sv[:d].copy(), "s2": sv[d:].copy()})
        reports.append(ExpertCalibReport(e, int(r[0]), bool(r[1]), float(r[2]), float(r[3]), float(r[4]),
                                         float(r[5]), float(r[6]), float(r[7])))
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
