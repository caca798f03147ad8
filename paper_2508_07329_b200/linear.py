"""W8A8Linear: the forward counterpart of the reference's fake-quant product
(quant.py:281-283, 475-478) as a real INT8 tensor-core linear layer.

y = dequant( Q_tok(x / s) . Q_row(W s)^T ) (+ bias): per-token activation
quantization of the smoothed input (K1, exact reference semantics) feeds the
tcgen05 kind::i8 GEMM (K2) whose epilogue applies the zero-point correction,
the per-token x per-output-channel scales and the bias.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from . import ops
from .quant import PER_OUTPUT_ROW, PER_TOKEN, QuantConfig, QuantizedMatrix, quantize_layer


class W8A8Linear:
    def __init__(self, weight: QuantizedMatrix, smooth=None, bias=None, act_bits: int = 8,
                 act_symmetric: bool = False, out_dtype=torch.bfloat16):
        if weight.granularity != PER_OUTPUT_ROW:
            raise ValueError("W8A8Linear weights must be quantized per output row")
        self.w = ops.with_wcorr(weight.device())     # pre-corrected sidecar: 2 IMADs per accumulator
        self.out_features, self.in_features = self.w["codes"].shape
        self.smooth = None
        self.smooth_recip = None
        self.smooth_recip_f32 = None
        if smooth is not None:
            s = torch.as_tensor(np.asarray(smooth.cpu() if isinstance(smooth, torch.Tensor) else smooth),
                                dtype=torch.float64).reshape(1, -1).cuda()
            if s.shape[1] != self.in_features:
                raise ValueError(f"expected {self.in_features} smoothing factors, got {s.shape[1]}")
            self.smooth = s
            self.smooth_recip, self.smooth_recip_f32 = ops.reciprocal(s, with_f32=True)
        self.bias = None if bias is None else torch.as_tensor(bias, dtype=torch.float32).reshape(-1).cuda()
        self.act_bits, self.act_symmetric, self.out_dtype = act_bits, act_symmetric, out_dtype

    @classmethod
    def from_float(cls, w, x_calib, cfg: QuantConfig | None = None, grid_steps: int = 21, ordering: str = "none",
                   bias=None, out_dtype=torch.bfloat16):
        """HAQ-calibrate a float weight [out, in] on calibration activations
        [in, tokens] (quantize_layer on device) and wrap the result."""
        cfg = cfg or QuantConfig(granularity=PER_TOKEN)
        res = quantize_layer(w, x_calib, cfg, grid_steps, ordering)
        lin = cls(res.quantized, res.smoothing.factors, bias, cfg.bits, cfg.symmetric, out_dtype)
        lin.calibration = res
        return lin

    @classmethod
    def from_rtn(cls, w: torch.Tensor, smooth=None, bias=None, bits: int = 8, out_dtype=torch.bfloat16):
        """Plain per-output-row RTN of (W diag s) on device."""
        wd = w.cuda().to(torch.float32).contiguous()
        sm = None if smooth is None else torch.as_tensor(smooth, dtype=torch.float64).reshape(1, -1).cuda()
        q = ops.act_quant(wd, smooth=sm, smooth_mode=L.SMOOTH_MULTIPLY, bits=bits, granularity=PER_OUTPUT_ROW)
        qm = QuantizedMatrix(q["codes"], q["scale"], q["zp"], bits, PER_OUTPUT_ROW)
        return cls(qm, smooth, bias, bits, False, out_dtype)

    def quantize_input(self, x: torch.Tensor) -> dict:
        return ops.act_quant(x, smooth=self.smooth, smooth_recip=self.smooth_recip,
                             smooth_recip_f32=self.smooth_recip_f32, bits=self.act_bits,
                             symmetric=self.act_symmetric, granularity=PER_TOKEN)

    def forward(self, x: torch.Tensor, out_dtype=None) -> torch.Tensor:
        if x.dim() != 2 or x.shape[1] != self.in_features:
            raise ValueError(f"expected input [T, {self.in_features}], got {tuple(x.shape)}")
        xq = self.quantize_input(x)
        return ops.w8a8_gemm(xq, self.w, epilogue=L.EPI_DEQUANT, out_dtype=out_dtype or self.out_dtype,
                             bias=self.bias)

    __call__ = forward
