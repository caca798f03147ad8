"""moekit.quant API (quant.py:37-610) executed on the B200.

Same names, signatures, defaults, dataclasses and exception types as the
reference, so ``from paper_2508_07329_b200 import quant`` is a drop-in for
``from moekit import quant``. Inputs may be host arrays in the reference's
layouts (W [out, in], X [channels, tokens]) or CUDA tensors; host inputs are
validated like numkit.ensure_matrix, uploaded once, and results come back
as host arrays. Every numeric step runs on the GPU:

  rtn_quantize / _quantize_* ........ K1 act_quant (exact float64 semantics)
  quant_loss / search_smoothing ..... K1 + K2 (tcgen05 int8, exact int32
                                      accumulators) + float64 loss reduction
  build_hessian ..................... K7
  hessian_quantize .................. cuSOLVER factor (library) + K8
  quantize_layer .................... the composition above

The smoothing factors stat**e are evaluated with numpy's pow on the n
per-channel statistics (quant.py:306) so they are bit-identical to the
reference's; everything per element happens on the device.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _lib as L
from . import formats, numkit, ops
from .errors import DegenerateHessianError, NotPositiveDefiniteError, QuantizationFailedError

PER_TENSOR = "per_tensor"
PER_TOKEN = "per_token"
PER_OUTPUT_ROW = "per_output_row"
GRANULARITIES = (PER_TENSOR, PER_TOKEN, PER_OUTPUT_ROW)

ORDER_NONE = "none"
ORDER_MAX_ABS = "max_abs"
ORDER_SUM_SQUARES = "sum_squares"
ORDERINGS = (ORDER_NONE, ORDER_MAX_ABS, ORDER_SUM_SQUARES)

TARGET_CPU_FP = "cpu_fp"
TARGET_GPU_INT = "gpu_int"
PACK_TARGETS = (TARGET_CPU_FP, TARGET_GPU_INT)

SCALE_FLOOR = 1e-12
STAT_FLOOR = 1e-8
DEFAULT_GRID_STEPS = 21
DEFAULT_DAMPING = 0.01


def _round_half_away(v):
    """Reference rounding helper (quant.py:64-67), host-side, for callers and
    tests that use it directly; the device kernels implement the same rule."""
    v = np.asarray(v, dtype=np.float64)
    return np.sign(v) * np.floor(np.abs(v) + 0.5)


@dataclass(frozen=True)
class QuantConfig:
    """bits in [2, 8], symmetric or asymmetric, and the parameter-group
    layout (quant.py:70-94)."""

    bits: int = 8
    symmetric: bool = False
    granularity: str = PER_TENSOR

    def __post_init__(self):
        if not 2 <= self.bits <= 8:
            raise ValueError(f"bits must be in [2, 8], got {self.bits}")
        if self.granularity not in GRANULARITIES:
            raise ValueError(f"unknown granularity {self.granularity!r}")

    @property
    def qmax(self) -> int:
        return (1 << self.bits) - 1


@dataclass(frozen=True)
class QuantParams:
    scale: float
    zero_point: int

    def __post_init__(self):
        if not (self.scale > 0.0 and np.isfinite(self.scale)):
            raise ValueError(f"scale must be positive and finite, got {self.scale}")


def _host(a):
    return a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)


@dataclass
class QuantizedMatrix:
    """Codes [rows, cols] plus per-group affine parameters (quant.py:109-156).
    Arrays may be host (numpy) or device (torch) resident; ``device()``
    returns the GEMM-ready device form (u8 codes, f32 scales, row sums)."""

    codes: object
    scales: object
    zero_points: object
    bits: int
    granularity: str

    def __post_init__(self):
        on_dev = isinstance(self.codes, torch.Tensor)
        if not on_dev:
            self.codes = np.asarray(self.codes)
            self.scales = np.asarray(self.scales, dtype=np.float64).ravel()
            self.zero_points = np.asarray(self.zero_points).ravel().astype(np.int32)
            if self.codes.ndim == 2 and self.codes.dtype.kind not in "iu":
                raise ValueError("codes must be integers")
        if self.codes.ndim != 2:
            raise ValueError("codes must be 2-D")
        if not 2 <= self.bits <= 8:
            raise ValueError(f"bits must be in [2, 8], got {self.bits}")
        if self.granularity not in GRANULARITIES:
            raise ValueError(f"unknown granularity {self.granularity!r}")
        expected = 1 if self.granularity == PER_TENSOR else self.codes.shape[0]
        if self.scales.shape[0] != expected or self.zero_points.shape[0] != expected:
            raise ValueError(f"expected {expected} parameter groups, got {self.scales.shape[0]}")
        qmax = (1 << self.bits) - 1
        codes, scales, zps = (_host(self.codes), _host(self.scales), _host(self.zero_points)) if on_dev else (
            self.codes, self.scales, self.zero_points)
        if codes.min() < 0 or codes.max() > qmax:
            raise ValueError(f"codes out of range [0, {qmax}]")
        if not (scales > 0.0).all() or not np.isfinite(scales).all():
            raise ValueError("scales must be positive and finite")
        if zps.min() < 0 or zps.max() > qmax:
            raise ValueError(f"zero points out of range [0, {qmax}]")

    @property
    def rows(self) -> int:
        return self.codes.shape[0]

    @property
    def cols(self) -> int:
        return self.codes.shape[1]

    def group_params(self) -> list[QuantParams]:
        return [QuantParams(float(s), int(z)) for s, z in zip(_host(self.scales), _host(self.zero_points))]

    def device(self) -> dict:
        """GEMM operand form: u8 codes, f64/f32 scales, i32 zero points and
        code row sums, expanded to one group per row."""
        codes = self.codes if isinstance(self.codes, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(self.codes, dtype=np.uint8))
        codes = codes.to(device="cuda", dtype=torch.uint8).contiguous()
        sc = torch.as_tensor(_host(self.scales), dtype=torch.float64, device="cuda")
        zp = torch.as_tensor(_host(self.zero_points), dtype=torch.int32, device="cuda")
        if sc.numel() == 1 and codes.shape[0] > 1:
            sc, zp = sc.expand(codes.shape[0]).contiguous(), zp.expand(codes.shape[0]).contiguous()
        return {"codes": codes, "scale": sc, "scale_f32": sc.float(), "zp": zp,
                "rowsum": codes.sum(dim=1, dtype=torch.int32)}


@dataclass
class SmoothingResult:
    exponent: float
    factors: np.ndarray
    loss: float


@dataclass
class LayerQuantResult:
    quantized: QuantizedMatrix
    smoothing: SmoothingResult
    ordering: np.ndarray | None
    output_mse: float
    rtn_baseline_mse: float


@dataclass
class PackedExpert:
    target: str
    rows: int
    cols: int
    bits: int
    byte_size: int
    blob: bytes


# ── K1 on reference layouts ───────────────────────────────────────────────
def _k1(xd: torch.Tensor, cfg: QuantConfig, granularity: str, smooth=None, mode=L.SMOOTH_DIVIDE) -> dict:
    sm = None if smooth is None else smooth.reshape(1, -1)
    return ops.act_quant(xd, smooth=sm, smooth_mode=mode, bits=cfg.bits, symmetric=cfg.symmetric,
                         granularity=granularity)


def _qm_from(res: dict, cfg: QuantConfig, granularity: str, host: bool) -> QuantizedMatrix:
    if host:
        return QuantizedMatrix(res["codes"].cpu().numpy().astype(np.int32), res["scale"].cpu().numpy(),
                               res["zp"].cpu().numpy(), cfg.bits, granularity)
    return QuantizedMatrix(res["codes"], res["scale"], res["zp"], cfg.bits, granularity)


def rtn_quantize(x, cfg: QuantConfig) -> QuantizedMatrix:
    """Round-to-nearest at the configured granularity (quant.py:214-231):
    one group (per_tensor) or one group per row (per_token, per_output_row)."""
    host = not isinstance(x, torch.Tensor)
    xd = numkit.to_device(x, "x", dtype=torch.float64 if host else x.dtype)
    return _qm_from(_k1(xd, cfg, cfg.granularity), cfg, cfg.granularity, host)


def dequantize(q: QuantizedMatrix):
    """(code - zero_point) * scale in float64 (quant.py:234-240), on device."""
    host = not isinstance(q.codes, torch.Tensor)
    codes = torch.as_tensor(np.ascontiguousarray(q.codes, dtype=np.uint8)).cuda() if host else q.codes.to(torch.uint8)
    sc = torch.as_tensor(_host(q.scales), dtype=torch.float64, device="cuda")
    zp = torch.as_tensor(_host(q.zero_points), dtype=torch.int32, device="cuda")
    out = ops.dequantize(codes, sc, zp, q.granularity)
    return out.cpu().numpy() if host else out


def _check_factors(factors, n: int) -> np.ndarray:
    f = np.asarray(_host(factors), dtype=np.float64).ravel()
    if f.shape[0] != n:
        raise ValueError(f"expected {n} factors, got {f.shape[0]}")
    if not np.isfinite(f).all() or (f <= 0.0).any():
        raise ValueError("smoothing factors must be positive and finite")
    return f


class _LossContext:
    """Device state shared by the grid points of one smoothing search: W
    [R, n], X^T [T, n] and the float64 reference product (X^T W^T, computed
    once where the reference recomputes it per grid point)."""

    def __init__(self, w, x, cfg: QuantConfig):
        self.cfg = cfg
        if cfg.granularity == PER_OUTPUT_ROW:
            raise ValueError("per_output_row granularity applies to weights only")
        self.wd = numkit.to_device(w, "w")
        xd = numkit.to_device(x, "x")
        if self.wd.shape[1] != xd.shape[0]:
            raise ValueError(f"w has {self.wd.shape[1]} input channels but x has {xd.shape[0]} rows")
        self.xt = xd.T.contiguous()                       # tokens-major
        self.ref = self.xt @ self.wd.T                    # [T, R] float64 (cuBLAS DGEMM)

    def sq_error_dev(self, f_dev: torch.Tensor | None, w_codes: dict | None = None) -> torch.Tensor:
        """||Q(W f) Q(X / f) - W X||_F^2 as a device scalar (no host sync)."""
        cfg = self.cfg
        wq = w_codes if w_codes is not None else _k1(self.wd, cfg, PER_OUTPUT_ROW, f_dev, L.SMOOTH_MULTIPLY)
        xq = _k1(self.xt, cfg, cfg.granularity, f_dev, L.SMOOTH_DIVIDE)
        acc = ops.w8a8_gemm(xq, wq, epilogue=L.EPI_ACC_I32)
        return ops.quant_sq_error(acc, xq["scale"], wq["scale"], self.ref)

    def sq_error(self, f_dev: torch.Tensor | None, w_codes: dict | None = None) -> float:
        return float(self.sq_error_dev(f_dev, w_codes).item())


def quant_loss(w, x, factors, cfg: QuantConfig) -> float:
    """||Q(W s) Q(s^-1 X) - W X||_F (quant.py:267-283) with the exact
    integer W8A8 product."""
    ctx = _LossContext(w, x, cfg)
    f = _check_factors(factors, ctx.wd.shape[1])
    return float(np.sqrt(ctx.sq_error(torch.from_numpy(f).cuda())))


def search_smoothing(w, x, cfg: QuantConfig, grid_steps: int = DEFAULT_GRID_STEPS) -> SmoothingResult:
    """Grid search of the smoothing exponent over [0, 1] (quant.py:286-311);
    strict improvement keeps the smaller exponent on ties."""
    if grid_steps < 2:
        raise ValueError(f"grid_steps must be at least 2, got {grid_steps}")
    ctx = _LossContext(w, x, cfg)
    stat_dev = ops.channel_stats(ctx.xt.T.contiguous(), L.ORDER_MAX_ABS)
    stat = np.maximum(stat_dev.cpu().numpy(), STAT_FLOOR)
    grid = np.linspace(0.0, 1.0, grid_steps)
    factors = [stat ** e for e in grid]                     # numpy pow: bit-identical to the reference's
    # every grid point's loss stays on the device; one host sync for all of them
    sq = torch.stack([ctx.sq_error_dev(torch.from_numpy(f).cuda()).reshape(()) for f in factors]).cpu().numpy()
    best = None
    for e, f, v in zip(grid, factors, sq):
        loss = float(np.sqrt(float(v)))
        if best is None or loss < best.loss:             # strict: ties keep the smaller exponent
            best = SmoothingResult(float(e), f, loss)
    return best


def apply_smoothing(w, x, factors):
    """(W diag(f), diag(f)^-1 X) on device (quant.py:314-324)."""
    host = not isinstance(w, torch.Tensor)
    wd = numkit.to_device(w, "w")
    xd = numkit.to_device(x, "x")
    if wd.shape[1] != xd.shape[0]:
        raise ValueError(f"w has {wd.shape[1]} input channels but x has {xd.shape[0]} rows")
    f = torch.from_numpy(_check_factors(factors, wd.shape[1])).cuda()
    ws, xs = ops.apply_smoothing(wd, xd, f)
    return (ws.cpu().numpy(), xs.cpu().numpy()) if host else (ws, xs)


def build_hessian(x_calib, damping_fraction: float = DEFAULT_DAMPING):
    """H = 2 X X^T + damping * mean(diag) I (quant.py:327-343), K7 on device."""
    host = not isinstance(x_calib, torch.Tensor)
    xd = numkit.to_device(x_calib, "x_calib")
    if damping_fraction < 0:
        raise ValueError(f"damping_fraction must be >= 0, got {damping_fraction}")
    try:
        h = ops.hessian(xd.T.contiguous(), damping_fraction=damping_fraction)
    except DegenerateHessianError:
        raise DegenerateHessianError("calibration activations are all zero") from None
    return h.cpu().numpy() if host else h


def channel_order(x_calib, strategy: str) -> np.ndarray:
    """Stable descending order of max|x| or sum x^2 per channel
    (quant.py:346-363); statistics and the stable sort run on device."""
    xd = numkit.to_device(x_calib, "x_calib")
    if strategy not in ORDERINGS:
        raise ValueError(f"unknown ordering strategy {strategy!r}")
    if strategy == ORDER_NONE:
        return np.arange(xd.shape[0], dtype=np.int64)
    stat = ops.channel_stats(xd, L.ORDER_MAX_ABS if strategy == ORDER_MAX_ABS else L.ORDER_SUM_SQUARES)
    return torch.argsort(-stat, stable=True).cpu().numpy().astype(np.int64)


def _inverse_upper_factor_device(h: torch.Tensor) -> torch.Tensor:
    """U with H^-1 = U^T U, damping retries 0, b, 10b, 100b (quant.py:366-385)."""
    base = DEFAULT_DAMPING * float(torch.diagonal(h).mean())
    eye = torch.eye(h.shape[0], dtype=h.dtype, device=h.device)
    last = None
    for attempt in range(4):
        damp = 0.0 if attempt == 0 else base * 10.0 ** (attempt - 1)
        try:
            inv = numkit.spd_inverse_device(h + damp * eye)
            return numkit.cholesky_device(inv).T.contiguous()
        except NotPositiveDefiniteError as exc:
            last = exc
    raise QuantizationFailedError(f"Hessian is not positive definite after damping escalation ({last})")


def _inverse_upper_factor(h):
    host = not isinstance(h, torch.Tensor)
    u = _inverse_upper_factor_device(numkit.to_device(h, "h"))
    return u.cpu().numpy() if host else u


def _hessian_quantize_dev(wd: torch.Tensor, hd: torch.Tensor, cfg: QuantConfig, order: np.ndarray):
    params = _k1(wd, cfg, PER_OUTPUT_ROW)                       # per-row params of the unpermuted W
    o = torch.from_numpy(order.astype(np.int64)).cuda()
    hp = hd.index_select(0, o).index_select(1, o).contiguous()
    upper = _inverse_upper_factor_device(hp)
    codes = ops.gptq_columns(wd, upper, params["scale"], params["zp"], cfg.bits,
                             None if np.array_equal(order, np.arange(order.shape[0])) else o)
    return codes, params


def hessian_quantize(w, h, cfg: QuantConfig, order: np.ndarray | None = None) -> QuantizedMatrix:
    """Sequential error-compensated weight quantization (quant.py:388-434):
    K8 reproduces the reference's per-element operation order exactly."""
    host = not isinstance(w, torch.Tensor)
    wd = numkit.to_device(w, "w")
    hd = numkit.to_device(h, "h")
    n = wd.shape[1]
    if tuple(hd.shape) != (n, n):
        raise ValueError(f"h must be {n}x{n}, got {hd.shape[0]}x{hd.shape[1]}")
    if order is None:
        order = np.arange(n, dtype=np.int64)
    else:
        order = np.asarray(_host(order), dtype=np.int64).ravel()
        if order.shape[0] != n or not np.array_equal(np.sort(order), np.arange(n)):
            raise ValueError("order must be a permutation of the column indices")
    codes, params = _hessian_quantize_dev(wd, hd, cfg, order)
    if host:
        return QuantizedMatrix(codes.cpu().numpy().astype(np.int32), params["scale"].cpu().numpy(),
                               params["zp"].cpu().numpy(), cfg.bits, PER_OUTPUT_ROW)
    return QuantizedMatrix(codes, params["scale"], params["zp"], cfg.bits, PER_OUTPUT_ROW)


def quantize_layer(w, x_calib, cfg: QuantConfig | None = None, grid_steps: int = DEFAULT_GRID_STEPS,
                   ordering: str = ORDER_NONE) -> LayerQuantResult:
    """HAQ for one linear layer (quant.py:437-490): smoothing search, Hessian,
    compensated quantization, and the output-MSE report — all on device."""
    cfg = cfg or QuantConfig()
    if cfg.granularity == PER_OUTPUT_ROW:
        raise ValueError("layer config granularity selects the activation side")
    if ordering not in ORDERINGS:
        raise ValueError(f"unknown ordering strategy {ordering!r}")
    ctx = _LossContext(w, x_calib, cfg)
    T = ctx.xt.shape[0]
    if T < 8:
        warnings.warn(f"only {T} calibration tokens; statistics may be unstable", UserWarning, stacklevel=2)
    sm = search_smoothing(ctx.wd, ctx.xt.T, cfg, grid_steps)
    f = torch.from_numpy(sm.factors).cuda()
    ws, xs = ops.apply_smoothing(ctx.wd, ctx.xt.T.contiguous(), f)
    try:
        h = ops.hessian(xs.T.contiguous())
    except DegenerateHessianError:
        raise DegenerateHessianError("calibration activations are all zero") from None
    perm = channel_order(xs, ordering)
    codes, params = _hessian_quantize_dev(ws, h, cfg, perm)
    wq = {"codes": codes, "scale": params["scale"], "scale_f32": params["scale_f32"], "zp": params["zp"],
          "rowsum": codes.sum(dim=1, dtype=torch.int32)}
    numel = float(ctx.wd.shape[0] * T)
    out_mse = ctx.sq_error(f, w_codes=wq) / numel
    rtn_mse = ctx.sq_error(None) / numel
    q = QuantizedMatrix(codes.cpu().numpy().astype(np.int32), params["scale"].cpu().numpy(),
                        params["zp"].cpu().numpy(), cfg.bits, PER_OUTPUT_ROW)
    return LayerQuantResult(q, sm, None if ordering == ORDER_NONE else perm, out_mse, rtn_mse)


# ── packing / persistence (host formats; formats.py) ──────────────────────
def precision_pack(q: QuantizedMatrix, target: str) -> PackedExpert:
    """MOEP serialization (quant.py:506-538)."""
    if target not in PACK_TARGETS:
        raise ValueError(f"unknown pack target {target!r}")
    deq = _host(dequantize(q)).astype(np.float32) if target == TARGET_CPU_FP else None
    blob = formats.moep_encode(_host(q.codes), _host(q.scales), _host(q.zero_points), q.bits, q.granularity,
                               target, deq)
    return PackedExpert(target, q.rows, q.cols, q.bits, len(blob), blob)


def unpack_expert(packed):
    """Inverse of precision_pack (quant.py:541-571)."""
    blob = packed.blob if isinstance(packed, PackedExpert) else packed
    res = formats.moep_decode(blob)
    if isinstance(res, np.ndarray):
        return res
    codes, scales, zps, bits, gran = res
    return QuantizedMatrix(codes, scales, zps, bits, gran)


def save_layer_result(result: LayerQuantResult, out_dir) -> None:
    q = result.quantized
    doc = {
        "exponent": result.smoothing.exponent,
        "factors": np.asarray(result.smoothing.factors).tolist(),
        "bits": q.bits,
        "mse": result.output_mse,
        "rtn_mse": result.rtn_baseline_mse,
        "ordering": None if result.ordering is None else np.asarray(result.ordering).tolist(),
        "scales": _host(q.scales).tolist(),
        "zero_points": _host(q.zero_points).tolist(),
        "granularity": q.granularity,
        "smoothing_loss": result.smoothing.loss,
    }
    formats.write_layer_result(out_dir, doc, _host(q.codes))


def load_layer_result(out_dir):
    codes, doc = formats.read_layer_result(out_dir)
    q = QuantizedMatrix(codes, np.asarray(doc["scales"]), np.asarray(doc["zero_points"]), int(doc["bits"]),
                        doc["granularity"])
    return q, doc


# internal helpers kept for API parity with the reference module
def _quantize_acts(x, cfg: QuantConfig):
    """Quantize-dequantize activations (quant.py:252-259), on device."""
    if cfg.granularity == PER_OUTPUT_ROW:
        raise ValueError("per_output_row granularity applies to weights only")
    host = not isinstance(x, torch.Tensor)
    xd = numkit.to_device(x, "x")
    if cfg.granularity == PER_TOKEN:
        r = _k1(xd.T.contiguous(), cfg, PER_TOKEN)
        out = ops.dequantize(r["codes"], r["scale"], r["zp"], PER_TOKEN).T.contiguous()
    else:
        r = _k1(xd, cfg, PER_TENSOR)
        out = ops.dequantize(r["codes"], r["scale"], r["zp"], PER_TENSOR)
    return out.cpu().numpy() if host else out


def _quantize_weights(w, cfg: QuantConfig):
    host = not isinstance(w, torch.Tensor)
    wd = numkit.to_device(w, "w")
    r = _k1(wd, replace(cfg, granularity=PER_OUTPUT_ROW), PER_OUTPUT_ROW)
    out = ops.dequantize(r["codes"], r["scale"], r["zp"], PER_OUTPUT_ROW)
    return out.cpu().numpy() if host else out
