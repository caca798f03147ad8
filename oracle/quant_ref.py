"""Oracle restatement of moekit/quant.py (TEST INFRASTRUCTURE ONLY).

Layouts follow the reference: W is [out R x in n], X is [channels n x
tokens T] (quant.py:3-5). Everything is float64 with int32 codes, exactly as
the reference computes it; bit-exactness of the CUDA path is judged against
these functions, which are themselves pinned to the unmodified reference by
tests/golden (see tests/test_oracle_pinned.py).
"""

from __future__ import annotations

import struct
import warnings
from collections import namedtuple

import numpy as np

from .numkit_ref import OracleNotPD, as_f64_matrix, cholesky_lower, spd_inverse

PER_TENSOR, PER_TOKEN, PER_OUTPUT_ROW = "per_tensor", "per_token", "per_output_row"
GRANS = (PER_TENSOR, PER_TOKEN, PER_OUTPUT_ROW)
SCALE_FLOOR = 1e-12   # quant.py:53
STAT_FLOOR = 1e-8     # quant.py:54
DAMPING = 0.01        # quant.py:57

Cfg = namedtuple("Cfg", "bits symmetric granularity")


def cfg(bits: int = 8, symmetric: bool = False, granularity: str = PER_TENSOR) -> Cfg:
    """QuantConfig (quant.py:70-94) as a plain tuple."""
    if not 2 <= bits <= 8 or granularity not in GRANS:
        raise ValueError("bad quantizer config")
    return Cfg(int(bits), bool(symmetric), granularity)


def rha(v):
    """Half-away-from-zero rounding in float64 (quant.py:64-67). Note the
    add of 0.5 is itself rounded: 0.49999999999999994 rounds to 1."""
    v = np.asarray(v, dtype=np.float64)
    return np.sign(v) * np.floor(np.abs(v) + 0.5)


def affine(gmin, gmax, c: Cfg):
    """Scale / zero point per group (quant.py:191-202)."""
    qmax = (1 << c.bits) - 1
    gmin = np.asarray(gmin, dtype=np.float64)
    gmax = np.asarray(gmax, dtype=np.float64)
    if c.symmetric:
        half = (1 << (c.bits - 1))
        amax = np.maximum(np.abs(gmin), np.abs(gmax))
        scale = np.maximum(amax / (half - 1), SCALE_FLOOR)
        zp = np.full(scale.shape, half, dtype=np.int32)
    else:
        scale = np.maximum((gmax - gmin) / qmax, SCALE_FLOOR)
        zp = np.clip(rha(-gmin / scale), 0, qmax).astype(np.int32)
    return scale, zp


def encode(x, scale, zp, qmax: int):
    """quant.py:209-211: clip(rha(x / scale) + zp, 0, qmax)."""
    return np.clip(rha(x / scale) + zp, 0, qmax).astype(np.int32)


def rtn(x, c: Cfg):
    """rtn_quantize (quant.py:214-231) -> (codes int32, scales f64, zps i32).
    per_token and per_output_row both group by row."""
    x = as_f64_matrix(x, "x")
    qmax = (1 << c.bits) - 1
    if c.granularity == PER_TENSOR:
        scale, zp = affine(np.array([x.min()]), np.array([x.max()]), c)
        return encode(x, scale[0], int(zp[0]), qmax), scale, zp
    scale, zp = affine(x.min(axis=1), x.max(axis=1), c)
    return encode(x, scale[:, None], zp[:, None], qmax), scale, zp


def dequant(codes, scale, zp, granularity: str):
    """dequantize (quant.py:234-240)."""
    codes = np.asarray(codes).astype(np.float64)
    scale = np.asarray(scale, dtype=np.float64).ravel()
    zp = np.asarray(zp).ravel()
    if granularity == PER_TENSOR:
        return (codes - float(zp[0])) * float(scale[0])
    return (codes - zp[:, None]) * scale[:, None]


def fake_quant_acts(x, c: Cfg):
    """_quantize_acts (quant.py:252-259): channels x tokens in, same out."""
    if c.granularity == PER_OUTPUT_ROW:
        raise ValueError("per_output_row applies to weights only")
    if c.granularity == PER_TOKEN:
        xt = np.ascontiguousarray(np.asarray(x, dtype=np.float64).T)
        codes, s, z = rtn(xt, c)
        return dequant(codes, s, z, PER_TOKEN).T
    codes, s, z = rtn(x, c)
    return dequant(codes, s, z, c.granularity)


def fake_quant_weights(w, c: Cfg):
    """_quantize_weights (quant.py:262-264): always per output row."""
    rc = Cfg(c.bits, c.symmetric, PER_OUTPUT_ROW)
    codes, s, z = rtn(w, rc)
    return dequant(codes, s, z, PER_OUTPUT_ROW)


def _factors(f, n: int) -> np.ndarray:
    f = np.asarray(f, dtype=np.float64).ravel()
    if f.shape[0] != n or not np.isfinite(f).all() or (f <= 0).any():
        raise ValueError("bad smoothing factors")
    return f


def quant_loss(w, x, f, c: Cfg) -> float:
    """quant.py:267-283: ||Q(W diag f) Q(diag(f)^-1 X) - W X||_F."""
    w = as_f64_matrix(w, "w")
    x = as_f64_matrix(x, "x")
    if w.shape[1] != x.shape[0]:
        raise ValueError("shape mismatch")
    f = _factors(f, w.shape[1])
    wq = fake_quant_weights(w * f[None, :], c)
    xq = fake_quant_acts(x / f[:, None], c)
    return float(np.linalg.norm(wq @ xq - w @ x, "fro"))


def smoothing_grid(x, steps: int):
    """The per-channel statistic and exponent grid of search_smoothing
    (quant.py:303-306)."""
    stat = np.maximum(np.abs(as_f64_matrix(x)).max(axis=1), STAT_FLOOR)
    return stat, np.linspace(0.0, 1.0, steps)


def search_smoothing(w, x, c: Cfg, steps: int = 21):
    """quant.py:286-311 -> (exponent, factors, loss). Strict '<' keeps the
    smallest exponent on ties."""
    if steps < 2:
        raise ValueError("grid_steps must be at least 2")
    stat, grid = smoothing_grid(x, steps)
    best = None
    for e in grid:
        f = stat ** e
        loss = quant_loss(w, x, f, c)
        if best is None or loss < best[2]:
            best = (float(e), f, loss)
    return best


def apply_smoothing(w, x, f):
    """quant.py:314-324."""
    w = as_f64_matrix(w, "w")
    x = as_f64_matrix(x, "x")
    f = _factors(f, w.shape[1])
    return w * f[None, :], x / f[:, None]


class OracleDegenerate(ArithmeticError):
    """Mirror of errors.DegenerateHessianError."""


class OracleQuantFailed(ArithmeticError):
    """Mirror of errors.QuantizationFailedError."""


def build_hessian(x, damping_fraction: float = DAMPING) -> np.ndarray:
    """quant.py:327-343: H = 2 X X^T, symmetrised, + damping * mean(diag)."""
    x = as_f64_matrix(x, "x_calib")
    if damping_fraction < 0:
        raise ValueError("damping_fraction must be >= 0")
    if not x.any():
        raise OracleDegenerate("all-zero calibration")
    h = 2.0 * (x @ x.T)
    h = (h + h.T) / 2.0
    h[np.diag_indices_from(h)] += damping_fraction * float(np.mean(np.diag(h)))
    return h


def channel_order(x, strategy: str) -> np.ndarray:
    """quant.py:346-363: stable descending sort of max|x| or sum x^2."""
    x = as_f64_matrix(x, "x_calib")
    if strategy == "none":
        return np.arange(x.shape[0], dtype=np.int64)
    if strategy == "max_abs":
        stat = np.abs(x).max(axis=1)
    elif strategy == "sum_squares":
        stat = (x ** 2).sum(axis=1)
    else:
        raise ValueError(f"unknown ordering strategy {strategy!r}")
    return np.argsort(-stat, kind="stable").astype(np.int64)


def inverse_upper_factor(h) -> np.ndarray:
    """quant.py:366-385: U with H^-1 = U^T U, damping retries 0, b, 10b, 100b
    where b = 0.01 mean(diag H)."""
    h = np.asarray(h, dtype=np.float64)
    base = DAMPING * float(np.mean(np.diag(h)))
    ident = np.eye(h.shape[0])
    for attempt in range(4):
        damp = 0.0 if attempt == 0 else base * 10.0 ** (attempt - 1)
        try:
            return cholesky_lower(spd_inverse(h + damp * ident)).T
        except OracleNotPD:
            continue
    raise OracleQuantFailed("Hessian not positive definite after damping escalation")


def gptq_columns(wp, upper, scale, zp, qmax: int) -> np.ndarray:
    """The strict-order column loop of hessian_quantize (quant.py:422-430) on
    already-permuted weights ``wp`` and factor ``upper``. Every trailing
    update is a separate multiply then subtract (no fusion), in column
    order; this is the sequence the GPU kernel must reproduce bit-exactly."""
    wp = np.array(wp, dtype=np.float64, copy=True)
    r, n = wp.shape
    sc = np.asarray(scale, dtype=np.float64)
    z = np.asarray(zp, dtype=np.int32)
    codes = np.empty((r, n), dtype=np.int32)
    for i in range(n):
        col = wp[:, i]
        ci = encode(col, sc, z, qmax)
        codes[:, i] = ci
        err = (col - (ci.astype(np.float64) - z) * sc) / upper[i, i]
        if i + 1 < n:
            wp[:, i + 1:] -= np.outer(err, upper[i, i + 1:])
    return codes


def hessian_quantize(w, h, c: Cfg, order=None):
    """quant.py:388-434 -> (codes, scales, zps) per output row."""
    w = as_f64_matrix(w, "w")
    h = as_f64_matrix(h, "h")
    n = w.shape[1]
    if h.shape != (n, n):
        raise ValueError("h shape mismatch")
    order = np.arange(n) if order is None else np.asarray(order, dtype=np.int64).ravel()
    if order.shape[0] != n or not np.array_equal(np.sort(order), np.arange(n)):
        raise ValueError("order must be a permutation")
    scale, zp = affine(w.min(axis=1), w.max(axis=1), c)
    upper = inverse_upper_factor(h[np.ix_(order, order)])
    codes_p = gptq_columns(w[:, order], upper, scale, zp, (1 << c.bits) - 1)
    codes = np.empty_like(codes_p)
    codes[:, order] = codes_p
    return codes, scale, zp


def quantize_layer(w, x, c: Cfg | None = None, steps: int = 21, ordering: str = "none"):
    """quant.py:437-490 -> dict with the LayerQuantResult fields."""
    c = c or cfg()
    w = as_f64_matrix(w, "w")
    x = as_f64_matrix(x, "x_calib")
    if w.shape[1] != x.shape[0] or c.granularity == PER_OUTPUT_ROW:
        raise ValueError("bad layer inputs")
    if x.shape[1] < 8:
        warnings.warn("few calibration tokens", UserWarning, stacklevel=2)
    e, f, loss = search_smoothing(w, x, c, steps)
    ws, xs = apply_smoothing(w, x, f)
    h = build_hessian(xs)
    perm = channel_order(xs, ordering)
    codes, scale, zp = hessian_quantize(ws, h, c, perm)
    ref = w @ x
    out = dequant(codes, scale, zp, PER_OUTPUT_ROW) @ fake_quant_acts(xs, c)
    base = fake_quant_weights(w, c) @ fake_quant_acts(x, c)
    return {
        "codes": codes, "scales": scale, "zero_points": zp,
        "exponent": e, "factors": f, "smoothing_loss": loss,
        "ordering": None if ordering == "none" else perm,
        "output_mse": float(np.mean((out - ref) ** 2)),
        "rtn_baseline_mse": float(np.mean((base - ref) ** 2)),
    }


def pack_gpu_int(codes, scales, zps, bits: int, granularity: str) -> bytes:
    """precision_pack(target=gpu_int) byte layout (quant.py:493-538): header
    '<4sBBBBIII', then (scale, zp) f64 pairs, then little-endian bit-packed
    codes. For 8 bits the code stream is the raw row-major u8 matrix."""
    codes = np.asarray(codes)
    head = struct.pack("<4sBBBBIII", b"MOEP", 1, 1, bits, GRANS.index(granularity),
                       codes.shape[0], codes.shape[1], len(scales))
    params = np.empty(2 * len(scales), dtype="<f8")
    params[0::2] = scales
    params[1::2] = np.asarray(zps, dtype=np.float64)
    flat = codes.astype(np.uint32).ravel()
    bitplanes = ((flat[:, None] >> np.arange(bits, dtype=np.uint32)) & 1).astype(np.uint8)
    return head + params.tobytes() + np.packbits(bitplanes.ravel(), bitorder="little").tobytes()
