"""Oracle for the attention half of the C5 token path —
TEST INFRASTRUCTURE ONLY; parity UNPINNED at the reference level (the
reference has no forward pass). Restated from the reference's quantizer
semantics (W8A8 linear = quant_ref per-token RTN of x / s times the
per-row weight codes, exact integer accumulators) plus textbook rotary
embedding (rotate-half pairs) and causal grouped-query softmax attention,
all in float64."""

from __future__ import annotations

import numpy as np

from . import moe_ref as M


def w8a8_linear(x, w_codes, w_scale, w_zp, smooth):
    """Y = sa * sw * sum (ca - za)(cw - zw) for per-token codes of x / s."""
    c, sa, za, _ = M.quantize_rows(x, smooth)
    y, _ = M.w8a8_linear(c, sa, za, w_codes, w_scale, w_zp)
    return y


def rope(x, heads: int, head_dim: int, positions, theta: float = 1e6):
    """Rotate-half rotary embedding of the first heads * head_dim columns."""
    x = np.array(x, dtype=np.float64, copy=True)
    half = head_dim // 2
    inv = theta ** (-2.0 * np.arange(half) / head_dim)
    ang = np.asarray(positions, np.float64)[:, None] * inv[None, :]
    c, s = np.cos(ang), np.sin(ang)
    for h in range(heads):
        a = x[:, h * head_dim: h * head_dim + half].copy()
        b = x[:, h * head_dim + half:(h + 1) * head_dim].copy()
        x[:, h * head_dim: h * head_dim + half] = a * c - b * s
        x[:, h * head_dim + half:(h + 1) * head_dim] = b * c + a * s
    return x


def causal_gqa(q, k, v, heads: int, kv_heads: int, head_dim: int, seq_len: int):
    """softmax(q k^T / sqrt(hd) + causal mask) v per packed sequence; query
    head h uses kv head h // (heads / kv_heads). Rows [T, heads * hd]."""
    T = q.shape[0]
    out = np.zeros((T, heads * head_dim))
    rep = heads // kv_heads
    mask = np.triu(np.full((seq_len, seq_len), -np.inf), 1)
    for b in range(T // seq_len):
        r = slice(b * seq_len, (b + 1) * seq_len)
        for h in range(heads):
            kh = h // rep
            qh = q[r, h * head_dim:(h + 1) * head_dim]
            kk = k[r, kh * head_dim:(kh + 1) * head_dim]
            vv = v[r, kh * head_dim:(kh + 1) * head_dim]
            s = qh @ kk.T / np.sqrt(head_dim) + mask
            p = np.exp(s - s.max(axis=1, keepdims=True))
            out[r, h * head_dim:(h + 1) * head_dim] = (p / p.sum(axis=1, keepdims=True)) @ vv
    return out
