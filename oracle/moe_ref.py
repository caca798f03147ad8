"""Oracle for the MoE forward pieces that the reference does NOT contain
(TEST INFRASTRUCTURE ONLY; parity UNPINNED at the reference level).

Router gating, token permutation, grouped expert FFN and combine are new in
this build. They are restated here from the reference's own primitives:
quantizer semantics from quant_ref (quant.py:191-264), smoothing as an
exact float64 division (quant.py:324), and the routing-event convention
that an event names top_k distinct experts per layer (trace.py:40-44).

Layouts here are tokens-major (x is [T, d]); "per token" therefore means
"per row", the same grouping rtn_quantize applies to per_token inputs
(quant.py:256-258).
"""

from __future__ import annotations

import numpy as np

from . import quant_ref as Q

QMAX8 = 255


# ── router (a'1) ─────────────────────────────────────────────────────────


def router_topk(logits: np.ndarray, k: int):
    """Top-k on the float32 logits with ties to the lower expert id; weights
    are the softmax restricted to the selected experts (float64).

    Returns idx [T, k] (descending logit order), w [T, k], counts [E]."""
    logits = np.asarray(logits, dtype=np.float32)
    t, e = logits.shape
    # lexsort: last key is primary -> sort by -logit, then by id
    ids = np.broadcast_to(np.arange(e), (t, e))
    order = np.lexsort((ids, -logits.astype(np.float64)), axis=1)[:, :k]
    sel = np.take_along_axis(logits, order, axis=1).astype(np.float64)
    ex = np.exp(sel - sel[:, :1])
    w = ex / ex.sum(axis=1, keepdims=True)
    counts = np.bincount(order.ravel(), minlength=e).astype(np.int64)
    return order.astype(np.int32), w, counts


def gate_logits(x: np.ndarray, wg: np.ndarray) -> np.ndarray:
    """Router logits x @ Wg^T in float64 (the GPU computes float32)."""
    return np.asarray(x, dtype=np.float64) @ np.asarray(wg, dtype=np.float64).T


# ── permutation (a'2) ────────────────────────────────────────────────────


def permute(idx: np.ndarray, experts: int):
    """Stable counting sort of the T*k (token, slot) pairs by expert; within
    an expert, pairs keep (token, slot) order.

    Returns offsets [E+1], src_token [T*k], src_slot [T*k], token_pos [T, k]
    (token_pos[t, j] = permuted row of pair (t, j))."""
    idx = np.asarray(idx)
    t, k = idx.shape
    flat = idx.ravel()
    order = np.argsort(flat, kind="stable")
    counts = np.bincount(flat, minlength=experts)
    offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    token_pos = np.empty(t * k, dtype=np.int32)
    token_pos[order] = np.arange(t * k, dtype=np.int32)
    return offsets, (order // k).astype(np.int32), (order % k).astype(np.int32), token_pos.reshape(t, k)


# ── per-token smoothed activation quantization (K1 semantics) ────────────


def quantize_rows(x: np.ndarray, smooth=None, bits: int = 8, symmetric: bool = False):
    """rtn_quantize(x / s, per_token) on tokens-in-rows x (quant.py:214-231
    with the smoothing division of quant.py:324). Returns codes u8-range
    int32, scale f64, zp i32 and the code row sums (int64)."""
    xs = np.asarray(x, dtype=np.float64)
    if smooth is not None:
        xs = xs / np.asarray(smooth, dtype=np.float64)
    codes, scale, zp = Q.rtn(xs, Q.cfg(bits, symmetric, Q.PER_TOKEN))
    return codes, scale, zp, codes.astype(np.int64).sum(axis=1)


def quantize_rows_grouped(x, row_group, smooth_table, bits=8, symmetric=False):
    """Per-row smoothing table lookup (row r uses smooth_table[row_group[r]])."""
    xs = np.asarray(x, dtype=np.float64) / np.asarray(smooth_table, np.float64)[np.asarray(row_group)]
    codes, scale, zp = Q.rtn(xs, Q.cfg(bits, symmetric, Q.PER_TOKEN))
    return codes, scale, zp, codes.astype(np.int64).sum(axis=1)


# ── W8A8 product with exact integer accumulators (a11 / K2) ──────────────


def int_acc(codes_a, za, codes_w, zw) -> np.ndarray:
    """sum_k (ca - za)(cw - zw) in int64: the exact value of the reference's
    fake-quant product before scaling (quant.py:281-283 with dequantize
    folded out)."""
    a = np.asarray(codes_a, dtype=np.int64) - np.asarray(za, dtype=np.int64).reshape(-1, 1)
    w = np.asarray(codes_w, dtype=np.int64) - np.asarray(zw, dtype=np.int64).reshape(-1, 1)
    # float64 BLAS is exact here: |terms| <= 255^2 and every partial sum is an
    # integer below K*255^2 < 2^53, so no rounding can occur.
    assert a.shape[1] * 255 * 255 < 2 ** 53
    return (a.astype(np.float64) @ w.T.astype(np.float64)).astype(np.int64)


def w8a8_linear(codes_a, sa, za, codes_w, sw, zw, bias=None):
    """Y[M, N] = sa_m * sw_n * acc_mn (+ bias_n), float64, plus acc."""
    acc = int_acc(codes_a, za, codes_w, zw)
    y = (np.asarray(sa, np.float64)[:, None] * np.asarray(sw, np.float64)[None, :]) * acc
    if bias is not None:
        y = y + np.asarray(bias, dtype=np.float64)[None, :]
    return y, acc


def silu(g):
    return g / (1.0 + np.exp(-g))


# ── quantized experts ────────────────────────────────────────────────────


def quantize_weight_rows(w, bits=8, symmetric=False):
    """Per-output-row RTN of a weight matrix (quant.py:262-264)."""
    codes, s, z = Q.rtn(w, Q.cfg(bits, symmetric, Q.PER_OUTPUT_ROW))
    return codes, s, z


def expert_forward_exact(x_rows, e: dict, bits=8):
    """One expert on its routed rows: K1(x / s13) -> W13 -> SwiGLU ->
    K1(h / s2) -> W2. ``e`` holds w1/w3/w2 codes/scales/zps and s13/s2.
    Returns the float64 output and the intermediates."""
    cx, sx, zx, _ = quantize_rows(x_rows, e["s13"], bits)
    g, acc1 = w8a8_linear(cx, sx, zx, e["w1_codes"], e["w1_scale"], e["w1_zp"])
    u, acc3 = w8a8_linear(cx, sx, zx, e["w3_codes"], e["w3_scale"], e["w3_zp"])
    h = silu(g) * u
    ch, sh, zh, _ = quantize_rows(h, e["s2"], bits)
    y, acc2 = w8a8_linear(ch, sh, zh, e["w2_codes"], e["w2_scale"], e["w2_zp"])
    return y, {"x_codes": cx, "acc1": acc1, "acc3": acc3, "h": h, "h_codes": ch, "acc2": acc2}


def moe_forward(x, wg, experts: list, k: int = 2, logits=None):
    """Full MoE layer in float64: gate -> top-k -> per-expert FFN -> weighted
    combine. ``logits`` may be supplied (e.g. the GPU's own float32 logits)
    so the routing is evaluated on identical inputs."""
    x = np.asarray(x, dtype=np.float64)
    if logits is None:
        logits = gate_logits(x, wg).astype(np.float32)
    idx, w, _ = router_topk(logits, k)
    out = np.zeros_like(x)
    for ei, ex in enumerate(experts):
        tok, slot = np.nonzero(idx == ei)
        if tok.size == 0:
            continue
        y, _ = expert_forward_exact(x[tok], ex)
        np.add.at(out, tok, w[tok, slot][:, None] * y)
    return out, idx, w


def moe_forward_fakequant(x, wg, experts_deq: list, k: int = 2, logits=None):
    """The reference-style CPU path used as the timed CPU baseline: float64
    fake quantization exactly as quant_loss forms the W8A8 product
    (quant.py:281-283) - per-token RTN then dequantize of the activations,
    pre-dequantized float64 weights, float64 BLAS products."""
    x = np.asarray(x, dtype=np.float64)
    if logits is None:
        logits = gate_logits(x, wg).astype(np.float32)
    idx, w, _ = router_topk(logits, k)
    out = np.zeros_like(x)
    for ei, ex in enumerate(experts_deq):
        tok, slot = np.nonzero(idx == ei)
        if tok.size == 0:
            continue
        c = Q.cfg(8, False, Q.PER_TOKEN)
        xq = Q.fake_quant_acts((x[tok] / ex["s13"]).T, c).T
        h = silu(xq @ ex["w1"].T) * (xq @ ex["w3"].T)
        hq = Q.fake_quant_acts((h / ex["s2"]).T, c).T
        np.add.at(out, tok, w[tok, slot][:, None] * (hq @ ex["w2"].T))
    return out
