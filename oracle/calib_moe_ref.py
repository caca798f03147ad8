"""Oracle for HAQ calibration of a whole MoE layer —
TEST INFRASTRUCTURE ONLY.

The reference calibrates one linear layer at a time (``quantize_layer``,
quant.py:437-490); the paper's Algorithm 1 applies it to
every layer of an MoE model on "the activations collected for that layer"
(X_layer <- collect_activations(X_calib, layer)). For an expert that is the
set of calibration tokens the router sends to it. This module composes the
pinned ``quant_ref.quantize_layer`` into exactly the calibration
``paper_2508_07329_b200.calib_moe.calibrate_moe_layer`` performs:

  1. routing: top-k of the router logits (``moe_ref.router_topk``; the test
     feeds the GPU router's float32 logits, so both sides see the same ids);
  2. per expert e, the tokens with e among their k experts, in token order
     (all tokens if fewer than ``min_tokens``);
  3. W1 and W3 share their input: one ``quantize_layer`` of the stacked
     ``[W1; W3]`` (one smoothing vector s13);
  4. W2: ``quantize_layer`` on the expert's float SwiGLU activation
     h = silu(x W1^T) * (x W3^T) of the same tokens (float64), or on a given
     ``h`` (stage-wise parity on the GPU's own h).
"""

from __future__ import annotations

import numpy as np

from . import moe_ref as M
from . import quant_ref as Q


def swiglu_acts(xe: np.ndarray, w1: np.ndarray, w3: np.ndarray) -> np.ndarray:
    """Float64 SwiGLU activation [tokens, F] of tokens ``xe`` [tokens, d]."""
    g = xe @ np.asarray(w1, np.float64).T
    return g / (1.0 + np.exp(-g)) * (xe @ np.asarray(w3, np.float64).T)


def expert_tokens(idx: np.ndarray, e: int, min_tokens: int) -> tuple[np.ndarray, bool]:
    """Token ids routed to expert ``e`` (ascending) and whether the expert
    falls back to all tokens (fewer than ``min_tokens`` routed)."""
    tok = np.flatnonzero((np.asarray(idx) == e).any(axis=1))
    if tok.size < min_tokens:
        return np.arange(idx.shape[0]), True
    return tok, False


def calibrate_expert(x: np.ndarray, tok: np.ndarray, ex: dict, c: Q.Cfg, steps: int, ordering: str,
                     h: np.ndarray | None = None) -> dict:
    """Steps 3-4 for one expert. ``x`` [T, d] float64 calibration tokens."""
    xe = x[tok]
    w1, w3, w2 = (np.asarray(ex[k], np.float64) for k in ("w1", "w3", "w2"))
    F = w1.shape[0]
    r13 = Q.quantize_layer(np.concatenate([w1, w3]), xe.T, c, steps, ordering)
    if h is None:
        h = swiglu_acts(xe, w1, w3)
    r2 = Q.quantize_layer(w2, np.asarray(h, np.float64).T, c, steps, ordering)
    return {"w1": (r13["codes"][:F], r13["scales"][:F], r13["zero_points"][:F]),
            "w3": (r13["codes"][F:], r13["scales"][F:], r13["zero_points"][F:]),
            "w2": (r2["codes"], r2["scales"], r2["zero_points"]),
            "s13": r13["factors"], "s2": r2["factors"],
            "exponent13": r13["exponent"], "exponent2": r2["exponent"],
            "mse13": r13["output_mse"], "rtn_mse13": r13["rtn_baseline_mse"],
            "mse2": r2["output_mse"], "rtn_mse2": r2["rtn_baseline_mse"], "h": h}


def calibrate_moe_layer(logits: np.ndarray, x: np.ndarray, experts_fp: list, top_k: int = 2,
                        c: Q.Cfg | None = None, steps: int = 21, ordering: str = "none", min_tokens: int = 16,
                        h_given: list | None = None) -> tuple[np.ndarray, list]:
    """Routing ids [T, k] and one ``calibrate_expert`` dict per expert (plus
    ``tokens`` / ``used_all_tokens``). ``h_given[e]`` replaces expert e's
    float SwiGLU activation (stage-wise parity)."""
    c = c or Q.cfg(8, False, Q.PER_TOKEN)
    idx, _, _ = M.router_topk(logits, top_k)
    x = np.asarray(x, np.float64)
    out = []
    for e, ex in enumerate(experts_fp):
        tok, used_all = expert_tokens(idx, e, min_tokens)
        r = calibrate_expert(x, tok, ex, c, steps, ordering, None if h_given is None else h_given[e])
        r.update(tokens=int((idx == e).any(axis=1).sum()), used_all_tokens=used_all, token_ids=tok)
        out.append(r)
    return idx, out
