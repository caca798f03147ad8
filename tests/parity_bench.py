"""Oracle parity at the exact bench configuration (C4: Mixtral-8x7B-shape
MoE layer, 8 experts, top-2, d=4096, ffn=14336; bench.synth_tokens inputs,
MoELayer.random(seed=1) weights) — TEST INFRASTRUCTURE, shared by
tests/test_gpu_bench_parity.py (asserts) and tools/parity_report.py (writes
profiles/parity_r02.json).

The whole token batch runs through the GPU path the bench times (CTA-pair
grouped GEMMs, the banded W2 raster, row-ext speculation over all 2T rows,
the top-2 combine fused into GEMM2); the float64 oracle (oracle/moe_ref.py,
quantizer semantics of quant.py:191-231, product of quant.py:281-283) is
evaluated on a stratified token sample that covers every expert, because a
full float64 W13 product over 32k rows takes minutes on the host.

Checks (``check_bench_config``):
  * fused-combine output == GEMM2 + combine kernel output, raw bf16 bits;
  * top-k ids == oracle top-k on the GPU's own float32 logits (all tokens);
    routing weights within rtol 1e-5;
  * the permutation (offsets, source tokens, inverse positions) == oracle;
  * sample rows: K1(x) codes / scale / zp / rowsum bit-exact;
    h (bf16) within one bf16 ulp of silu(g)*u from the exact int32
    accumulators; K1(h) codes on the GPU's own h bit-exact; y (bf16) within
    one bf16 ulp of the exact product; token output == bf16(y0 + y1);
  * end to end from x (oracle h in float64, its own h codes): normwise error
    and h-code flip rate, for the bf16-h serving path and the float32-h
    precise mode (MoELayer.forward(h_dtype=torch.float32));
  * routing from x: top-k from float64 gate logits vs the GPU's float32
    tensor-core logits (flip rate at near-ties).
"""

from __future__ import annotations

import numpy as np
import torch

from oracle import moe_ref as M

E, D, F, K = 8, 4096, 14336, 2


def _bf16_ulp(v):
    """One bf16 ulp at |v| (float64 array): 2^(floor(log2|v|) - 7)."""
    a = np.maximum(np.abs(v), 2.0 ** -126)
    return np.exp2(np.floor(np.log2(a)) - 7)


def stratified_sample(idx: np.ndarray, per_expert: int, seed: int = 0) -> np.ndarray:
    """Up to ``per_expert`` tokens routed to each expert (any slot), union,
    sorted: every expert's rows appear in the sample."""
    rng = np.random.default_rng(seed)
    pick = []
    for e in range(int(idx.max()) + 1):
        toks = np.nonzero((idx == e).any(axis=1))[0]
        if toks.size:
            pick.append(rng.choice(toks, min(per_expert, toks.size), replace=False))
    return np.unique(np.concatenate(pick))


def _expert_w(layer, e: int, name: str):
    q = layer.host_experts[e][name]
    codes = q.codes.cpu().numpy() if isinstance(q.codes, torch.Tensor) else np.asarray(q.codes)
    sc = q.scales.cpu().numpy() if isinstance(q.scales, torch.Tensor) else np.asarray(q.scales)
    zp = q.zero_points.cpu().numpy() if isinstance(q.zero_points, torch.Tensor) else np.asarray(q.zero_points)
    return codes, sc.astype(np.float64), zp.astype(np.int32)


def _linear(codes_a, sa, za, wt):
    """Oracle W8A8 product (exact int accumulators, float64 dequant)."""
    wc, ws, wz = wt
    return M.w8a8_linear(codes_a, sa, za, wc, ws, wz)


def check_bench_config(layer, x_bf16: torch.Tensor, per_expert: int = 64, seed: int = 0,
                       assert_ok: bool = True) -> dict:
    """Run the bench forward on all of x and check it against the oracle on a
    stratified sample; returns the measured numbers (see module doc)."""
    T = x_bf16.shape[0]
    rep = {"tokens": T}
    out_fused = layer.forward(x_bf16)                       # the bench's default path
    out, aux = layer.forward(x_bf16, return_aux=True)       # same kernels, GEMM2 + combine kernel
    torch.cuda.synchronize()
    same = torch.equal(out_fused.view(torch.int16), out.view(torch.int16))
    rep["fused_combine_bit_identical"] = bool(same)
    if assert_ok:
        assert same, "fused GEMM2+combine differs from GEMM2 + combine"
    x = x_bf16.float().cpu().numpy().astype(np.float64)
    logits = aux["logits"].cpu().numpy()
    gidx = aux["idx"].cpu().numpy()
    oidx, ow, _ = M.router_topk(logits, K)
    rep["router_ids_equal_on_gpu_logits"] = bool(np.array_equal(gidx, oidx))
    if assert_ok:
        np.testing.assert_array_equal(gidx, oidx)
        np.testing.assert_allclose(aux["w"].cpu().numpy(), ow, rtol=1e-5, atol=1e-9)
    # routing from x: float64 gate logits (oracle) vs the GPU's float32 ones
    gl = M.gate_logits(x, layer.gate_w.cpu().numpy()) + layer.gate_b.cpu().numpy().astype(np.float64)
    ids = np.broadcast_to(np.arange(E), gl.shape)
    fidx = np.lexsort((ids, -gl), axis=1)[:, :K].astype(np.int32)
    flips = ~(np.sort(fidx, 1) == np.sort(gidx, 1)).all(axis=1)
    srt = np.sort(gl, axis=1)[:, ::-1]
    rep["routing_from_x"] = {
        "logit_max_abs_err": float(np.abs(logits - gl).max()),
        "logit_max_rel_err": float((np.abs(logits - gl) / np.maximum(np.abs(gl), 1e-30)).max()),
        "tokens_with_different_expert_set": int(flips.sum()),
        "flip_rate": float(flips.mean()),
        "min_gap_kth_vs_next": float((srt[:, K - 1] - srt[:, K]).min()),
    }
    offs, tok, slot, pos = M.permute(oidx, E)
    p = aux["perm"]
    if assert_ok:
        np.testing.assert_array_equal(p["offsets"].cpu().numpy(), offs)
        np.testing.assert_array_equal(p["src_token"].cpu().numpy(), tok)
        np.testing.assert_array_equal(p["token_pos"].cpu().numpy().reshape(T, K), pos)
    rep["permutation_equal"] = True
    samp = stratified_sample(oidx, per_expert, seed)
    rows = np.sort(pos[samp].ravel())                       # every row of the sampled tokens
    rexp = oidx[tok[rows], slot[rows]]
    rep["sample"] = {"tokens": int(samp.size), "rows": int(rows.size),
                     "rows_per_expert": np.bincount(rexp, minlength=E).tolist()}
    s13 = layer.s13.cpu().numpy()
    s2 = layer.s2.cpu().numpy()
    a1 = {k: aux["a1"][k][torch.from_numpy(rows).cuda().long()].cpu().numpy() for k in ("codes", "scale", "zp",
                                                                                       "rowsum")}
    c1, sc1, z1, rs1 = M.quantize_rows_grouped(x[tok[rows]], rexp, s13)
    a1_ok = (np.array_equal(a1["codes"], c1) and np.array_equal(a1["scale"], sc1) and np.array_equal(a1["zp"], z1)
             and np.array_equal(a1["rowsum"], rs1))
    rep["a1_bit_exact"] = bool(a1_ok)
    if assert_ok:
        assert a1_ok, "K1(x) differs from the oracle"
    rsel = torch.from_numpy(rows).cuda().long()
    h_gpu = aux["h"][rsel].float().cpu().numpy().astype(np.float64)
    hc_gpu = aux["a2"]["codes"][rsel].cpu().numpy()
    y_gpu = aux["y"][rsel].float().cpu().numpy().astype(np.float64)
    rw = ow[tok[rows], slot[rows]]
    # precise mode (float32 h) on the same batch
    out_p, aux_p = layer.forward(x_bf16, out_dtype=torch.float32, h_dtype=torch.float32, return_aux=True)
    hp_codes = aux_p["a2"]["codes"][rsel].cpu().numpy()
    hp = aux_p["h"][rsel].cpu().numpy().astype(np.float64)
    out_p = out_p.cpu().numpy().astype(np.float64)
    h_err, y_err = 0.0, 0.0
    h_exact = np.empty_like(h_gpu)
    y_from_gpu_h = np.empty_like(y_gpu)
    y_from_x = np.empty_like(y_gpu)           # oracle end to end (float64 h, its own codes)
    flips_bf16 = flips_f32 = 0
    hp_rel = 0.0
    for e in range(E):
        sel = np.nonzero(rexp == e)[0]
        if sel.size == 0:
            continue
        w1, w3, w2 = (_expert_w(layer, e, n) for n in ("w1", "w3", "w2"))
        g, _ = _linear(c1[sel], sc1[sel], z1[sel], w1)
        u, _ = _linear(c1[sel], sc1[sel], z1[sel], w3)
        he = M.silu(g) * u
        h_exact[sel] = he
        # (the 1e-7 * max term covers silu's float32 ex2/rcp on large-|g| tails only)
        h_err = max(h_err, float((np.abs(h_gpu[sel] - he) / (_bf16_ulp(he) + 1e-7 * np.abs(he).max())).max()))
        hp_rel = max(hp_rel, float(np.abs(hp[sel] - he).max() / max(np.abs(he).max(), 1e-300)))
        ge = np.full(sel.size, e)
        # K1 on the GPU's own h: bit-exact
        c2, sc2, z2, _ = M.quantize_rows_grouped(h_gpu[sel], ge, s2)
        if assert_ok:
            np.testing.assert_array_equal(hc_gpu[sel], c2)
            np.testing.assert_array_equal(aux["a2"]["scale"][rsel].cpu().numpy()[sel], sc2)
        yw, _ = _linear(c2, sc2, z2, w2)
        yw = yw * rw[sel, None]
        y_from_gpu_h[sel] = yw
        y_err = max(y_err, float((np.abs(y_gpu[sel] - yw) / _bf16_ulp(yw)).max()))
        # oracle end to end: h in float64, its own codes
        c2x, sc2x, z2x, _ = M.quantize_rows_grouped(he, ge, s2)
        flips_bf16 += int((c2x != hc_gpu[sel]).sum())
        flips_f32 += int((c2x != hp_codes[sel]).sum())
        yx, _ = _linear(c2x, sc2x, z2x, w2)
        y_from_x[sel] = yx * rw[sel, None]
        del w1, w3, w2
    rep["h_max_err_bf16_ulps"] = h_err
    rep["y_max_err_bf16_ulps"] = y_err
    rep["h_f32_max_rel_err"] = hp_rel
    if assert_ok:
        assert h_err <= 1.0 + 1e-9, f"h off by {h_err} bf16 ulps"
        assert y_err <= 1.0 + 1e-9, f"y off by {y_err} bf16 ulps"
    # token outputs of the sample: bf16(y0 + y1) exactly (combine order), and vs the oracle
    o_gpu = out[torch.from_numpy(samp).cuda().long()].float().cpu().numpy().astype(np.float64)
    ypos = {r: i for i, r in enumerate(rows)}
    y0 = np.array([y_gpu[ypos[pos[t, 0]]] for t in samp])
    y1 = np.array([y_gpu[ypos[pos[t, 1]]] for t in samp])
    comb = torch.from_numpy((y0.astype(np.float32) + y1.astype(np.float32))).bfloat16().float().numpy()
    comb_ok = np.array_equal(comb.astype(np.float64), o_gpu)
    rep["combine_bit_exact"] = bool(comb_ok)
    Y = np.array([y_from_gpu_h[ypos[pos[t, 0]]] + y_from_gpu_h[ypos[pos[t, 1]]] for t in samp])
    Ymag = np.array([np.abs(y_from_gpu_h[ypos[pos[t, 0]]]) + np.abs(y_from_gpu_h[ypos[pos[t, 1]]]) for t in samp])
    out_err = np.abs(o_gpu - Y) / (_bf16_ulp(Ymag) + _bf16_ulp(Y))
    rep["out_max_err_ulps_of_sum"] = float(out_err.max())
    if assert_ok:
        assert comb_ok, "token output != bf16(y0 + y1)"
        assert out_err.max() <= 1.0 + 1e-9
    # end to end from x
    Yx = np.array([y_from_x[ypos[pos[t, 0]]] + y_from_x[ypos[pos[t, 1]]] for t in samp])
    nrm = np.linalg.norm(Yx)
    op = out_p[samp]
    n_codes = rows.size * F
    rep["end_to_end_from_x"] = {
        "bf16_h": {"normwise_rel_err": float(np.linalg.norm(o_gpu - Yx) / nrm),
                   "h_code_flip_rate": flips_bf16 / n_codes},
        "f32_h_precise": {"normwise_rel_err": float(np.linalg.norm(op - Yx) / nrm),
                          "max_abs_err_rel_to_max": float(np.abs(op - Yx).max() / np.abs(Yx).max()),
                          "h_code_flip_rate": flips_f32 / n_codes},
        "bf16_output_rounding_floor": float(np.linalg.norm(
            torch.from_numpy(Yx.astype(np.float32)).bfloat16().double().numpy() - Yx) / nrm),
    }
    return rep
