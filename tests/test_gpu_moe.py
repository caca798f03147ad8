"""GPU: the full MoE layer forward, checked stage by stage against the oracle
on the GPU's own inputs (identical bytes), at the C2 toy-MoE configuration
(d=1024, 8 experts, top-2, 4096 tokens, ffn=3584) and a small C4-shape
slice; plus W8A8Linear (C1 / C3 shapes)."""

import numpy as np
import pytest
import torch

from oracle import moe_ref as M
from paper_2508_07329_b200 import _lib as L
from paper_2508_07329_b200.linear import W8A8Linear
from paper_2508_07329_b200.moe import MoELayer

from .conftest import bf16_round

pytestmark = pytest.mark.gpu


def _x(rng, T, d):
    x = rng.normal(size=(T, d)).astype(np.float32)
    x[:, rng.choice(d, max(1, d // 100), replace=False)] *= 100.0
    return bf16_round(x)


def _stagewise(cuda, T, d, F, E=8, k=2, seed=0):
    layer = MoELayer.random(E, d, F, top_k=k, seed=seed + 1, out_dtype=torch.float32)
    rng = np.random.default_rng(seed)
    x = _x(rng, T, d)
    xd = torch.from_numpy(x).to(cuda).bfloat16()
    out, aux = layer.forward(xd, out_dtype=torch.float32, return_aux=True)
    lg = aux["logits"].cpu().numpy()
    # router on identical logits
    oidx, ow, _ = M.router_topk(lg, k)
    np.testing.assert_array_equal(aux["idx"].cpu().numpy(), oidx)
    np.testing.assert_allclose(aux["w"].cpu().numpy(), ow, rtol=1e-5, atol=1e-9)  # float32 expf
    # permutation
    offs, tok, slot, pos = M.permute(oidx, E)
    p = aux["perm"]
    np.testing.assert_array_equal(p["offsets"].cpu().numpy(), offs)
    np.testing.assert_array_equal(p["src_token"].cpu().numpy(), tok)
    rexp = oidx[tok, slot]
    experts = [layer.expert_host(e) for e in range(E)]
    s13 = np.stack([e["s13"] for e in experts])
    s2 = np.stack([e["s2"] for e in experts])
    # K1 on x (gather + per-expert smoothing): bit-exact
    c1, sc1, z1, rs1 = M.quantize_rows_grouped(x.astype(np.float64)[tok], rexp, s13)
    np.testing.assert_array_equal(aux["a1"]["codes"].cpu().numpy(), c1)
    np.testing.assert_array_equal(aux["a1"]["scale"].cpu().numpy(), sc1)
    np.testing.assert_array_equal(aux["a1"]["zp"].cpu().numpy(), z1)
    # GEMM1 + SwiGLU vs exact accumulators (h stored bf16: 1 bf16 ulp)
    h = aux["h"].float().cpu().numpy()
    h_codes = aux["a2"]["codes"].cpu().numpy()
    y = aux["y"].cpu().numpy()
    for e in range(E):
        lo, hi = offs[e], offs[e + 1]
        if hi == lo:
            continue
        ex = experts[e]
        g, _ = M.w8a8_linear(c1[lo:hi], sc1[lo:hi], z1[lo:hi], ex["w1_codes"], ex["w1_scale"], ex["w1_zp"])
        u, _ = M.w8a8_linear(c1[lo:hi], sc1[lo:hi], z1[lo:hi], ex["w3_codes"], ex["w3_scale"], ex["w3_zp"])
        hw = M.silu(g) * u
        np.testing.assert_allclose(h[lo:hi], hw, rtol=2.0 ** -7, atol=1e-3 * np.abs(hw).max())
    # K1 on the GPU's own h: bit-exact
    c2, sc2, z2, _ = M.quantize_rows_grouped(h.astype(np.float64), rexp, s2)
    np.testing.assert_array_equal(h_codes, c2)
    np.testing.assert_array_equal(aux["a2"]["scale"].cpu().numpy(), sc2)
    # GEMM2 (dequant * routing weight) vs exact accumulators
    rw = ow[tok, slot]
    for e in range(E):
        lo, hi = offs[e], offs[e + 1]
        if hi == lo:
            continue
        ex = experts[e]
        yw, _ = M.w8a8_linear(c2[lo:hi], sc2[lo:hi], z2[lo:hi], ex["w2_codes"], ex["w2_scale"], ex["w2_zp"])
        yw = yw * rw[lo:hi, None]
        np.testing.assert_allclose(y[lo:hi], yw, rtol=1e-5, atol=1e-6 * np.abs(yw).max())
    # combine
    np.testing.assert_allclose(out.cpu().numpy(), y[pos].sum(axis=1), rtol=1e-6, atol=1e-7)
    return layer, x, out


def test_moe_c2_stagewise(cuda):
    _stagewise(cuda, T=4096, d=1024, F=3584)


@pytest.mark.parametrize("E,k", [(16, 4), (4, 1), (32, 2)])
def test_moe_expert_counts_stagewise(cuda, E, k):
    """Other expert counts / top-k: every stage bit-exact / within tolerance."""
    _stagewise(cuda, T=1024, d=512, F=1024, E=E, k=k, seed=E + k)


def test_moe_mixtral_shape_slice_stagewise(cuda):
    _stagewise(cuda, T=512, d=4096, F=14336, seed=3)


def test_moe_end_to_end_vs_oracle(cuda):
    """Whole-layer output vs the float64 oracle run from x alone (routing on
    the GPU's logits); differences come only from bf16 storage of h
    flipping rare codes, so the check is normwise."""
    layer = MoELayer.random(8, 1024, 1024, seed=5, out_dtype=torch.float32)
    rng = np.random.default_rng(9)
    x = _x(rng, 1024, 1024)
    out, aux = layer.forward(torch.from_numpy(x).to(cuda).bfloat16(), out_dtype=torch.float32, return_aux=True)
    ref, _, _ = M.moe_forward(x.astype(np.float64), None, [layer.expert_host(e) for e in range(8)],
                              logits=aux["logits"].cpu().numpy())
    o = out.cpu().numpy()
    assert np.linalg.norm(o - ref) / np.linalg.norm(ref) < 1e-2


def test_moe_bf16_output_matches_f32(cuda):
    layer = MoELayer.random(8, 512, 1024, seed=2)
    x = torch.from_numpy(_x(np.random.default_rng(1), 700, 512)).to(cuda).bfloat16()
    a = layer.forward(x, out_dtype=torch.float32)
    b = layer.forward(x)
    assert b.dtype == torch.bfloat16
    torch.testing.assert_close(b.float(), a, rtol=2e-2, atol=2e-2 * a.abs().max().item())


@pytest.mark.parametrize("T,din,dout", [(512, 256, 1024), (8192, 4096, 16384)])
def test_w8a8_linear(cuda, T, din, dout):
    rng = np.random.default_rng(din)
    w = torch.randn(dout, din, device=cuda) * 0.02
    s = np.exp(rng.normal(size=din) * 0.5)
    bias = rng.normal(size=dout).astype(np.float32)
    lin = W8A8Linear.from_rtn(w, smooth=s, bias=bias, out_dtype=torch.float32)
    x = _x(rng, T, din)
    y = lin(torch.from_numpy(x).to(cuda).bfloat16()).cpu().numpy()
    xq = lin.quantize_input(torch.from_numpy(x).to(cuda).bfloat16())
    cx, sx, zx, _ = M.quantize_rows(x.astype(np.float64), s)
    np.testing.assert_array_equal(xq["codes"].cpu().numpy(), cx)
    want, _ = M.w8a8_linear(cx, sx, zx, lin.w["codes"].cpu().numpy(), lin.w["scale"].cpu().numpy(),
                            lin.w["zp"].cpu().numpy(), bias)
    np.testing.assert_allclose(y, want, rtol=1e-5, atol=1e-5 * np.abs(want).max())
    assert L.EPI_DEQUANT == 0


@pytest.fixture(scope="module")
def small_layer(cuda):
    return MoELayer.random(8, 512, 1024, seed=11)


def test_moe_token_independence(cuda, small_layer):
    """Each token's output depends on that token alone, bit for bit — across
    batch sizes that take the single-CTA (M < 2048 rows) and the CTA-pair
    GEMM paths, the CTA-per-row (<= 256 rows) and per-warp K1 kernels,
    ragged expert groups and the host pipeline's chunking."""
    x = torch.from_numpy(_x(np.random.default_rng(4), 2500, 512)).to(cuda).bfloat16()
    full = small_layer.forward(x)
    for n in (1, 7, 128, 129, 300, 1024):
        assert torch.equal(small_layer.forward(x[:n].contiguous()), full[:n]), n
    part = small_layer.forward(x[1000:2100].contiguous())
    assert torch.equal(part, full[1000:2100])


@pytest.mark.parametrize("T", [300, 1500, 2500])
def test_moe_fused_quant_gemm2_matches(cuda, small_layer, T):
    """K1 of h fused into the second grouped GEMM (its epilogue warps
    quantize rows while the tensor cores run; single-CTA and CTA-pair tiles)
    gives the same codes, row parameters and layer output as K1 + GEMM."""
    from paper_2508_07329_b200 import _lib as L
    x = torch.from_numpy(_x(np.random.default_rng(T), T, 512)).to(cuda).bfloat16()
    outs = []
    for fused in (0, 1):
        with L.tuned(L.TUNE_FUSED_QUANT, fused):
            outs.append(small_layer.forward(x, return_aux=True))
    (ref, a0), (got, a1) = outs
    for k in ("codes", "scale", "scale_f32", "zp", "rowsum"):
        assert torch.equal(a1["a2"][k], a0["a2"][k]), k
    assert torch.equal(got, ref)


@pytest.mark.parametrize("T", [1, 100, 300, 1500, 2500])
def test_moe_fused_combine_matches(cuda, small_layer, T):
    """The top-2 combine fused into GEMM2's epilogue (first row of a token
    parks its chunk, the second adds it) equals GEMM2 + combine bit for bit
    (compared as raw bf16 bits, signed zeros included)."""
    from paper_2508_07329_b200 import _lib as L
    x = torch.from_numpy(_x(np.random.default_rng(T + 7), T, 512)).to(cuda).bfloat16()
    outs = []
    for fused in (0, 1):
        # (small-row threshold 0: the fused path also runs at decode sizes)
        with L.tuned(L.TUNE_FUSED_COMBINE, fused), L.tuned(L.TUNE_K1_SMALL_ROWS, 0):
            outs.append(small_layer.forward(x))
    outs.append(small_layer.forward(x))            # default knobs
    assert torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16))
    assert torch.equal(outs[0].view(torch.int16), outs[2].view(torch.int16))


def test_moe_edge_batches(cuda, small_layer):
    """Empty batch, one token, a batch whose tokens all pick the same two
    experts (six experts idle), and k = 1 / E = 1 layers."""
    x0 = torch.empty((0, 512), dtype=torch.bfloat16, device=cuda)
    assert small_layer.forward(x0).shape == (0, 512)
    x = torch.from_numpy(_x(np.random.default_rng(31), 64, 512)).to(cuda).bfloat16()
    one = small_layer.forward(x[:1].contiguous())
    assert torch.equal(one, small_layer.forward(x)[:1])
    same = x[:1].repeat(300, 1).contiguous()          # identical tokens -> identical routing
    ys = small_layer.forward(same)
    assert torch.equal(ys, one.repeat(300, 1))
    for E, k in ((4, 1), (1, 1)):
        lay = MoELayer.random(E, 256, 512, top_k=k, seed=E)
        xx = x[:, :256].contiguous()
        full = lay.forward(xx)
        assert torch.equal(lay.forward(xx[:10].contiguous()), full[:10])


def test_moe_permutation_equivariance(cuda, small_layer):
    x = torch.from_numpy(_x(np.random.default_rng(5), 1500, 512)).to(cuda).bfloat16()
    perm = torch.from_numpy(np.random.default_rng(6).permutation(1500)).to(cuda)
    assert torch.equal(small_layer.forward(x[perm].contiguous()), small_layer.forward(x)[perm])


def test_forward_host_matches_device(cuda, small_layer):
    x = torch.from_numpy(_x(np.random.default_rng(7), 5000, 512)).bfloat16()
    dev = small_layer.forward(x.to(cuda))
    host = small_layer.forward_host(x.pin_memory(), chunk_tokens=4096)      # chunks 4096 + 904
    assert torch.equal(host, dev.cpu())
    host2 = small_layer.forward_host(x.pin_memory(), chunks=[1000, 3000, 1000])
    assert torch.equal(host2, dev.cpu())


def test_forward_host_stream_matches_device(cuda, small_layer):
    rng = np.random.default_rng(8)
    xs = [torch.from_numpy(_x(rng, t, 512)).bfloat16().pin_memory() for t in (700, 1500, 3, 900, 1500)]
    outs = small_layer.forward_host_stream([(x, None) for x in xs], depth=2)
    for x, o in zip(xs, outs):
        assert torch.equal(o, small_layer.forward(x.to(cuda)).cpu())


def test_graphed_forward_matches_eager(cuda, small_layer):
    rng = np.random.default_rng(21)
    g = small_layer.graphed(700)
    for _ in range(2):
        x = torch.from_numpy(_x(rng, 700, 512)).to(cuda).bfloat16()
        assert torch.equal(g(x), small_layer.forward(x))


def test_layer_save_load_reference_formats(cuda, small_layer, tmp_path):
    """save -> MOEP gpu_int blobs (byte-identical to the oracle's packing of
    the same codes) + MOEK vectors; load uploads the 8-bit payloads as the
    GEMM operand; the reloaded layer's forward is bit-identical."""
    from oracle import quant_ref as Q
    small_layer.save(tmp_path)
    ex0 = small_layer.expert_host(0)
    blob = (tmp_path / "expert0_w2.moep").read_bytes()
    assert blob == Q.pack_gpu_int(ex0["w2_codes"], ex0["w2_scale"], ex0["w2_zp"], 8, "per_output_row")
    back = MoELayer.load(tmp_path)
    x = torch.from_numpy(_x(np.random.default_rng(31), 600, 512)).to(cuda).bfloat16()
    assert torch.equal(back.forward(x), small_layer.forward(x))


def test_attention_block_stagewise(cuda):
    """The C5 attention half (attention.W8A8Attention) against the float64
    oracle (oracle/attn_ref.py), stage by stage on the GPU's own inputs:
    fused W8A8 QKV projection, RoPE on q and k, causal grouped-query
    attention of packed sequences, W8A8 output projection."""
    _attention_stagewise(256, 4, 2, 32, 64, 3, seed=21)


def _attention_stagewise(d, H, Hk, hd, S, B, seed=21):
    from oracle import attn_ref as A
    from paper_2508_07329_b200.attention import W8A8Attention

    rng = np.random.default_rng(seed)
    att = W8A8Attention.random(d, H, Hk, hd, seed=seed + 5, max_pos=max(128, S))
    x = torch.from_numpy((rng.normal(size=(B * S, d)) * 2).astype(np.float32)).cuda().bfloat16()
    xf = x.double().cpu().numpy()
    wq = att.qkv.w
    sm = att.qkv.smooth.cpu().numpy().ravel()
    qkv_raw = att.qkv(x, out_dtype=torch.float32).double().cpu().numpy()
    want = A.w8a8_linear(xf, wq["codes"].cpu().numpy().astype(np.int32), wq["scale"].cpu().numpy(),
                         wq["zp"].cpu().numpy(), sm)
    np.testing.assert_allclose(qkv_raw, want, rtol=1e-5, atol=1e-5 * np.abs(want).max())
    qkv = att.project_qkv(x, S)
    pos = np.arange(B * S) % S
    base = att.qkv(x, out_dtype=torch.bfloat16).double().cpu().numpy()
    rq = A.rope(base, H, hd, pos)
    rk = A.rope(base[:, H * hd:], Hk, hd, pos)
    got = qkv.double().cpu().numpy()
    ulp = 2.0 ** -7
    np.testing.assert_allclose(got[:, :H * hd], rq[:, :H * hd], rtol=ulp, atol=1e-3)
    np.testing.assert_allclose(got[:, H * hd:(H + Hk) * hd], rk[:, :Hk * hd], rtol=ulp, atol=1e-3)
    np.testing.assert_array_equal(got[:, (H + Hk) * hd:], base[:, (H + Hk) * hd:])     # v untouched
    a = att.attend(qkv, S).double().cpu().numpy()
    wa = A.causal_gqa(got[:, :H * hd], got[:, H * hd:(H + Hk) * hd], got[:, (H + Hk) * hd:], H, Hk, hd, S)
    np.testing.assert_allclose(a, wa, rtol=2e-2, atol=2e-2 * np.abs(wa).max())
    y = att(x, S).double().cpu().numpy()
    wo = att.o.w
    wy = A.w8a8_linear(att.attend(qkv, S).double().cpu().numpy(), wo["codes"].cpu().numpy().astype(np.int32),
                       wo["scale"].cpu().numpy(), wo["zp"].cpu().numpy(), att.o.smooth.cpu().numpy().ravel())
    np.testing.assert_allclose(y, wy, rtol=1e-2, atol=1e-2 * np.abs(wy).max())
