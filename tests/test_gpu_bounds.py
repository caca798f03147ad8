"""Write bounds: every kernel writes only inside its output views.

Outputs are carved out of larger buffers pre-filled with a sentinel (extra
columns to the right of every row, extra rows below); after the call the
margins must still hold the sentinel and the carved result must equal an
ordinary call's. Shapes are ragged on purpose (row counts off the 128 / 256
tile grid, columns off the 256-wide tile and the 4 KB K1 chunk, expert
segments with partial tiles). (compute-sanitizer is not available on the
GPU pool, so out-of-bounds writes are caught this way.)
"""

import numpy as np
import pytest
import torch

from paper_2508_07329_b200 import _lib as L
from paper_2508_07329_b200 import ops
from paper_2508_07329_b200.moe import MoELayer

from .conftest import bf16_round
from .test_gpu_kernels import _acts, _dev_operand, _rand_operand, _smooth, _true_records

pytestmark = pytest.mark.gpu

PAD_C, PAD_R = 40, 3          # extra columns (keeps 8-element row alignment) and rows


def _carve(rows, cols, dtype, dev, sentinel):
    buf = torch.empty((rows + PAD_R, cols + PAD_C), dtype=dtype, device=dev)
    buf.view(torch.uint8).fill_(sentinel)
    return buf, buf[:rows, :cols]


def _assert_margins(buf, rows, cols, sentinel):
    b = buf.view(torch.uint8)
    esz = buf.element_size()
    assert bool((b[:rows, cols * esz:] == sentinel).all()), "write past the end of a row"
    assert bool((b[rows:] == sentinel).all()), "write past the last row"


@pytest.mark.parametrize("T,d", [(257, 2056), (33, 14336), (5, 96), (1000, 4096)])
def test_k1_writes_in_bounds(cuda, T, d, k1_kernel):
    rng = np.random.default_rng(T + d)
    x = torch.from_numpy(_acts(rng, T, d)).to(cuda).bfloat16()
    s = _smooth(rng, 4, d)
    group = rng.integers(0, 4, size=T).astype(np.int32)
    sd, gd = torch.from_numpy(s).to(cuda), torch.from_numpy(group).to(cuda)
    rec = torch.from_numpy(_true_records(x.float().cpu().numpy(), (1.0 / s).astype(np.float32)[group])).to(cuda)
    for ext in (None, rec):
        want = ops.act_quant(x, smooth=sd, row_group=gd, row_ext=ext)
        buf, view = _carve(T, d, torch.uint8, cuda, 0xA5)
        got = ops.act_quant(x, smooth=sd, row_group=gd, row_ext=ext, out_codes=view)
        torch.cuda.synchronize()
        _assert_margins(buf, T, d, 0xA5)
        assert torch.equal(view, want["codes"]) and torch.equal(got["scale"], want["scale"])


@pytest.mark.parametrize("mode", [1, 2])
def test_k1_tokens_writes_in_bounds(cuda, mode):
    rng = np.random.default_rng(7)
    T, d, k, G = 700, 4096, 2, 8
    x = torch.from_numpy(_acts(rng, T, d)).to(cuda).bfloat16()
    s = torch.from_numpy(_smooth(rng, G, d)).to(cuda)
    rec, rec32 = ops.reciprocal(s, with_f32=True)
    pos = torch.from_numpy(rng.permutation(T * k).astype(np.int32).reshape(T, k)).to(cuda)
    grp = torch.from_numpy(rng.integers(0, G, size=T * k).astype(np.int32)).to(cuda)
    with L.tuned(L.TUNE_K1_TOKENS, mode):
        want = ops.act_quant_tokens(x, pos, grp, smooth=s, smooth_recip=rec, smooth_recip_f32=rec32)
        buf, view = _carve(T * k, d, torch.uint8, cuda, 0x5A)
        ops.act_quant_tokens(x, pos, grp, smooth=s, smooth_recip=rec, smooth_recip_f32=rec32, out_codes=view)
    torch.cuda.synchronize()
    _assert_margins(buf, T * k, d, 0x5A)
    assert torch.equal(view, want["codes"])


@pytest.mark.parametrize("counts,F,K", [([700, 0, 1301, 3], 384, 512), ([2100, 77, 1500], 512, 1024)])
def test_grouped_gemm_writes_in_bounds(cuda, counts, F, K):
    """SwiGLU (TMA-stored bf16 h + extreme records) and dequant epilogues of
    the grouped GEMM, single-CTA and CTA-pair tiles, partial m / n tiles."""
    rng = np.random.default_rng(sum(counts) + F)
    E = len(counts)
    offs = torch.from_numpy(np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)).to(cuda)
    Mt = int(sum(counts))
    a = _dev_operand(cuda, *_rand_operand(rng, Mt, K))
    w13 = _dev_operand(cuda, *_rand_operand(rng, E * 2 * F, K))
    s2 = torch.from_numpy(_smooth(rng, E, F)).to(cuda)
    _, r32 = ops.reciprocal(s2, with_f32=True)
    ext = torch.empty((Mt, 2), dtype=torch.int64, device=cuda)
    want = ops.w8a8_gemm(a, w13, epilogue=L.EPI_SWIGLU, out_dtype=torch.bfloat16, group_offsets=offs,
                         num_groups=E, n_per_group=2 * F, next_smooth_recip_f32=r32, row_ext=ext)
    buf, view = _carve(Mt, F, torch.bfloat16, cuda, 0x7B)
    ext2 = torch.empty((Mt, 2), dtype=torch.int64, device=cuda)
    ops.w8a8_gemm(a, w13, epilogue=L.EPI_SWIGLU, out_dtype=torch.bfloat16, group_offsets=offs, num_groups=E,
                  n_per_group=2 * F, next_smooth_recip_f32=r32, row_ext=ext2, out=view)
    torch.cuda.synchronize()
    _assert_margins(buf, Mt, F, 0x7B)
    assert torch.equal(view, want) and torch.equal(ext, ext2)
    N = 328                                                       # partial last 256-wide N tile
    w2 = _dev_operand(cuda, *_rand_operand(rng, E * N, K))
    for dt in (torch.float32, torch.bfloat16):
        want = ops.w8a8_gemm(a, w2, epilogue=L.EPI_DEQUANT, out_dtype=dt, group_offsets=offs, num_groups=E,
                             n_per_group=N)
        buf, view = _carve(Mt, N, dt, cuda, 0x6C)
        ops.w8a8_gemm(a, w2, epilogue=L.EPI_DEQUANT, out_dtype=dt, group_offsets=offs, num_groups=E,
                      n_per_group=N, out=view)
        torch.cuda.synchronize()
        _assert_margins(buf, Mt, N, 0x6C)
        assert torch.equal(view, want)


@pytest.mark.parametrize("T", [1000, 9])
def test_moe_forward_writes_in_bounds(cuda, T):
    """The whole layer writing into a carved output (fused GEMM2 + top-2
    combine at 1000 tokens, the separate combine kernel at decode size)."""
    layer = MoELayer.random(8, 512, 1024, top_k=2, seed=3)
    rng = np.random.default_rng(T)
    x = torch.from_numpy(bf16_round(rng.normal(size=(T, 512)).astype(np.float32))).to(cuda).bfloat16()
    want = layer.forward(x)
    buf, view = _carve(T, 512, torch.bfloat16, cuda, 0x3D)
    layer.forward(x, out=view)
    torch.cuda.synchronize()
    _assert_margins(buf, T, 512, 0x3D)
    assert torch.equal(view, want)


# ── reads: input rows live inside wider buffers whose margins are poisoned;
# a kernel that read past a row end (or past the last row) would change its
# result ────────────────────────────────────────────────────────────────────
def _poisoned_view(src: torch.Tensor, pad_c: int, fill_byte: int) -> torch.Tensor:
    rows, cols = src.shape
    buf = torch.empty((rows + PAD_R, cols + pad_c), dtype=src.dtype, device=src.device)
    buf.view(torch.uint8).fill_(fill_byte)
    view = buf[:rows, :cols]
    view.copy_(src)
    return view


@pytest.mark.parametrize("T,d", [(257, 2056), (33, 14336), (1000, 4096)])
def test_k1_reads_in_bounds(cuda, T, d, k1_kernel):
    rng = np.random.default_rng(T * 3 + d)
    x = torch.from_numpy(_acts(rng, T, d)).to(cuda).bfloat16()
    xp = _poisoned_view(x, PAD_C, 0xFF)                           # bf16 0xFFFF = NaN
    s = torch.from_numpy(_smooth(rng, 1, d)).to(cuda)
    rec = torch.from_numpy(_true_records(x.float().cpu().numpy(),
                                         np.broadcast_to((1.0 / s.cpu().numpy()).astype(np.float32), (T, d)))).to(cuda)
    for ext in (None, rec):
        want = ops.act_quant(x, smooth=s, row_ext=ext)
        got = ops.act_quant(xp, smooth=s, row_ext=ext)
        for key in ("codes", "scale", "zp", "rowsum"):
            assert torch.equal(got[key], want[key]), key


@pytest.mark.parametrize("mode", [1, 2])
def test_k1_tokens_reads_in_bounds(cuda, mode):
    rng = np.random.default_rng(11)
    T, d, k, G = 600, 4096, 2, 8
    x = torch.from_numpy(_acts(rng, T, d)).to(cuda).bfloat16()
    xp = _poisoned_view(x, PAD_C, 0xFF)
    s = torch.from_numpy(_smooth(rng, G, d)).to(cuda)
    rec, rec32 = ops.reciprocal(s, with_f32=True)
    pos = torch.from_numpy(rng.permutation(T * k).astype(np.int32).reshape(T, k)).to(cuda)
    grp = torch.from_numpy(rng.integers(0, G, size=T * k).astype(np.int32)).to(cuda)
    with L.tuned(L.TUNE_K1_TOKENS, mode):
        want = ops.act_quant_tokens(x, pos, grp, smooth=s, smooth_recip=rec, smooth_recip_f32=rec32)
        got = ops.act_quant_tokens(xp, pos, grp, smooth=s, smooth_recip=rec, smooth_recip_f32=rec32)
    for key in ("codes", "scale", "zp", "rowsum"):
        assert torch.equal(got[key], want[key]), key


@pytest.mark.parametrize("M_,N,K", [(300, 512, 520), (2500, 768, 4096), (2049, 328, 1040)])
def test_gemm_reads_in_bounds(cuda, M_, N, K):
    """A and W codes with row strides past K (margins 0xFF): the TMA boxes of
    the last k-block must stop at K (zero fill), not read the neighbour bytes."""
    rng = np.random.default_rng(M_ + N + K)
    a = _dev_operand(cuda, *_rand_operand(rng, M_, K))
    w = _dev_operand(cuda, *_rand_operand(rng, N, K))
    want = ops.w8a8_gemm(a, w, epilogue=L.EPI_ACC_I32)
    ap = dict(a, codes=_poisoned_view(a["codes"], 48, 0xFF))
    wp = dict(w, codes=_poisoned_view(w["codes"], 48, 0xFF))
    assert torch.equal(ops.w8a8_gemm(ap, wp, epilogue=L.EPI_ACC_I32), want)
    want = ops.w8a8_gemm(a, w, epilogue=L.EPI_DEQUANT, out_dtype=torch.bfloat16)
    assert torch.equal(ops.w8a8_gemm(ap, wp, epilogue=L.EPI_DEQUANT, out_dtype=torch.bfloat16), want)


@pytest.mark.parametrize("T", [16, 300, 9000])
def test_router_reads_in_bounds(cuda, T):
    """Tensor-core router (cluster kernel for small batches, persistent
    kernel for large ones) and the SIMT router on token rows with poisoned
    margins and a ragged last 128-token tile: identical logits, ids, weights."""
    rng = np.random.default_rng(T)
    d, E = 1024, 8
    x = torch.from_numpy(bf16_round(rng.normal(size=(T, d)).astype(np.float32))).to(cuda).bfloat16()
    xp = _poisoned_view(x, 64, 0xFF)
    gw = torch.from_numpy(rng.normal(size=(E, d)).astype(np.float32) / np.sqrt(d)).to(cuda)
    for tc in (True, False):
        want = ops.router_gate(x, gw, 2, tensor_cores=tc)
        got = ops.router_gate(xp, gw, 2, tensor_cores=tc)
        for a, b in zip(got, want):
            assert torch.equal(a, b)


def test_gather_rows_writes_in_bounds(cuda):
    rng = np.random.default_rng(4)
    src = torch.from_numpy(rng.integers(0, 256, size=(500, 1000)).astype(np.uint8)).to(cuda)
    idx = torch.from_numpy(rng.integers(0, 500, size=777).astype(np.int32)).to(cuda)
    buf, view = _carve(777, 1000, torch.uint8, cuda, 0x11)
    ops.gather_rows(_poisoned_view(src, 24, 0x22), idx, out=view)
    torch.cuda.synchronize()
    _assert_margins(buf, 777, 1000, 0x11)
    assert torch.equal(view, src[idx.long()])


def test_rope_writes_in_bounds(cuda):
    """RoPE rotates only the first heads * head_dim columns of each row (the
    q and k heads of the fused QKV rows): v columns and margins untouched."""
    rng = np.random.default_rng(6)
    T, heads, hd, extra = 77, 12, 128, 4 * 128
    cos, sin = ops.rope_tables(4096, hd)
    x = torch.from_numpy(bf16_round(rng.normal(size=(T, heads * hd + extra)).astype(np.float32))).to(cuda).bfloat16()
    buf, view = _carve(T, x.shape[1], torch.bfloat16, cuda, 0x44)
    view.copy_(x)
    pos = torch.from_numpy(rng.integers(0, 4096, size=T).astype(np.int32)).to(cuda)
    ops.rope_(view, heads, hd, cos, sin, positions=pos)
    want = ops.rope_(x.clone(), heads, hd, cos, sin, positions=pos)
    torch.cuda.synchronize()
    _assert_margins(buf, T, x.shape[1], 0x44)
    assert torch.equal(view[:, heads * hd:], x[:, heads * hd:])
    assert torch.equal(view, want)


def test_apply_smoothing_strided_inputs(cuda):
    """apply_smoothing on transposed / column-sliced views equals the dense call."""
    rng = np.random.default_rng(8)
    w = torch.from_numpy(rng.normal(size=(96, 64))).to(cuda)
    x = torch.from_numpy(rng.normal(size=(64, 40))).to(cuda)
    f = torch.from_numpy(np.exp(rng.normal(size=64))).to(cuda)
    want = ops.apply_smoothing(w, x, f)
    wt = w.t().contiguous().t()                                  # same values, column-major storage
    xs = torch.cat([x, x], dim=1)[:, :40]                        # row stride 80
    got = ops.apply_smoothing(wt, xs, f)
    assert torch.equal(got[0], want[0]) and torch.equal(got[1], want[1])


def test_index_dtypes_refused(cuda):
    """Index and per-row arguments are raw int32 / float32 arrays to the
    kernels: a tensor of another dtype raises instead of being reinterpreted."""
    x = torch.zeros((4, 64), dtype=torch.bfloat16, device=cuda)
    s = torch.ones((2, 64), dtype=torch.float64, device=cuda)
    with pytest.raises(ValueError, match="row_group"):
        ops.act_quant(x, smooth=s, row_group=torch.zeros(4, dtype=torch.int64, device=cuda))
    with pytest.raises(ValueError, match="gather"):
        ops.act_quant(x, gather=torch.zeros(4, dtype=torch.int64, device=cuda))
    with pytest.raises(ValueError, match="idx"):
        ops.route_permute(torch.zeros((4, 2), dtype=torch.int64, device=cuda), None, 8)
    with pytest.raises(ValueError, match="token_pos"):
        ops.combine(torch.zeros((8, 64), dtype=torch.bfloat16, device=cuda),
                    torch.arange(8, dtype=torch.int64, device=cuda), 4, 2)
    with pytest.raises(ValueError, match="smoothing table"):
        ops.act_quant(x, smooth=s.float())


@pytest.mark.parametrize("T", [9, 1000, 2600])
def test_moe_forward_strided_input(cuda, T):
    """The layer on token rows that are a column slice of wider rows (row
    stride > d, margins poisoned) equals the layer on the dense rows."""
    layer = MoELayer.random(8, 512, 1024, top_k=2, seed=5)
    rng = np.random.default_rng(T + 1)
    x = torch.from_numpy(bf16_round(rng.normal(size=(T, 512)).astype(np.float32))).to(cuda).bfloat16()
    assert torch.equal(layer.forward(_poisoned_view(x, 64, 0xFF)), layer.forward(x))


@pytest.mark.parametrize("T", [9, 1000])
def test_moe_forward_nonfinite_tokens_are_contained(cuda, T):
    """The reference refuses non-finite input (numkit.py:52-53); the device
    forward does not scan for it (that would need a host sync), so a NaN /
    Inf token must at least stay contained: no fault, no hang, valid routing
    ids, and every other token's output bit-identical to the clean batch."""
    layer = MoELayer.random(8, 512, 1024, top_k=2, seed=5)
    rng = np.random.default_rng(T + 2)
    x = torch.from_numpy(bf16_round(rng.normal(size=(T, 512)).astype(np.float32))).to(cuda).bfloat16()
    clean = layer.forward(x)
    bad = x.clone()
    bad[0, 3] = float("nan")
    bad[T // 2, :] = float("inf")
    bad[T - 1, 7] = float("-inf")
    out = layer.forward(bad)                      # default path (fused combine at 1000 tokens)
    _, aux = layer.forward(bad, return_aux=True)
    torch.cuda.synchronize()
    idx = aux["idx"]
    assert bool(((idx >= 0) & (idx < 8)).all())
    keep = torch.ones(T, dtype=torch.bool, device=cuda)
    keep[[0, T // 2, T - 1]] = False
    assert torch.equal(out[keep], clean[keep])
