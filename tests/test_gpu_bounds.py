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
