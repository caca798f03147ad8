"""GPU parity of each kernel against the CPU oracle on identical inputs.

Bar (north star): INT8 codes, zero points, scales (float64), expert
assignments, permutations and INT32 accumulators are BIT-EXACT; dequantised
float outputs are within rtol 1e-5 (float32 epilogue vs float64 oracle on
the same exact accumulators), well inside the stated 1e-3.
"""

import numpy as np
import pytest
import torch

from oracle import moe_ref as M
from oracle import quant_ref as Q
from paper_2508_07329_b200 import _lib as L
from paper_2508_07329_b200 import ops

from .conftest import bf16_round

pytestmark = pytest.mark.gpu

RTOL_DEQ = 1e-5


def _acts(rng, T, d, outlier_frac=0.01, scale=100.0):
    x = rng.normal(size=(T, d)).astype(np.float32)
    cols = rng.choice(d, max(1, int(d * outlier_frac)), replace=False)
    x[:, cols] *= scale
    return bf16_round(x)


def _smooth(rng, G, d):
    return np.exp(rng.normal(size=(G, d)) * 0.7)


# ── K1 ───────────────────────────────────────────────────────────────────
@pytest.mark.parametrize("T,d", [(64, 96), (257, 1024), (1024, 4096), (33, 14336)])
def test_act_quant_per_token_bitexact(cuda, T, d, k1_kernel):
    rng = np.random.default_rng(T + d)
    x = _acts(rng, T, d)
    s = _smooth(rng, 1, d)
    xd = torch.from_numpy(x).to(cuda).to(torch.bfloat16)
    r = ops.act_quant(xd, smooth=torch.from_numpy(s).to(cuda))
    codes, scale, zp, rs = M.quantize_rows(x.astype(np.float64), s[0])
    np.testing.assert_array_equal(r["codes"].cpu().numpy(), codes)
    np.testing.assert_array_equal(r["scale"].cpu().numpy(), scale)
    np.testing.assert_array_equal(r["zp"].cpu().numpy(), zp)
    np.testing.assert_array_equal(r["rowsum"].cpu().numpy(), rs)


def test_act_quant_gather_grouped_bitexact(cuda, k1_kernel):
    rng = np.random.default_rng(5)
    T, d, G = 300, 512, 8
    x = _acts(rng, T, d)
    s = _smooth(rng, G, d)
    gather = rng.integers(0, T, size=2 * T).astype(np.int32)
    group = rng.integers(0, G, size=2 * T).astype(np.int32)
    r = ops.act_quant(torch.from_numpy(x).to(cuda).bfloat16(), smooth=torch.from_numpy(s).to(cuda),
                      gather=torch.from_numpy(gather).to(cuda), row_group=torch.from_numpy(group).to(cuda))
    codes, scale, zp, rs = M.quantize_rows_grouped(x.astype(np.float64)[gather], group, s)
    np.testing.assert_array_equal(r["codes"].cpu().numpy(), codes)
    np.testing.assert_array_equal(r["scale"].cpu().numpy(), scale)
    np.testing.assert_array_equal(r["zp"].cpu().numpy(), zp)
    np.testing.assert_array_equal(r["rowsum"].cpu().numpy(), rs)


@pytest.mark.parametrize("sym", [False, True])
def test_act_quant_one_sided_rows(cuda, sym, k1_kernel):
    """ReLU-like rows (min exactly 0, many zeros), non-positive rows and
    symmetric codes take the general fast path (code window [0, 255] plus an
    explicit candidate check, zero extremes exempt): bit-exact vs the oracle."""
    rng = np.random.default_rng(31 + sym)
    T, d = 257, 2048
    x = rng.normal(size=(T, d)).astype(np.float32) * np.exp(rng.normal(size=(T, 1)))
    x[: T // 3] = np.maximum(x[: T // 3], 0.0)                 # ReLU rows: ~50 % exact zeros
    x[T // 3: 2 * T // 3] = -np.abs(x[T // 3: 2 * T // 3])     # non-positive rows
    x[5, :] = 0.0
    x[6, :] = 0.0
    x[6, 100] = 3.0                                             # a single non-zero
    x = bf16_round(x)
    s = _smooth(rng, 1, d)
    xd = torch.from_numpy(x).to(cuda).bfloat16()
    r = ops.act_quant(xd, smooth=torch.from_numpy(s).to(cuda), symmetric=sym)
    codes, sc, zp = Q.rtn(x.astype(np.float64) / s[0], Q.cfg(8, sym, "per_token"))
    np.testing.assert_array_equal(r["codes"].cpu().numpy(), codes)
    np.testing.assert_array_equal(r["scale"].cpu().numpy(), sc)
    np.testing.assert_array_equal(r["zp"].cpu().numpy(), zp)
    np.testing.assert_array_equal(r["rowsum"].cpu().numpy(), codes.astype(np.int64).sum(1))


def test_act_quant_golden_k1(cuda, golden, k1_kernel):
    x = golden["k1_x_bf16"]
    r = ops.act_quant(torch.from_numpy(x.astype(np.float32)).to(cuda).bfloat16(),
                      smooth=torch.from_numpy(golden["k1_smooth"]).to(cuda))
    np.testing.assert_array_equal(r["codes"].cpu().numpy(), golden["k1_codes"])
    np.testing.assert_array_equal(r["scale"].cpu().numpy(), golden["k1_scales"])
    np.testing.assert_array_equal(r["zp"].cpu().numpy(), golden["k1_zps"])


def test_act_quant_bf16_fast_path_ties(cuda, k1_kernel):
    """bf16 rows whose quotients land exactly on k + 0.5 (and next to it), plus
    all-positive rows far from zero (clip saturation) — the cases where the
    float32 filter must defer to the exact float64 path."""
    rows = []
    k = np.arange(0, 128)
    rows.append(np.r_[0.0, 255 / 8, (k + 0.5) / 8, np.zeros(6)])   # scale = 1/8 exactly -> ties
    rows.append(-np.r_[0.0, 255 / 8, (k + 0.5) / 8, np.zeros(6)])
    rows.append(100.0 + np.arange(136) / 64)                         # all positive, zp = 0, clipped
    rows.append(np.r_[np.full(68, 3.0), np.full(68, -1.0)])
    rng = np.random.default_rng(0)
    rows.append(rng.normal(size=136) * 1e-30)                        # tiny values
    rows.append(rng.normal(size=136) * 3e4)
    x = bf16_round(np.array(rows, dtype=np.float32))
    for s in (None, np.ones((1, 136)), np.exp(rng.normal(size=(1, 136)))):
        r = ops.act_quant(torch.from_numpy(x).to(cuda).bfloat16(),
                          smooth=None if s is None else torch.from_numpy(s).to(cuda))
        codes, sc, zp, rs = M.quantize_rows(x.astype(np.float64), None if s is None else s[0])
        np.testing.assert_array_equal(r["codes"].cpu().numpy(), codes)
        np.testing.assert_array_equal(r["scale"].cpu().numpy(), sc)
        np.testing.assert_array_equal(r["zp"].cpu().numpy(), zp)
        np.testing.assert_array_equal(r["rowsum"].cpu().numpy(), rs)


def test_act_quant_edge_values(cuda, k1_kernel):
    # constant rows (scale floor), all-zero rows, exact ties at .5 of the grid,
    # negative zero
    x = np.zeros((6, 64))
    x[1] = 5.0
    x[2] = np.linspace(-1, 3, 64)
    x[3, :] = -0.0
    x[4] = np.arange(64) * 0.5 - 7.25
    x[5] = np.r_[np.full(32, 0.49999999999999994), np.full(32, -0.5)]
    for gran in ("per_token", "per_tensor"):
        for bits in (2, 4, 8):
            for sym in (False, True):
                c = Q.cfg(bits, sym, gran)
                r = ops.act_quant(torch.from_numpy(x).to(cuda), bits=bits, symmetric=sym, granularity=gran)
                codes, sc, zp = Q.rtn(x, c)
                np.testing.assert_array_equal(r["codes"].cpu().numpy(), codes)
                np.testing.assert_array_equal(r["scale"].cpu().numpy(), sc)
                np.testing.assert_array_equal(r["zp"].cpu().numpy(), zp)


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("T,d,k,G", [(1, 8, 1, 1), (300, 512, 2, 8), (257, 1024, 4, 16), (1000, 4096, 2, 8),
                                      (70, 2056, 3, 5), (5, 4096, 8, 8), (40, 6144, 2, 4)])
def test_act_quant_tokens_bitexact(cuda, T, d, k, G, mode):
    """Token-major K1 (x read from HBM once per token; mode 1: all k expert
    rows encoded from one warp's registers, mode 2: the row kernel walking
    tokens in order, a token's rows on adjacent warps; d > 4096 always takes
    mode 2) == the oracle on the gathered rows, bit for bit, with per-row
    smoothing groups, ragged d (not a multiple of 256), tie rows, constant /
    zero / one-sided / tiny / huge rows."""
    rng = np.random.default_rng(T * 7 + d + k)
    x = _acts(rng, T, d)
    special = [np.zeros(d), np.full(d, 5.0), np.abs(x[0]) + 1.0, -np.abs(x[0]),
               rng.normal(size=d) * 1e-30, rng.normal(size=d) * 3e4,
               np.r_[0.0, 255 / 8, (np.arange(d - 2) % 255 + 0.5) / 8]]
    for i, row in enumerate(special[: T]):
        x[i] = bf16_round(np.asarray(row, np.float32))
    s = _smooth(rng, G, d)
    s[0] = 1.0                                     # exact-tie rows survive group 0
    # token_pos: a random permutation of the T*k rows; groups per row
    pos = rng.permutation(T * k).astype(np.int32).reshape(T, k)
    grp = rng.integers(0, G, size=T * k).astype(np.int32)
    grp[pos[: len(special), 0]] = 0
    sd = torch.from_numpy(s).to(cuda)
    rec, rec32 = ops.reciprocal(sd, with_f32=True)
    xd = torch.from_numpy(x).to(cuda).bfloat16()
    with L.tuned(L.TUNE_K1_TOKENS, mode):
        r = ops.act_quant_tokens(xd, torch.from_numpy(pos).to(cuda), torch.from_numpy(grp).to(cuda), smooth=sd,
                                 smooth_recip=rec, smooth_recip_f32=rec32)
    src = np.empty(T * k, np.int64)
    src[pos.ravel()] = np.repeat(np.arange(T), k)
    codes, sc, zp, rs = M.quantize_rows_grouped(x.astype(np.float64)[src], grp, s)
    np.testing.assert_array_equal(r["codes"].cpu().numpy(), codes)
    np.testing.assert_array_equal(r["scale"].cpu().numpy(), sc)
    np.testing.assert_array_equal(r["scale_f32"].cpu().numpy(), sc.astype(np.float32))
    np.testing.assert_array_equal(r["zp"].cpu().numpy(), zp)
    np.testing.assert_array_equal(r["rowsum"].cpu().numpy(), rs)


def _ext_key(v32, col):
    """(order-preserving key of a float32 << 32) | column, as int64 bits."""
    i = np.asarray(v32, np.float32).view(np.int32).astype(np.int64)
    u = np.where(i >= 0, i, i ^ 0x7FFFFFFF) & 0xFFFFFFFF
    k = u ^ 0x80000000
    return ((k << 32) | np.asarray(col, np.int64)).astype(np.uint64).view(np.int64)


def _true_records(x32, recip32):
    xs = x32 * recip32
    cM, cm = xs.argmax(1), xs.argmin(1)
    r = np.arange(len(xs))
    return np.stack([_ext_key(xs[r, cm], cm), _ext_key(xs[r, cM], cM)], 1)


def test_act_quant_row_ext_speculation(cuda, k1_kernel):
    """K1 fed (value, column) extreme records: correct records, records that
    point at the wrong element, stale values, duplicated extremes, empty
    (never-written) records and out-of-range columns all give the exact
    result — the kernel verifies the speculation and re-encodes on failure."""
    rng = np.random.default_rng(21)
    T, d, G = 96, 1024, 4
    x = _acts(rng, T, d)
    x[5, 7] = x[5, 900] = 50.0                                   # duplicated maximum
    x[6, 3] = x[6, 4] = -70.0                                    # duplicated minimum (same column scale below)
    s = _smooth(rng, G, d)
    s[:, 4] = s[:, 3]
    group = rng.integers(0, G, size=T).astype(np.int32)
    recip32 = (1.0 / s).astype(np.float32)
    rec = _true_records(x.astype(np.float32), recip32[group])
    bad = rec.copy()
    bad[10, 1] = _ext_key(np.float32(1e9), 3)                     # stale value
    bad[11, 0] = _ext_key(np.float32(-1e9), 5)
    bad[12, 1] = (bad[12, 1] & ~np.int64(0xFFFFFFFF)) | 17       # right value, wrong column
    bad[13] = [-1, 0]                                            # never written (init records)
    bad[14, 1] = (bad[14, 1] & ~np.int64(0xFFFFFFFF)) | (d + 5)  # column out of range
    xd = torch.from_numpy(x).to(cuda).bfloat16()
    sd = torch.from_numpy(s).to(cuda)
    gd = torch.from_numpy(group).to(cuda)
    want = M.quantize_rows_grouped(x.astype(np.float64), group, s)
    for records in (rec, bad):
        r = ops.act_quant(xd, smooth=sd, row_group=gd, row_ext=torch.from_numpy(records).to(cuda))
        for got, exp in zip((r["codes"], r["scale"], r["zp"], r["rowsum"]), want):
            np.testing.assert_array_equal(got.cpu().numpy(), exp)


def test_act_quant_near_rounding_boundaries(cuda, k1_kernel):
    """Rows whose quotients x / s / scale sit within +-2^-11 of half-integers
    (a quarter of them inside the float32 filter's margin band 2^-14 .. 2^-13
    around the boundary, and exact ties): every code, scale, zero point and
    row sum equals the float64 oracle's, with and without producer records.
    Each row's extremes are -127.5 and +127.5 (scale ~1, zero point 128), so
    the target quotient of column j is exactly what the smoothing encodes."""
    rng = np.random.default_rng(31)
    R, d = 64, 2048
    n = rng.integers(-120, 120, size=(R, d)).astype(np.float64)
    delta = rng.uniform(-2.0 ** -11, 2.0 ** -11, size=(R, d))
    band = rng.random(size=(R, d)) < 0.25
    delta[band] = np.sign(delta[band]) * rng.uniform(2.0 ** -14, 2.0 ** -13, size=int(band.sum()))
    delta[:, 2:40] = 0.0                                          # exact ties
    target = n + 0.5 + delta
    target[:, 0], target[:, 1] = 127.5, -127.5
    x = np.where(target < 0, -1.0, 1.0).astype(np.float32)        # bf16-exact
    s = 1.0 / np.abs(target)                                      # one smoothing group per row
    group = np.arange(R, dtype=np.int32)
    want = M.quantize_rows_grouped(x.astype(np.float64), group, s)
    assert ((want[2] >= 16) & (want[2] <= 239)).all()             # two-sided rows: the fast window applies
    xd = torch.from_numpy(x).to(cuda).bfloat16()
    sd = torch.from_numpy(s).to(cuda)
    gd = torch.from_numpy(group).to(cuda)
    recip32 = (1.0 / s).astype(np.float32)
    rec = _true_records(x, recip32)
    for records in (None, rec):
        r = ops.act_quant(xd, smooth=sd, row_group=gd,
                          row_ext=None if records is None else torch.from_numpy(records).to(cuda))
        for got, exp in zip((r["codes"], r["scale"], r["zp"], r["rowsum"]), want):
            np.testing.assert_array_equal(got.cpu().numpy(), exp)


def test_swiglu_row_ext_feeds_k1(cuda, k1_kernel):
    """The grouped SwiGLU epilogue's extreme records of h * RN32(1/s2) match
    the stored bf16 h, and K1 fed those records equals K1 without them."""
    rng = np.random.default_rng(22)
    E, F, K = 3, 512, 256
    counts = np.array([300, 0, 211])
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    Mt = int(offs[-1])
    a = _rand_operand(rng, Mt, K)
    w = _rand_operand(rng, E * 2 * F, K)
    s2 = _smooth(rng, E, F)
    s2d = torch.from_numpy(s2).to(cuda)
    recip, recip32 = ops.reciprocal(s2d, with_f32=True)
    od = torch.from_numpy(offs).to(cuda)
    ext = torch.empty((Mt, 2), dtype=torch.int64, device=cuda)
    h = ops.w8a8_gemm(_dev_operand(cuda, *a), _dev_operand(cuda, *w), epilogue=L.EPI_SWIGLU,
                      out_dtype=torch.bfloat16, group_offsets=od, num_groups=E, n_per_group=2 * F,
                      next_smooth_recip_f32=recip32, row_ext=ext)
    group = np.repeat(np.arange(E), counts).astype(np.int32)
    xs = h.float().cpu().numpy() * recip32.cpu().numpy()[group]
    e = ext.cpu().numpy().view(np.uint64)
    r = np.arange(Mt)
    want = _true_records(h.float().cpu().numpy(), recip32.cpu().numpy()[group]).view(np.uint64)
    np.testing.assert_array_equal(e >> np.uint64(32), want >> np.uint64(32))     # extreme values
    cols = (e & np.uint64(0xFFFFFFFF)).astype(np.int64)
    # the recorded column starts the 32-column chunk holding the extreme
    win = np.minimum(cols[:, :, None] + np.arange(32)[None, None, :], xs.shape[1] - 1)
    assert (xs[r[:, None], win[:, 0]] == xs.min(1)[:, None]).any(axis=1).all()
    assert (xs[r[:, None], win[:, 1]] == xs.max(1)[:, None]).any(axis=1).all()
    gd = torch.from_numpy(group).to(cuda)
    with_ext = ops.act_quant(h, smooth=s2d, smooth_recip=recip, smooth_recip_f32=recip32, row_group=gd,
                             row_ext=ext)
    plain = ops.act_quant(h, smooth=s2d, row_group=gd)
    for k in ("codes", "scale", "zp", "rowsum"):
        assert torch.equal(with_ext[k], plain[k]), k


# ── K2 / K5 ──────────────────────────────────────────────────────────────
def _rand_operand(rng, rows, K, zp_lo=0, zp_hi=255):
    codes = rng.integers(0, 256, size=(rows, K)).astype(np.uint8)
    zp = rng.integers(zp_lo, zp_hi + 1, size=rows).astype(np.int32)
    scale = np.exp(rng.normal(size=rows) - 4)
    return codes, zp, scale


def _dev_operand(cuda, codes, zp, scale):
    c = torch.from_numpy(codes).to(cuda)
    sc = torch.from_numpy(scale).to(cuda)
    return {"codes": c, "zp": torch.from_numpy(zp).to(cuda), "scale": sc, "scale_f32": sc.float(),
            "rowsum": c.sum(dim=1, dtype=torch.int32)}


@pytest.mark.parametrize("M_,N,K", [(300, 512, 512), (128, 256, 4096), (1000, 768, 272), (77, 40, 48),
                                    (513, 1024, 14336),
                                    # CTA-pair (cta_group::2) path: M >= 2048, ragged last tile
                                    (2500, 768, 4096), (4096, 512, 1024), (2049, 256, 14336),
                                    # N not a multiple of the 256-wide tile (partial last N tile)
                                    (2300, 200, 512), (700, 328, 256)])
def test_gemm_accumulators_bitexact(cuda, M_, N, K):
    rng = np.random.default_rng(M_ * 7 + N + K)
    a = _rand_operand(rng, M_, K)
    w = _rand_operand(rng, N, K)
    acc = ops.w8a8_gemm(_dev_operand(cuda, *a), _dev_operand(cuda, *w), epilogue=L.EPI_ACC_I32)
    want = M.int_acc(a[0], a[1], w[0], w[1])
    np.testing.assert_array_equal(acc.cpu().numpy().astype(np.int64), want)


def test_gemm_extreme_zero_points(cuda):
    # all-255 codes with zp 0 vs all-0 codes with zp 255: |acc| = K*255^2
    K = 33024
    a = (np.full((128, K), 255, np.uint8), np.zeros(128, np.int32), np.ones(128))
    w = (np.zeros((256, K), np.uint8), np.full(256, 255, np.int32), np.ones(256))
    acc = ops.w8a8_gemm(_dev_operand(cuda, *a), _dev_operand(cuda, *w), epilogue=L.EPI_ACC_I32)
    assert (acc.cpu().numpy() == -K * 255 * 255).all()


@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_gemm_dequant_epilogue(cuda, out_dtype):
    rng = np.random.default_rng(11)
    M_, N, K = 333, 512, 1024
    a, w = _rand_operand(rng, M_, K), _rand_operand(rng, N, K)
    bias = rng.normal(size=N).astype(np.float32)
    y = ops.w8a8_gemm(_dev_operand(cuda, *a), _dev_operand(cuda, *w), out_dtype=out_dtype,
                      bias=torch.from_numpy(bias).to(cuda))
    want, _ = M.w8a8_linear(a[0], a[2], a[1], w[0], w[2], w[1], bias)
    tol = RTOL_DEQ if out_dtype == torch.float32 else 2.0 ** -8
    np.testing.assert_allclose(y.float().cpu().numpy(), want, rtol=tol, atol=tol * np.abs(want).max() * 1e-3)


@pytest.mark.parametrize("counts", [[0, 129, 1, 300, 77], [0, 1029, 1, 1300, 777], [2048, 0, 256, 513, 3]])
def test_grouped_gemm_ragged(cuda, counts):
    rng = np.random.default_rng(12)
    E, N, K = 5, 256, 512
    counts = np.array(counts)
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    Mt = int(offs[-1])
    a = _rand_operand(rng, Mt, K)
    w = _rand_operand(rng, E * N, K)
    rw = rng.random(Mt).astype(np.float32)
    od = torch.from_numpy(offs).to(cuda)
    acc = ops.w8a8_gemm(_dev_operand(cuda, *a), _dev_operand(cuda, *w), epilogue=L.EPI_ACC_I32,
                        group_offsets=od, num_groups=E, n_per_group=N).cpu().numpy()
    y = ops.w8a8_gemm(_dev_operand(cuda, *a), _dev_operand(cuda, *w), row_weight=torch.from_numpy(rw).to(cuda),
                      group_offsets=od, num_groups=E, n_per_group=N).cpu().numpy()
    for e in range(E):
        lo, hi = offs[e], offs[e + 1]
        if hi == lo:
            continue
        sl = slice(e * N, (e + 1) * N)
        want_acc = M.int_acc(a[0][lo:hi], a[1][lo:hi], w[0][sl], w[1][sl])
        np.testing.assert_array_equal(acc[lo:hi].astype(np.int64), want_acc)
        want_y = (a[2][lo:hi, None] * w[2][None, sl]) * want_acc * rw[lo:hi, None]
        np.testing.assert_allclose(y[lo:hi], want_y, rtol=RTOL_DEQ, atol=1e-12)


def test_swiglu_epilogue(cuda):
    rng = np.random.default_rng(13)
    M_, F, K = 200, 384, 512
    a = _rand_operand(rng, M_, K)
    w = _rand_operand(rng, 2 * F, K)             # interleaved blocks of 128 (gate, up)
    h = ops.w8a8_gemm(_dev_operand(cuda, *a), _dev_operand(cuda, *w), epilogue=L.EPI_SWIGLU,
                      out_dtype=torch.float32).cpu().numpy()
    y, _ = M.w8a8_linear(a[0], a[2], a[1], w[0], w[2], w[1])
    blk = y.reshape(M_, F // 128, 2, 128)
    want = (M.silu(blk[:, :, 0]) * blk[:, :, 1]).reshape(M_, F)
    np.testing.assert_allclose(h, want, rtol=1e-4, atol=1e-6 * np.abs(want).max())


# ── K3 / K4 / K6 ─────────────────────────────────────────────────────────
@pytest.mark.parametrize("E,k,T,d", [(8, 2, 2048, 1024), (16, 4, 2048, 1024), (5, 1, 2048, 1024),
                                     (8, 2, 333, 256), (8, 2, 1001, 4096), (7, 3, 517, 512), (8, 2, 77, 96)])
@pytest.mark.parametrize("tc", [False, True])
def test_router_gate_topk(cuda, E, k, T, d, tc):
    """SIMT kernels (register gate for d % 256 == 0, d <= 4096, E <= 8 with
    1-16 warps per CTA and ragged batches; shared-memory; generic) and the
    tensor-core kernel (bf16 3-piece gate, d % 64 == 0, E <= 16)."""
    if tc and (d % 64 or E > 16):
        pytest.skip("shape outside the tensor-core router")
    rng = np.random.default_rng(E * 10 + k + d)
    x = _acts(rng, T, d, scale=3.0)
    wg = (rng.normal(size=(E, d)) / np.sqrt(d)).astype(np.float32)
    gb = rng.normal(size=E).astype(np.float32) * 0.1
    logits, idx, w = ops.router_gate(torch.from_numpy(x).to(cuda).bfloat16(), torch.from_numpy(wg).to(cuda), k,
                                     gate_bias=torch.from_numpy(gb).to(cuda), tensor_cores=tc)
    lg = logits.cpu().numpy()
    want = x.astype(np.float64) @ wg.T.astype(np.float64) + gb
    np.testing.assert_allclose(lg, want, rtol=1e-5, atol=1e-5 * np.abs(want).max())
    oidx, ow, _ = M.router_topk(lg, k)               # identical float32 logits
    np.testing.assert_array_equal(idx.cpu().numpy(), oidx)
    np.testing.assert_allclose(w.cpu().numpy(), ow, rtol=1e-5, atol=1e-9)  # float32 expf


@pytest.mark.parametrize("d", [256, 640, 1024, 4096])
def test_router_tc_cluster_and_persistent_agree(cuda, d):
    """The two tensor-core router kernels — K split over a thread-block
    cluster (small batches) and the persistent multi-accumulator kernel
    (large batches) — give bit-identical logits, ids and weights, so a
    token's routing does not depend on its batch size."""
    from paper_2508_07329_b200 import _lib
    rng = np.random.default_rng(d)
    x = torch.from_numpy(_acts(rng, 3000, d, scale=3.0)).to(cuda).bfloat16()
    wg = torch.from_numpy((rng.normal(size=(8, d)) / np.sqrt(d)).astype(np.float32)).to(cuda)
    gb = torch.from_numpy(rng.normal(size=8).astype(np.float32) * 0.1).to(cuda)
    for T in (1, 100, 700, 3000):
        outs = []
        for tiles in (1 << 40, 0):
            with _lib.tuned(_lib.TUNE_ROUTER_CLUSTER_TILES, tiles):
                outs.append(ops.router_gate(x[:T], wg, 2, gate_bias=gb, tensor_cores=True))
        for a, b in zip(*outs):
            assert torch.equal(a, b), (d, T)
    full = ops.router_gate(x, wg, 2, gate_bias=gb, tensor_cores=True)
    one = ops.router_gate(x[:5], wg, 2, gate_bias=gb, tensor_cores=True)
    for a, b in zip(full, one):
        assert torch.equal(a[:5], b)


@pytest.mark.parametrize("T,d", [(37, 4096), (5, 1024), (300, 256)])
def test_rmsnorm_residual(cuda, T, d):
    """Stack glue kernel: residual add exactly as bf16(float(x) + float(y)),
    RMSNorm within one bf16 ulp of a float32 torch reference, rows
    independent of the batch."""
    rng = np.random.default_rng(T + d)
    x = torch.from_numpy(rng.normal(size=(T, d)).astype(np.float32) * 3).to(cuda).bfloat16()
    y = torch.from_numpy(rng.normal(size=(T, d)).astype(np.float32)).to(cuda).bfloat16()
    s, n = ops.rmsnorm_residual(x, y)
    assert torch.equal(s, (x.float() + y.float()).to(torch.bfloat16))
    sf = s.float()
    ref = sf * torch.rsqrt(sf.pow(2).mean(dim=-1, keepdim=True) + 1e-5)
    torch.testing.assert_close(n.float(), ref, rtol=2 ** -7, atol=1e-6)
    _, n2 = ops.rmsnorm_residual(s, None)
    assert torch.equal(n2, n)                       # fused norm == norm of the sum
    _, n3 = ops.rmsnorm_residual(s[: T // 2 + 1].contiguous(), None)
    assert torch.equal(n3, n[: T // 2 + 1])


def test_router_topk_ties(cuda):
    lg = np.array([[1, 1, 1, 1], [0, 2, 2, 0], [3, 3, 1, 3], [-1, -1, -1, -2]], dtype=np.float32)
    idx, w = ops.router_topk(torch.from_numpy(lg).to(cuda), 2)
    np.testing.assert_array_equal(idx.cpu().numpy(), [[0, 1], [1, 2], [0, 1], [0, 1]])
    np.testing.assert_allclose(w.cpu().numpy(), 0.5, rtol=1e-7)


@pytest.mark.parametrize("T,k,E", [(4096, 2, 8), (1, 2, 8), (5000, 4, 16), (777, 1, 3), (70000, 2, 8), (20000, 4, 64)])
def test_route_permute(cuda, T, k, E):
    rng = np.random.default_rng(T + k + E)
    idx = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
    w = rng.random((T, k)).astype(np.float32)
    p = ops.route_permute(torch.from_numpy(idx).to(cuda), torch.from_numpy(w).to(cuda), E)
    offs, tok, slot, pos = M.permute(idx, E)
    np.testing.assert_array_equal(p["offsets"].cpu().numpy(), offs)
    np.testing.assert_array_equal(p["src_token"].cpu().numpy(), tok)
    np.testing.assert_array_equal(p["token_pos"].cpu().numpy(), pos.ravel())
    np.testing.assert_array_equal(p["row_expert"].cpu().numpy(), idx[tok, slot])
    np.testing.assert_array_equal(p["row_weight"].cpu().numpy(), w[tok, slot])


def test_combine(cuda):
    rng = np.random.default_rng(3)
    T, k, d = 500, 2, 1024
    y = rng.normal(size=(T * k, d)).astype(np.float32)
    pos = rng.permutation(T * k).astype(np.int32)
    out = ops.combine(torch.from_numpy(y).to(cuda), torch.from_numpy(pos).to(cuda), T, k,
                      out_dtype=torch.float32).cpu().numpy()
    want = y[pos.reshape(T, k)].sum(axis=1)
    np.testing.assert_allclose(out, want, rtol=1e-6, atol=1e-6)


def test_expert_histogram(cuda):
    rng = np.random.default_rng(4)
    T, k, E = 3000, 2, 8
    idx = np.stack([np.sort(rng.permutation(E)[:k]) for _ in range(T)]).astype(np.int32)
    counts = torch.zeros((2, E), dtype=torch.int64, device=cuda)
    masks = torch.empty(T, dtype=torch.int32, device=cuda)
    ops.expert_histogram(torch.from_numpy(idx).to(cuda), E, 1, counts, masks)
    np.testing.assert_array_equal(counts.cpu().numpy()[1], np.bincount(idx.ravel(), minlength=E))
    np.testing.assert_array_equal(masks.cpu().numpy(), (1 << idx).sum(axis=1))


# ── K7 / K8 ──────────────────────────────────────────────────────────────
def test_hessian_matches_oracle(cuda):
    rng = np.random.default_rng(6)
    n, T = 200, 333
    x = rng.normal(size=(n, T))
    x[3] *= 40
    s = np.exp(rng.normal(size=n) * 0.5)
    H = ops.hessian(torch.from_numpy((x / s[:, None]).T.copy()).to(cuda)).cpu().numpy()
    np.testing.assert_allclose(H, Q.build_hessian(x / s[:, None]), rtol=1e-12, atol=1e-9)
    Hs = ops.hessian(torch.from_numpy(x.T.copy()).to(cuda), smooth=torch.from_numpy(s).to(cuda)).cpu().numpy()
    np.testing.assert_allclose(Hs, Q.build_hessian(x / s[:, None]), rtol=1e-12, atol=1e-9)
    assert np.array_equal(Hs, Hs.T)


@pytest.mark.parametrize("R,n,bits,permute", [(10, 24, 4, False), (130, 256, 8, True), (64, 300, 3, False)])
def test_gptq_columns_bitexact_given_u(cuda, R, n, bits, permute):
    rng = np.random.default_rng(R + n)
    x = rng.normal(size=(n, 4 * n // 3 + 8))
    w = rng.normal(size=(R, n))
    h = Q.build_hessian(x)
    order = rng.permutation(n) if permute else np.arange(n)
    U = Q.inverse_upper_factor(h[np.ix_(order, order)])
    c = Q.cfg(bits)
    sc, zp = Q.affine(w.min(axis=1), w.max(axis=1), c)
    want_p = Q.gptq_columns(w[:, order], U, sc, zp, (1 << bits) - 1)
    want = np.empty_like(want_p)
    want[:, order] = want_p
    got = ops.gptq_columns(torch.from_numpy(w).to(cuda), torch.from_numpy(U).to(cuda),
                           torch.from_numpy(sc).to(cuda), torch.from_numpy(zp).to(cuda), bits,
                           torch.from_numpy(order).to(cuda) if permute else None)
    np.testing.assert_array_equal(got.cpu().numpy(), want)


def _gptq_case(rng, R, n, bits, cuda):
    """W [R, n] and the given U from a real (GPU, float64) damped Hessian
    inverse factor; the oracle column loop runs on the same U."""
    x = torch.from_numpy(rng.normal(size=(n, n + 64))).to(cuda)
    H = 2.0 * x @ x.T
    H += 0.01 * H.diagonal().mean() * torch.eye(n, device=cuda, dtype=torch.float64)
    U = torch.linalg.cholesky(torch.cholesky_inverse(torch.linalg.cholesky(H))).T.contiguous()
    w = rng.normal(size=(R, n)) * 0.02
    sc, zp = Q.affine(w.min(axis=1), w.max(axis=1), Q.cfg(bits))
    return w, U, sc, zp


@pytest.mark.parametrize("n", [4096, 14336])
@pytest.mark.parametrize("lanes", [8, 16, 32])
def test_gptq_columns_bitexact_mixtral_shapes(cuda, n, lanes):
    """K8 at the Mixtral expert shapes (W1||W3: n = d = 4096; W2: n = ffn =
    14336) on a 64-row slice (rows are independent, quant.py:423-430), with
    every lane split forced: 8 lanes per row (4 contiguous tile columns
    each), 16 (2 each: the automatic choice) and 32 (one each)."""
    rng = np.random.default_rng(n + lanes)
    w, U, sc, zp = _gptq_case(rng, 64, n, 8, cuda)
    want = Q.gptq_columns(w, U.cpu().numpy(), sc, zp, 255)
    with L.tuned(L.TUNE_GPTQ_LANES, lanes):
        got = ops.gptq_columns(torch.from_numpy(w).to(cuda), U, torch.from_numpy(sc).to(cuda),
                               torch.from_numpy(zp).to(cuda), 8)
    np.testing.assert_array_equal(got.cpu().numpy(), want)


def test_gptq_columns_bitexact_many_rows(cuda):
    """More than 8192 rows with the automatic lane split (16 lanes per row)."""
    rng = np.random.default_rng(9)
    w, U, sc, zp = _gptq_case(rng, 8200, 96, 8, cuda)
    want = Q.gptq_columns(w, U.cpu().numpy(), sc, zp, 255)
    got = ops.gptq_columns(torch.from_numpy(w).to(cuda), U, torch.from_numpy(sc).to(cuda),
                           torch.from_numpy(zp).to(cuda), 8)
    np.testing.assert_array_equal(got.cpu().numpy(), want)


def test_gptq_columns_bad_factor_reports_pivot(cuda):
    """A factor whose diagonal is not positive: MOE_ENOTPD through the C ABI,
    raised as NotPositiveDefiniteError with the pivot and value
    (numkit.py:89-90) from moe_last_error_detail."""
    from paper_2508_07329_b200.errors import NotPositiveDefiniteError
    rng = np.random.default_rng(3)
    n = 40
    U = torch.eye(n, dtype=torch.float64, device=cuda)
    U[17, 17] = -0.25
    w = torch.from_numpy(rng.normal(size=(5, n))).to(cuda)
    sc = torch.full((5,), 0.01, dtype=torch.float64, device=cuda)
    zp = torch.full((5,), 128, dtype=torch.int32, device=cuda)
    with pytest.raises(NotPositiveDefiniteError) as exc:
        ops.gptq_columns(w, U, sc, zp, 8)
    assert exc.value.pivot == 17 and exc.value.value == -0.25


@pytest.mark.parametrize("n,T,dt", [(256, 100, "f64"), (300, 333, "f64"), (1000, 77, "bf16"), (640, 1, "f32")])
def test_hessian_dmma_matches_oracle(cuda, n, T, dt):
    """K7 on the FP64 tensor cores (DMMA, n >= 256): ragged tiles, a single
    token, bf16 / f32 / f64 inputs, fused smoothing division; rtol 1e-12
    against build_hessian (quant.py:327-343) and exactly symmetric."""
    rng = np.random.default_rng(n + T)
    x = rng.normal(size=(n, T))
    x[5] *= 30
    s = np.exp(rng.normal(size=n) * 0.5)
    tdt = {"f64": torch.float64, "f32": torch.float32, "bf16": torch.bfloat16}[dt]
    xt = torch.from_numpy(x.T.copy()).to(cuda).to(tdt)
    xr = xt.double().cpu().numpy().T
    Hs = ops.hessian(xt, smooth=torch.from_numpy(s).to(cuda)).cpu().numpy()
    np.testing.assert_allclose(Hs, Q.build_hessian(xr / s[:, None]), rtol=1e-12, atol=1e-9)
    assert np.array_equal(Hs, Hs.T)
    with pytest.raises(Exception):
        ops.hessian(torch.zeros((T, n), dtype=tdt, device=cuda))


def test_gemm_serpentine_order_bit_identical(cuda, tmp_path):
    """The grouped GEMM's serpentine k order (every other tile of a CTA pair
    walks k downwards, MOE_B200_GEMM_SERP, read once per process) cannot
    change a bit: int32 accumulation is exact. Same accumulators and dequant
    outputs with it on (this process) and off (a subprocess)."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2508_07329_b200 import _lib as L, ops
from tests.test_gpu_kernels import _rand_operand, _dev_operand
rng = np.random.default_rng(77)
a = _dev_operand("cuda", *_rand_operand(rng, 4096, 1040))
w = _dev_operand("cuda", *_rand_operand(rng, 2 * 2048, 1040))   # 17 m x 8 n = 136 tiles > 74 pairs
offs = torch.tensor([0, 1500, 4096], dtype=torch.int32, device="cuda")
acc = ops.w8a8_gemm(a, w, epilogue=L.EPI_ACC_I32, group_offsets=offs, num_groups=2, n_per_group=2048)
y = ops.w8a8_gemm(a, w, epilogue=L.EPI_DEQUANT, out_dtype=torch.bfloat16, group_offsets=offs, num_groups=2,
                  n_per_group=2048)
np.save(sys.argv[1], np.concatenate([acc.cpu().numpy().ravel().view(np.uint32),
                                     y.view(torch.int16).cpu().numpy().ravel().astype(np.uint32)]))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for serp in ("1", "0"):
        f = tmp_path / f"serp{serp}.npy"
        env = dict(os.environ, MOE_B200_GEMM_SERP=serp)
        subprocess.run([sys.executable, "-c", code, str(f)], cwd=root, env=env, check=True, timeout=300)
        outs.append(np.load(f))
    np.testing.assert_array_equal(outs[0], outs[1])


def test_act_quant_params_many_rows(cuda, k1_kernel):
    """Scale and zero point of 120k short rows whose extremes span ~60 decades
    (the fast kernels derive them through a corrected reciprocal instead of two
    IEEE divisions): bit-identical to the oracle's float64 divisions."""
    rng = np.random.default_rng(41)
    R, d = 120_000, 16
    mag = 10.0 ** rng.uniform(-30, 30, size=(R, 1))
    x = rng.normal(size=(R, d)) * mag
    x[::7] = np.abs(x[::7]) + mag[::7]                       # all-positive rows (zp 0)
    x[1::7] = -np.abs(x[1::7])                                # non-positive rows
    x = bf16_round(x.astype(np.float32))
    r = ops.act_quant(torch.from_numpy(x).to(cuda).bfloat16())
    codes, sc, zp, rs = M.quantize_rows(x.astype(np.float64))
    np.testing.assert_array_equal(r["scale"].cpu().numpy(), sc)
    np.testing.assert_array_equal(r["zp"].cpu().numpy(), zp)
    np.testing.assert_array_equal(r["codes"].cpu().numpy(), codes)
