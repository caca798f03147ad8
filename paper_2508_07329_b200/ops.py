"""Tensor-level wrappers over the C ABI (one function per entry point).

Every function takes / returns torch CUDA tensors, allocates outputs and
workspaces with torch (device memory is plumbing), and launches on the
current torch stream. Nothing here computes on the host.
"""

from __future__ import annotations

import torch

from . import _lib as L

_DT = {torch.float32: L.DT_F32, torch.float64: L.DT_F64, torch.bfloat16: L.DT_BF16, torch.float16: L.DT_F16}


def _dt(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise ValueError(f"unsupported dtype {t.dtype}") from None


def _cuda(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.device.index != torch.cuda.current_device():
        # kernels launch on the current device's current stream
        raise ValueError(f"{name} is on {t.device} but the current device is cuda:{torch.cuda.current_device()} "
                         "(wrap the call in torch.cuda.device(...))")
    return t


def _vec(t: torch.Tensor | None, name: str, dtype) -> torch.Tensor | None:
    """Index / table / per-row argument: a dense CUDA tensor of ``dtype``
    (None passes through). The kernels read these as raw arrays, so a wrong
    dtype would be reinterpreted silently: refuse it instead."""
    if t is None:
        return None
    _cuda(t, name)
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    return t.contiguous()


def _rowmajor(t: torch.Tensor, name: str) -> torch.Tensor:
    _cuda(t, name)
    if t.dim() != 2:
        raise ValueError(f"{name} must be 2-D, got shape {tuple(t.shape)}")
    if t.stride(1) != 1:
        t = t.contiguous()
    return t


def _s():
    return L.stream_ptr()


# ── K1 ────────────────────────────────────────────────────────────────────
def reciprocal(s: torch.Tensor, with_f32: bool = False):
    """RN(1/s) in float64 (and its RN32 copy when with_f32)."""
    s = _cuda(s, "s").contiguous().to(torch.float64)
    out = torch.empty_like(s)
    out32 = torch.empty(s.shape, dtype=torch.float32, device=s.device) if with_f32 else None
    L.call("moe_reciprocal_f64", L.ptr(s), s.numel(), L.ptr(out), L.ptr(out32), _s())
    return (out, out32) if with_f32 else out


_ONES: dict = {}


def _ones_table(cols: int, dev) -> tuple:
    key = (cols, str(dev))
    if key not in _ONES:
        one = torch.ones((1, cols), dtype=torch.float64, device=dev)
        _ONES[key] = (one, one.clone(), torch.ones((1, cols), dtype=torch.float32, device=dev))
    return _ONES[key]


def act_quant(x: torch.Tensor, *, smooth: torch.Tensor | None = None, smooth_recip: torch.Tensor | None = None,
              smooth_recip_f32: torch.Tensor | None = None,
              smooth_mode: int = L.SMOOTH_DIVIDE, row_group: torch.Tensor | None = None,
              gather: torch.Tensor | None = None, rows: int | None = None, bits: int = 8,
              symmetric: bool = False, granularity: str = "per_token", rowsum: bool = True,
              out_codes: torch.Tensor | None = None, row_ext: torch.Tensor | None = None) -> dict:
    """K1: codes/scales/zero points of (x[gather] (/ or *) smooth[row_group])."""
    x = _rowmajor(x, "x")
    gather = _vec(gather, "gather", torch.int32)
    row_group = _vec(row_group, "row_group", torch.int32)
    row_ext = _vec(row_ext, "row_ext", torch.int64)
    n_rows = rows if rows is not None else (gather.numel() if gather is not None else x.shape[0])
    cols = x.shape[1]
    gran = L.GRAN[granularity]
    groups = 1 if gran == L.GRAN["per_tensor"] else n_rows
    dev = x.device
    codes = out_codes if out_codes is not None else torch.empty((n_rows, cols), dtype=torch.uint8, device=dev)
    scale = torch.empty(groups, dtype=torch.float64, device=dev)
    scale_f32 = torch.empty(groups, dtype=torch.float32, device=dev)
    zp = torch.empty(groups, dtype=torch.int32, device=dev)
    rs = torch.empty(n_rows, dtype=torch.int32, device=dev) if rowsum else None
    lib = L.load()
    wsb = lib.moe_act_quant_workspace(n_rows, cols, gran)
    ws = torch.empty(max(wsb, 8), dtype=torch.uint8, device=dev) if wsb else None
    if smooth is None and x.dtype == torch.bfloat16 and gran == L.GRAN["per_token"]:
        # unsmoothed bf16 rows: a table of ones keeps them on the fast K1
        # kernels (x / 1 is exact in both the float32 filter and float64)
        smooth, smooth_recip, smooth_recip_f32 = _ones_table(cols, dev)
        smooth_mode = L.SMOOTH_DIVIDE
        row_group = None
    mode = L.SMOOTH_NONE if smooth is None else smooth_mode
    if smooth is not None:
        smooth = _vec(smooth, "smoothing table", torch.float64)
        if smooth_recip is None and mode == L.SMOOTH_DIVIDE:
            smooth_recip, smooth_recip_f32 = reciprocal(smooth, with_f32=True)
        smooth_recip = _vec(smooth_recip, "smooth_recip", torch.float64)
        smooth_recip_f32 = _vec(smooth_recip_f32, "smooth_recip_f32", torch.float32)
    div = mode == L.SMOOTH_DIVIDE
    L.call("moe_act_quant", L.ptr(x), _dt(x), n_rows, cols, x.stride(0), L.ptr(gather), L.ptr(smooth),
           L.ptr(smooth_recip) if div else None, L.ptr(smooth_recip_f32) if div else None, mode,
           L.ptr(row_group), bits,
           int(bool(symmetric)), gran, L.ptr(codes), codes.stride(0), L.ptr(scale), L.ptr(scale_f32), L.ptr(zp),
           L.ptr(rs), L.ptr(row_ext), L.ptr(ws), wsb, _s())
    return {"codes": codes, "scale": scale, "scale_f32": scale_f32, "zp": zp, "rowsum": rs,
            "granularity": granularity, "bits": bits}


def act_quant_tokens_ok(x: torch.Tensor) -> bool:
    """Whether moe_act_quant_tokens takes x (bf16, d % 8 == 0, aligned rows)."""
    return (x.dtype == torch.bfloat16 and x.dim() == 2 and x.stride(1) == 1 and x.shape[1] % 8 == 0
            and x.stride(0) % 8 == 0 and x.data_ptr() % 16 == 0)


def act_quant_tokens(x: torch.Tensor, token_pos: torch.Tensor, row_group: torch.Tensor, *, smooth: torch.Tensor,
                     smooth_recip: torch.Tensor, smooth_recip_f32: torch.Tensor, bits: int = 8,
                     symmetric: bool = False, out_codes: torch.Tensor | None = None) -> dict:
    """Token-major K1 for the MoE dispatch: row token_pos[t, j] = x[t] /
    smooth[row_group[row]], per-token RTN; x is read once per token. Same
    result as act_quant(x, gather=src_token, row_group=row_group, ...)."""
    x = _rowmajor(x, "x")
    token_pos = _vec(token_pos, "token_pos", torch.int32)
    row_group = _vec(row_group, "row_group", torch.int32)
    smooth = _vec(smooth, "smooth", torch.float64)
    smooth_recip = _vec(smooth_recip, "smooth_recip", torch.float64)
    smooth_recip_f32 = _vec(smooth_recip_f32, "smooth_recip_f32", torch.float32)
    T, cols = x.shape
    k = token_pos.numel() // max(T, 1)
    rows = T * k
    dev = x.device
    codes = out_codes if out_codes is not None else torch.empty((rows, cols), dtype=torch.uint8, device=dev)
    scale = torch.empty(rows, dtype=torch.float64, device=dev)
    scale_f32 = torch.empty(rows, dtype=torch.float32, device=dev)
    zp = torch.empty(rows, dtype=torch.int32, device=dev)
    rs = torch.empty(rows, dtype=torch.int32, device=dev)
    L.call("moe_act_quant_tokens", L.ptr(x), _dt(x), T, cols, x.stride(0), k, L.ptr(token_pos),
           L.ptr(row_group), L.ptr(smooth), L.ptr(smooth_recip), L.ptr(smooth_recip_f32), bits, int(bool(symmetric)),
           L.ptr(codes), codes.stride(0), L.ptr(scale), L.ptr(scale_f32), L.ptr(zp), L.ptr(rs), _s())
    return {"codes": codes, "scale": scale, "scale_f32": scale_f32, "zp": zp, "rowsum": rs,
            "granularity": "per_token", "bits": bits}


def dequantize(codes: torch.Tensor, scale: torch.Tensor, zp: torch.Tensor, granularity: str) -> torch.Tensor:
    codes = _rowmajor(codes, "codes")
    out = torch.empty(codes.shape, dtype=torch.float64, device=codes.device)
    L.call("moe_dequantize", L.ptr(codes), codes.shape[0], codes.shape[1], codes.stride(0),
           L.ptr(scale.contiguous()), L.ptr(zp.contiguous()), L.GRAN[granularity], L.ptr(out), _s())
    return out


def apply_smoothing(w: torch.Tensor | None, x: torch.Tensor | None, f: torch.Tensor):
    f = f.contiguous()
    w = w.contiguous() if w is not None else None       # the kernel walks dense row-major matrices
    x = x.contiguous() if x is not None else None
    ws = torch.empty_like(w) if w is not None else None
    xs = torch.empty_like(x) if x is not None else None
    n = f.numel()
    L.call("moe_apply_smoothing", L.ptr(w), w.shape[0] if w is not None else 0, n, L.ptr(x),
           x.shape[1] if x is not None else 0, L.ptr(f), L.ptr(ws), L.ptr(xs), _s())
    return ws, xs


def channel_stats(x: torch.Tensor, strategy: int) -> torch.Tensor:
    x = _rowmajor(x, "x").contiguous()
    out = torch.empty(x.shape[0], dtype=torch.float64, device=x.device)
    L.call("moe_channel_stats", L.ptr(x), x.shape[0], x.shape[1], strategy, L.ptr(out), _s())
    return out


# ── K2 / K5 ───────────────────────────────────────────────────────────────
def w8a8_gemm(a: dict, w: dict, *, epilogue: int = L.EPI_DEQUANT, out_dtype=torch.float32,
              bias: torch.Tensor | None = None, row_weight: torch.Tensor | None = None,
              group_offsets: torch.Tensor | None = None, num_groups: int = 1, n_per_group: int | None = None,
              out: torch.Tensor | None = None, next_smooth_recip_f32: torch.Tensor | None = None,
              row_ext: torch.Tensor | None = None, row_ext_ready: bool = False) -> torch.Tensor:
    """a: dict from act_quant (codes [M, K], scale_f32, zp, rowsum per row).
    w: dict with codes [G*N, K], scale_f32, zp, rowsum per row. With
    ``row_ext_ready`` the records were initialised by the caller
    (step_init) and the call adds no init kernel."""
    ac, wc = a["codes"], w["codes"]
    M, K = ac.shape
    N = n_per_group if n_per_group is not None else wc.shape[0] // num_groups
    group_offsets = _vec(group_offsets, "group_offsets", torch.int32)
    row_weight = _vec(row_weight, "row_weight", torch.float32)
    row_ext = _vec(row_ext, "row_ext", torch.int64)
    if wc.shape[1] != K:
        raise ValueError(f"A has K={K} but W has K={wc.shape[1]}")
    dev = ac.device
    a_scale, a_zp = a.get("scale_f32"), a["zp"]
    if a_zp.numel() == 1 and M > 1:                 # per_tensor activations
        a_zp = a_zp.expand(M).contiguous()
        a_scale = a_scale.expand(M).contiguous() if a_scale is not None else None
    acc = None
    if epilogue == L.EPI_ACC_I32:
        acc = out if out is not None else torch.empty((M, N), dtype=torch.int32, device=dev)
        o = None
        ldo = 0
        odt = L.DT_F32
    else:
        cols = N // 2 if epilogue == L.EPI_SWIGLU else N
        o = out if out is not None else torch.empty((M, cols), dtype=out_dtype, device=dev)
        ldo = o.stride(0)
        odt = L.DT_BF16 if o.dtype == torch.bfloat16 else L.DT_F32
    # weights may carry the pre-corrected sidecar rowsum - K*zp (with_wcorr)
    w_rs, flags = (w["rowsum_corr"], L.EPI_FLAG_WCORR) if "rowsum_corr" in w else (w["rowsum"], 0)
    if row_ext is not None and row_ext_ready:
        flags |= L.EPI_FLAG_EXT_READY
    L.call("moe_w8a8_gemm", L.ptr(ac), M, K, ac.stride(0), L.ptr(a_scale), L.ptr(a_zp), L.ptr(a["rowsum"]),
           L.ptr(wc), N, wc.stride(0), L.ptr(w.get("scale_f32")), L.ptr(w["zp"]), L.ptr(w_rs),
           L.ptr(bias), L.ptr(row_weight), L.ptr(group_offsets), num_groups, epilogue | flags, L.ptr(o), odt, ldo,
           L.ptr(acc), acc.stride(0) if acc is not None else 0,
           L.ptr(next_smooth_recip_f32),
           next_smooth_recip_f32.shape[-1] if next_smooth_recip_f32 is not None else 0, L.ptr(row_ext), _s())
    return acc if epilogue == L.EPI_ACC_I32 else o


def w8a8_gemm_quant_a(x: torch.Tensor, w: dict, *, smooth: torch.Tensor, smooth_recip: torch.Tensor,
                      smooth_recip_f32: torch.Tensor, row_group: torch.Tensor, row_ext: torch.Tensor,
                      group_offsets: torch.Tensor, num_groups: int, n_per_group: int, out_dtype=torch.bfloat16,
                      row_weight: torch.Tensor | None = None, out: torch.Tensor | None = None) -> tuple:
    """The MoE second grouped GEMM with K1 of its A operand fused in
    (moe_w8a8_gemm_quant_a): x [M, K] bf16 rows with producer records ->
    (out, a) where a is act_quant's dict for x. Same results as act_quant
    followed by w8a8_gemm."""
    x = _rowmajor(x, "x")
    M, K = x.shape
    dev = x.device
    codes = torch.empty((M, K), dtype=torch.uint8, device=dev)
    scale = torch.empty(M, dtype=torch.float64, device=dev)
    scale_f32 = torch.empty(M, dtype=torch.float32, device=dev)
    zp = torch.empty(M, dtype=torch.int32, device=dev)
    rs = torch.empty(M, dtype=torch.int32, device=dev)
    N = n_per_group
    o = out if out is not None else torch.empty((M, N), dtype=out_dtype, device=dev)
    wsb = L.load().moe_w8a8_gemm_quant_a_workspace(M)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    wc = w["codes"]
    w_rs, flags = (w["rowsum_corr"], L.EPI_FLAG_WCORR) if "rowsum_corr" in w else (w["rowsum"], 0)
    L.call("moe_w8a8_gemm_quant_a", L.ptr(x), x.stride(0), L.ptr(smooth), L.ptr(smooth_recip),
           L.ptr(smooth_recip_f32), L.ptr(row_group), L.ptr(row_ext), L.ptr(codes), codes.stride(0), L.ptr(scale),
           L.ptr(scale_f32), L.ptr(zp), L.ptr(rs), M, K, L.ptr(wc), N, wc.stride(0), L.ptr(w.get("scale_f32")),
           L.ptr(w["zp"]), L.ptr(w_rs), None, L.ptr(row_weight), L.ptr(group_offsets), num_groups,
           L.EPI_DEQUANT | flags, L.ptr(o), L.DT_BF16 if o.dtype == torch.bfloat16 else L.DT_F32, o.stride(0),
           L.ptr(ws), wsb, _s())
    a = {"codes": codes, "scale": scale, "scale_f32": scale_f32, "zp": zp, "rowsum": rs,
         "granularity": "per_token", "bits": 8}
    return o, a


def step_init(T: int, N: int, rows: int, device, combine: bool, records: bool) -> tuple:
    """(combine workspace zeroed | None, [rows, 2] extreme records initialised |
    None), both prepared by one moe_step_init launch."""
    wsb = L.load().moe_w8a8_gemm_combine_workspace(T, N) if combine else 0
    wsb16 = (wsb + 15) // 16 * 16
    ws = torch.empty(max(wsb16, 16), dtype=torch.uint8, device=device) if combine else None
    ext = torch.empty((rows, 2), dtype=torch.int64, device=device) if records else None
    if combine or records:
        L.call("moe_step_init", L.ptr(ws), wsb16, L.ptr(ext), rows if records else 0, _s())
    return ws, ext


def combine_workspace(T: int, N: int, device) -> torch.Tensor:
    """Zeroed workspace for w8a8_gemm_combine (allocate it before the kernel
    that precedes the GEMM so no memset sits between them)."""
    return torch.zeros(L.load().moe_w8a8_gemm_combine_workspace(T, N), dtype=torch.uint8, device=device)


def w8a8_gemm_combine(a: dict, w: dict, *, row_weight: torch.Tensor, group_offsets: torch.Tensor, num_groups: int,
                      n_per_group: int, src_token: torch.Tensor, token_pos: torch.Tensor, T: int,
                      out: torch.Tensor | None = None, workspace: torch.Tensor | None = None) -> torch.Tensor:
    """The MoE second grouped GEMM with the top-2 combine fused in
    (moe_w8a8_gemm_combine): returns out [T, N] bf16, equal to
    combine(w8a8_gemm(a, w, bf16), token_pos, T, 2)."""
    ac, wc = a["codes"], w["codes"]
    M, K = ac.shape
    N = n_per_group
    dev = ac.device
    src_token = _vec(src_token, "src_token", torch.int32)
    token_pos = _vec(token_pos, "token_pos", torch.int32)
    row_weight = _vec(row_weight, "row_weight", torch.float32)
    group_offsets = _vec(group_offsets, "group_offsets", torch.int32)
    y = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
    o = out if out is not None else torch.empty((T, N), dtype=torch.bfloat16, device=dev)
    wsb = L.load().moe_w8a8_gemm_combine_workspace(T, N)
    w_rs, flags = (w["rowsum_corr"], L.EPI_FLAG_WCORR) if "rowsum_corr" in w else (w["rowsum"], 0)
    if workspace is not None:           # pre-zeroed by the caller
        ws = workspace
        flags |= L.EPI_FLAG_WS_ZEROED
    else:
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    L.call("moe_w8a8_gemm_combine", L.ptr(ac), M, K, ac.stride(0), L.ptr(a["scale_f32"]), L.ptr(a["zp"]),
           L.ptr(a["rowsum"]), L.ptr(wc), N, wc.stride(0), L.ptr(w.get("scale_f32")), L.ptr(w["zp"]), L.ptr(w_rs),
           L.ptr(row_weight), L.ptr(group_offsets), num_groups, L.EPI_DEQUANT | flags, L.ptr(y), y.stride(0),
           L.ptr(src_token), L.ptr(token_pos), T, L.ptr(o), o.stride(0), L.ptr(ws), wsb, _s())
    return o


def rmsnorm_residual(x: torch.Tensor, y: torch.Tensor | None = None, eps: float = 1e-5,
                     want_sum: bool = True, want_norm: bool = True) -> tuple:
    """(s, norm): s = bf16(x + y) (x when y is None), norm = RMSNorm(s) without
    gain, one fused pass (moe_rmsnorm_residual). bf16 [T, d] rows."""
    x = x.contiguous()
    T, d = x.shape
    s_out = torch.empty_like(x) if (y is not None and want_sum) else None
    n_out = torch.empty_like(x) if want_norm else None
    if T:
        L.call("moe_rmsnorm_residual", L.ptr(x), L.ptr(y.contiguous()) if y is not None else None, L.ptr(s_out),
               L.ptr(n_out), T, d, eps, _s())
    return (s_out if y is not None else x), n_out


def with_wcorr(w: dict) -> dict:
    """Add the pre-corrected weight sidecar rowsum - K * zp (int32, wrapping)
    used by the GEMM epilogue instead of rowsum (MOE_EPI_FLAG_WCORR)."""
    K = w["codes"].shape[1]
    corr = (w["rowsum"].to(torch.int64) - K * w["zp"].to(torch.int64)).to(torch.int32)
    return {**w, "rowsum_corr": corr.contiguous()}


def quant_sq_error(acc: torch.Tensor, a_scale: torch.Tensor, w_scale: torch.Tensor, ref: torch.Tensor) -> torch.Tensor:
    acc = acc.contiguous()
    M, N = acc.shape
    lib = L.load()
    wsb = lib.moe_quant_sq_error_workspace(M, N)
    ws = torch.empty(wsb, dtype=torch.uint8, device=acc.device)
    out = torch.empty(1, dtype=torch.float64, device=acc.device)
    stride = 0 if a_scale.numel() == 1 else 1
    L.call("moe_quant_sq_error", L.ptr(acc), M, N, L.ptr(a_scale.contiguous()), stride, L.ptr(w_scale.contiguous()),
           L.ptr(ref.contiguous()), L.ptr(out), L.ptr(ws), wsb, _s())
    return out


# ── K3 / K4 / K6 ──────────────────────────────────────────────────────────
def router_pieces(gate_w: torch.Tensor) -> torch.Tensor:
    """bf16 (hi, mid, lo) split of a float32 gate for the tensor-core router
    (moe_router_prepare), cached ON the gate tensor (valid while its version
    counter is unchanged; freed with it)."""
    cached = getattr(gate_w, "_moe_router_pieces", None)
    if cached is not None and cached[0] == gate_w._version:
        return cached[1]
    E, d = gate_w.shape
    lib = L.load()
    pc = torch.empty(lib.moe_router_tc_workspace(d) // 2, dtype=torch.bfloat16, device=gate_w.device)
    L.call("moe_router_prepare", L.ptr(gate_w.contiguous()), E, d, L.ptr(pc), _s())
    gate_w._moe_router_pieces = (gate_w._version, pc)
    return pc


def router_gate(x: torch.Tensor, gate_w: torch.Tensor, k: int, want_logits: bool = True,
                gate_bias: torch.Tensor | None = None, tensor_cores: bool | None = None):
    """K3: logits = x Wg^T (+ bias), top-k (ties -> lower id), softmax over the
    selected. bf16 x with d % 64 == 0 and E <= 16 runs on the tensor cores
    (exact 3-piece bf16 split of the float32 gate); else the SIMT kernels."""
    x = _rowmajor(x, "x")
    T, d = x.shape
    E = gate_w.shape[0]
    gw = gate_w.contiguous().to(torch.float32)
    logits = torch.empty((T, E), dtype=torch.float32, device=x.device) if want_logits else None
    idx = torch.empty((T, k), dtype=torch.int32, device=x.device)
    w = torch.empty((T, k), dtype=torch.float32, device=x.device)
    gb = gate_bias.contiguous().to(torch.float32) if gate_bias is not None else None
    if tensor_cores is None:
        tensor_cores = (x.dtype == torch.bfloat16 and d % 64 == 0 and E <= 16 and k <= 8
                        and (x.stride(0) * 2) % 16 == 0 and x.data_ptr() % 16 == 0)
    if tensor_cores:
        L.call("moe_router_gate_tc", L.ptr(x), T, d, x.stride(0), L.ptr(router_pieces(gw)), L.ptr(gb), E, k,
               L.ptr(logits), L.ptr(idx), L.ptr(w), _s())
    else:
        L.call("moe_router_gate", L.ptr(x), _dt(x), T, d, x.stride(0), L.ptr(gw), L.ptr(gb), E, k, L.ptr(logits), L.ptr(idx),
               L.ptr(w), _s())
    return logits, idx, w


def router_topk(logits: torch.Tensor, k: int):
    logits = logits.contiguous().to(torch.float32)
    T, E = logits.shape
    idx = torch.empty((T, k), dtype=torch.int32, device=logits.device)
    w = torch.empty((T, k), dtype=torch.float32, device=logits.device)
    L.call("moe_router_topk", L.ptr(logits), T, E, k, L.ptr(idx), L.ptr(w), _s())
    return idx, w


def route_permute(idx: torch.Tensor, w: torch.Tensor | None, E: int) -> dict:
    idx = _vec(idx, "idx", torch.int32)
    w = _vec(w, "w", torch.float32)
    T, k = idx.shape
    dev = idx.device
    n = T * k
    lib = L.load()
    wsb = lib.moe_route_permute_workspace(T, k, E)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    out = {
        "offsets": torch.empty(E + 1, dtype=torch.int32, device=dev),
        "src_token": torch.empty(n, dtype=torch.int32, device=dev),
        "row_expert": torch.empty(n, dtype=torch.int32, device=dev),
        "row_weight": torch.empty(n, dtype=torch.float32, device=dev) if w is not None else None,
        "token_pos": torch.empty(n, dtype=torch.int32, device=dev),
    }
    L.call("moe_route_permute", L.ptr(idx), L.ptr(w.contiguous() if w is not None else None), T, k, E,
           L.ptr(out["offsets"]), L.ptr(out["src_token"]), L.ptr(out["row_expert"]), L.ptr(out["row_weight"]),
           L.ptr(out["token_pos"]), L.ptr(ws), wsb, _s())
    return out


def combine(y: torch.Tensor, token_pos: torch.Tensor, T: int, k: int, out_dtype=torch.bfloat16,
            out: torch.Tensor | None = None) -> torch.Tensor:
    y = _rowmajor(y, "y").contiguous()                  # y rows are read as dense [T*k, d]
    token_pos = _vec(token_pos, "token_pos", torch.int32)
    d = y.shape[1]
    o = out if out is not None else torch.empty((T, d), dtype=out_dtype, device=y.device)
    if o.shape != (T, d) or o.stride(1) != 1:
        raise ValueError(f"combine: out must be [{T}, {d}] with unit column stride")
    L.call("moe_combine", L.ptr(y), _dt(y), L.ptr(token_pos), T, k, d, L.ptr(o), _dt(o), o.stride(0), _s())
    return o


def expert_histogram(idx: torch.Tensor, E: int, layer: int, counts: torch.Tensor,
                     path_codes: torch.Tensor | None = None) -> None:
    T, k = idx.shape
    idx = _vec(idx, "idx", torch.int32)
    if counts.dtype != torch.int64 or not counts.is_contiguous():
        raise ValueError("counts must be a dense int64 tensor")
    L.call("moe_expert_histogram", L.ptr(idx), T, k, E, layer, L.ptr(counts), L.ptr(path_codes), _s())


# ── K7 / K8 ───────────────────────────────────────────────────────────────
def hessian(x_tokens: torch.Tensor, smooth: torch.Tensor | None = None, damping_fraction: float = 0.01,
            H: torch.Tensor | None = None, finalize: bool = True, nonzero: torch.Tensor | None = None):
    """H = 2 xs^T xs (+ damping) from tokens-major x [T, n]."""
    x = _rowmajor(x_tokens, "x")
    T, n = x.shape
    if H is None:
        H = torch.zeros((n, n), dtype=torch.float64, device=x.device)
    if nonzero is None:
        nonzero = torch.zeros(1, dtype=torch.int64, device=x.device)
    srec = reciprocal(smooth) if smooth is not None else None
    L.call("moe_hessian_accum", L.ptr(x), _dt(x), T, n, x.stride(0), L.ptr(smooth), L.ptr(srec), L.ptr(H),
           L.ptr(nonzero), _s())
    if finalize:
        L.call("moe_hessian_finalize", L.ptr(H), n, float(damping_fraction), L.ptr(nonzero), _s())
    return H


def gptq_columns(w: torch.Tensor, U: torch.Tensor, scale: torch.Tensor, zp: torch.Tensor, bits: int,
                 order: torch.Tensor | None = None) -> torch.Tensor:
    w = _rowmajor(w, "w")
    R, n = w.shape
    codes = torch.empty((R, n), dtype=torch.uint8, device=w.device)
    lib = L.load()
    wsb = lib.moe_gptq_workspace(R, n)
    ws = torch.empty(wsb, dtype=torch.uint8, device=w.device)
    o32 = order.to(torch.int32).contiguous() if order is not None else None
    L.call("moe_gptq_columns", L.ptr(w), R, n, w.stride(0), L.ptr(o32), L.ptr(U.contiguous()),
           L.ptr(scale.contiguous()), L.ptr(zp.contiguous()), bits, L.ptr(codes), codes.stride(0), L.ptr(ws), wsb,
           _s())
    return codes


# ── expert-parallel plumbing ──────────────────────────────────────────────
def route_keys(idx: torch.Tensor, dest_rank: torch.Tensor, E: int) -> torch.Tensor:
    """keys = dest_rank[idx] * E + idx (sort keys grouping rows by destination rank, then expert)."""
    idx = idx.contiguous()
    keys = torch.empty_like(idx)
    L.call("moe_route_keys", L.ptr(idx), idx.numel(), L.ptr(dest_rank.contiguous()), E, L.ptr(keys), _s())
    return keys


def gather_rows(src: torch.Tensor, index: torch.Tensor | None, out: torch.Tensor | None = None) -> torch.Tensor:
    """out[r] = src[index[r]] for a row-major 2-D tensor (any dtype)."""
    src = _rowmajor(src, "src")
    index = _vec(index, "index", torch.int32)
    n = index.numel() if index is not None else src.shape[0]
    o = out if out is not None else torch.empty((n,) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
    row_bytes = src[0].numel() * src.element_size() if src.shape[0] else o[0].numel() * o.element_size()
    L.call("moe_gather_rows", L.ptr(src), src.stride(0) * src.element_size(),
           L.ptr(index), n, row_bytes, L.ptr(o),
           o.stride(0) * o.element_size(), _s())
    return o


def ep_pack_params(a: dict, weight: torch.Tensor | None) -> torch.Tensor:
    """[n, 4] int32 sidecar of dispatched rows: (scale_f32 bits, zp, rowsum, weight bits)."""
    n = a["codes"].shape[0]
    params = torch.empty((n, 4), dtype=torch.int32, device=a["codes"].device)
    L.call("moe_ep_pack_params", L.ptr(a["scale_f32"]), L.ptr(a["zp"]), L.ptr(a["rowsum"]), L.ptr(weight), n,
           L.ptr(params), _s())
    return params


def ep_unpack_params(params: torch.Tensor, index: torch.Tensor | None, n: int | None = None,
                     n_dev: torch.Tensor | None = None) -> dict:
    """SoA (scale_f32, zp, rowsum, weight) of params[index[r]] (or params[r]),
    r < n; with ``n_dev`` (device int32) only r < min(n, n_dev[0])."""
    if n is None:
        n = index.numel() if index is not None else params.shape[0]
    dev = params.device
    out = {"scale_f32": torch.empty(n, dtype=torch.float32, device=dev),
           "zp": torch.empty(n, dtype=torch.int32, device=dev),
           "rowsum": torch.empty(n, dtype=torch.int32, device=dev),
           "weight": torch.empty(n, dtype=torch.float32, device=dev)}
    L.call("moe_ep_unpack_params", L.ptr(params.contiguous()), L.ptr(index), n, L.ptr(n_dev), L.ptr(out["scale_f32"]),
           L.ptr(out["zp"]), L.ptr(out["rowsum"]), L.ptr(out["weight"]), _s())
    return out


# ── fused expert-parallel transport (peer memory) ──────────────────────────
def block_map(n: int, block_start: torch.Tensor, val0: torch.Tensor, val1: torch.Tensor,
              val2: torch.Tensor | None = None, valid: torch.Tensor | None = None,
              n_dev: torch.Tensor | None = None, nblocks: int | None = None):
    """Rows in blocks [start[b], start[b+1]) -> (val0[b], val1[b] + i - start[b]
    [, val2[b]]) for i < n (i < min(n, n_dev[0]) with a device count);
    ``valid`` (device int32, optional): 0 makes every val0 output -1."""
    dev = block_start.device
    o0 = torch.empty(n, dtype=torch.int32, device=dev)
    o1 = torch.empty(n, dtype=torch.int32, device=dev)
    o2 = torch.empty(n, dtype=torch.int32, device=dev) if val2 is not None else None
    L.call("moe_block_map", n, L.ptr(n_dev), nblocks if nblocks is not None else val0.numel(),
           L.ptr(block_start.contiguous()), L.ptr(val0.contiguous()), L.ptr(val1.contiguous()),
           L.ptr(val2), L.ptr(valid), L.ptr(o0), L.ptr(o1), L.ptr(o2), _s())
    return (o0, o1) if o2 is None else (o0, o1, o2)


def ep_peer_plan(offsets_all: torch.Tensor, me: int, local: torch.Tensor, cap: int, cap_home: int,
                 out: torch.Tensor | None = None, host_flag: torch.Tensor | None = None) -> torch.Tensor:
    """Device-side exchange plan of a peer-memory EP forward (moe_ep_peer_plan):
    offsets_all [W, W*E+1] int32 (every rank's route_permute offsets over
    its W*E keys) -> int32 plan [valid, R, send_base[W*E], starts[G*W+1],
    ranks[G*W], homes[G*W], group[G*W], goff[G+1]]; ``host_flag`` (pinned
    int32, optional) receives valid from the kernel."""
    W = offsets_all.shape[0]
    E = (offsets_all.shape[1] - 1) // W
    G = local.numel()
    size = L.load().moe_ep_peer_plan_size(W, E, G)
    plan = out if out is not None else torch.empty(size, dtype=torch.int32, device=offsets_all.device)
    L.call("moe_ep_peer_plan", L.ptr(offsets_all.contiguous()), W, E, me, L.ptr(local), G, cap, cap_home,
           L.ptr(plan), host_flag.data_ptr() if host_flag is not None else None, _s())
    return plan


def plan_views(plan: torch.Tensor, W: int, E: int, G: int) -> dict:
    """Named slices of an ep_peer_plan buffer (device views, no copies)."""
    o = 2
    views = {"valid": plan[0:1], "R": plan[1:2]}
    for name, n in (("send_base", W * E), ("starts", G * W + 1), ("ranks", G * W), ("homes", G * W),
                    ("group", G * W), ("goff", G + 1)):
        views[name] = plan[o:o + n]
        o += n
    return views


def act_quant_dispatch(x: torch.Tensor, gather: torch.Tensor | None, row_group: torch.Tensor, *, smooth, smooth_recip,
                       smooth_recip_f32, codes_tab: torch.Tensor, params_tab: torch.Tensor, dst_rank: torch.Tensor,
                       dst_row: torch.Tensor, row_weight: torch.Tensor | None, ldc: int, bits: int = 8,
                       symmetric: bool = False, token_pos: torch.Tensor | None = None, k: int = 1) -> None:
    """K1 whose rows land directly in the destination ranks' receive buffers:
    token-major (x read once per token) when ``token_pos`` is given, else
    one warp per gathered row."""
    x = _rowmajor(x, "x")
    n = token_pos.numel() if token_pos is not None else gather.numel()
    L.call("moe_act_quant_dispatch", L.ptr(x), _dt(x), n, x.shape[1], x.stride(0),
           L.ptr(gather.contiguous() if gather is not None else None),
           L.ptr(token_pos.contiguous() if token_pos is not None else None), k,
           L.ptr(smooth), L.ptr(smooth_recip), L.ptr(smooth_recip_f32), L.ptr(row_group.contiguous()), bits,
           int(bool(symmetric)), L.ptr(codes_tab), L.ptr(params_tab), L.ptr(dst_rank), L.ptr(dst_row),
           L.ptr(row_weight), ldc, _s())


def act_quant_given_dev(h: torch.Tensor, rows_dev: torch.Tensor, row_group: torch.Tensor, row_ext: torch.Tensor, *,
                        smooth, smooth_recip, smooth_recip_f32, bits: int = 8, symmetric: bool = False) -> dict:
    """K1 with producer records over rows r < rows_dev[0] of h (capacity
    h.shape[0] rows; the count stays on the device)."""
    h = _rowmajor(h, "h")
    n, cols = h.shape
    dev = h.device
    out = {"codes": torch.empty((n, cols), dtype=torch.uint8, device=dev),
           "scale": torch.empty(n, dtype=torch.float64, device=dev),
           "scale_f32": torch.empty(n, dtype=torch.float32, device=dev),
           "zp": torch.empty(n, dtype=torch.int32, device=dev),
           "rowsum": torch.empty(n, dtype=torch.int32, device=dev),
           "granularity": "per_token", "bits": bits}
    L.call("moe_act_quant_given_dev", L.ptr(h), _dt(h), n, L.ptr(rows_dev), cols, h.stride(0), L.ptr(smooth),
           L.ptr(smooth_recip), L.ptr(smooth_recip_f32), L.ptr(row_group), bits, int(bool(symmetric)),
           L.ptr(out["codes"]), out["codes"].stride(0), L.ptr(out["scale"]), L.ptr(out["scale_f32"]),
           L.ptr(out["zp"]), L.ptr(out["rowsum"]), L.ptr(row_ext), _s())
    return out


def w8a8_gemm_scatter(a: dict, w: dict, *, out_tab: torch.Tensor, out_rank: torch.Tensor, out_row: torch.Tensor,
                      ldo: int, out_dtype=torch.bfloat16, row_weight: torch.Tensor | None = None,
                      group_offsets: torch.Tensor | None = None, num_groups: int = 1,
                      n_per_group: int | None = None) -> None:
    """DEQUANT grouped GEMM whose output rows go to out_tab[out_rank[m]] + out_row[m] * ldo."""
    ac, wc = a["codes"], w["codes"]
    M, K = ac.shape
    N = n_per_group if n_per_group is not None else wc.shape[0] // num_groups
    w_rs, flags = (w["rowsum_corr"], L.EPI_FLAG_WCORR) if "rowsum_corr" in w else (w["rowsum"], 0)
    L.call("moe_w8a8_gemm_scatter", L.ptr(ac), M, K, ac.stride(0), L.ptr(a["scale_f32"]), L.ptr(a["zp"]),
           L.ptr(a["rowsum"]), L.ptr(wc), N, wc.stride(0), L.ptr(w["scale_f32"]), L.ptr(w["zp"]), L.ptr(w_rs), None,
           L.ptr(row_weight), L.ptr(group_offsets), num_groups, L.EPI_DEQUANT | flags, L.ptr(out_tab),
           L.ptr(out_rank), L.ptr(out_row), L.DT_BF16 if out_dtype == torch.bfloat16 else L.DT_F32, ldo, _s())


# ── attention block glue (C5 token path) ───────────────────────────────────
def rope_tables(max_pos: int, head_dim: int, theta: float = 1e6, device="cuda"):
    """float32 cos / sin tables [max_pos, head_dim/2] of position *
    theta^(-2i/head_dim), computed in float64."""
    i = torch.arange(head_dim // 2, dtype=torch.float64, device=device)
    inv = theta ** (-2.0 * i / head_dim)
    ang = torch.arange(max_pos, dtype=torch.float64, device=device)[:, None] * inv[None, :]
    return torch.cos(ang).float().contiguous(), torch.sin(ang).float().contiguous()


def rope_(x: torch.Tensor, heads: int, head_dim: int, cos_tab: torch.Tensor, sin_tab: torch.Tensor,
          positions: torch.Tensor | None = None) -> torch.Tensor:
    """In place: rotary embedding of the first heads * head_dim columns of the
    bf16 rows of x (moe_rope_bf16)."""
    if x.dtype != torch.bfloat16 or x.stride(1) != 1:
        raise ValueError("rope_: bf16 rows with unit column stride")
    L.call("moe_rope_bf16", L.ptr(x), x.shape[0], heads, head_dim, x.stride(0), L.ptr(positions), L.ptr(cos_tab),
           L.ptr(sin_tab), _s())
    return x
