"""MoELayer: the W8A8 Mixture-of-Experts forward on the B200.

The reference quantizes expert weights (HAQ, quant.py) but never runs a MoE
forward; this module is the forward path the north star asks for, built on
the same quantizer semantics:

  x [T, d] bf16
   -> K3 router_gate: logits = x Wg^T, top-k (ties -> lower id), softmax
   -> K4 route_permute: stable counting sort of (token, slot) by expert
   -> K1 act_quant (gather + per-expert smoothing x / s13_e, per-token RTN)
   -> K5 grouped W8A8 GEMM, W1||W3 interleaved, SwiGLU epilogue -> h bf16
   -> K1 act_quant (h / s2_e, per-token RTN)
   -> K5 grouped W8A8 GEMM with W2, dequant * routing weight -> y
   -> K6 combine: out[t] = sum_j y[pos(t, j)]

All routing state stays on the device (expert offsets feed the persistent
GEMM scheduler directly), so one forward is 8 kernel launches and no host
synchronisation.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from . import ops
from .quant import PER_OUTPUT_ROW, QuantizedMatrix

INTERLEAVE = 128   # W1/W3 row-block interleave consumed by the SwiGLU epilogue


def _stack_dev(qms: list[QuantizedMatrix]) -> dict:
    parts = [q.device() for q in qms]
    out = {k: torch.cat([p[k] for p in parts], dim=0).contiguous() for k in ("codes", "scale", "scale_f32", "zp",
                                                                             "rowsum")}
    return out


def _interleave_rows(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """[F, ...] x2 -> [2F, ...] as blocks (a[0:128], b[0:128], a[128:256], ...)."""
    F = a.shape[0]
    rest = a.shape[1:]
    ai = a.reshape(F // INTERLEAVE, INTERLEAVE, *rest)
    bi = b.reshape(F // INTERLEAVE, INTERLEAVE, *rest)
    return torch.stack([ai, bi], dim=1).reshape(2 * F, *rest).contiguous()


class MoELayer:
    def __init__(self, gate_weight, experts: list[dict], top_k: int = 2, out_dtype=torch.bfloat16,
                 gate_bias=None):
        """experts[e] = {"w1": QM [F, d], "w3": QM [F, d], "w2": QM [d, F],
        "s13": [d] smoothing of the shared W1/W3 input, "s2": [F]}."""
        self.E = len(experts)
        if not 1 <= top_k <= self.E:
            raise ValueError("top_k must be within [1, num_experts]")
        self.k = top_k
        self.gate_w = torch.as_tensor(gate_weight, dtype=torch.float32).cuda().contiguous()
        self.gate_b = None if gate_bias is None else torch.as_tensor(gate_bias, dtype=torch.float32).cuda()
        F, d = experts[0]["w1"].codes.shape
        if F % INTERLEAVE:
            raise ValueError(f"ffn dim must be a multiple of {INTERLEAVE}")
        self.d, self.F = d, F
        w13 = []
        for e in experts:
            for q in (e["w1"], e["w3"], e["w2"]):
                if q.granularity != PER_OUTPUT_ROW:
                    raise ValueError("expert weights must be quantized per output row")
            a, b = e["w1"].device(), e["w3"].device()
            w13.append({k: _interleave_rows(a[k], b[k]) for k in ("codes", "scale", "scale_f32", "zp", "rowsum")})
        self.w13 = ops.with_wcorr({k: torch.cat([p[k] for p in w13], 0).contiguous() for k in w13[0]})
        self.w2 = ops.with_wcorr(_stack_dev([e["w2"] for e in experts]))
        self.s13 = torch.stack([torch.as_tensor(np.asarray(_np(e["s13"])), dtype=torch.float64)
                                for e in experts]).cuda().contiguous()
        self.s2 = torch.stack([torch.as_tensor(np.asarray(_np(e["s2"])), dtype=torch.float64)
                               for e in experts]).cuda().contiguous()
        self.s13_recip, self.s13_recip32 = ops.reciprocal(self.s13, with_f32=True)
        self.s2_recip, self.s2_recip32 = ops.reciprocal(self.s2, with_f32=True)
        self.out_dtype = out_dtype
        self.host_experts = experts

    # ------------------------------------------------------------------
    @classmethod
    def random(cls, E: int, d: int, F: int, top_k: int = 2, seed: int = 1, out_dtype=torch.bfloat16,
               router_seed: int = 2, zipf_s: float = 1.2, smooth_exponent: float = 0.5):
        """Synthetic random-init layer of the given shape (the bench's Mixtral
        8x7B-shape layer): W ~ N(0, 0.02^2), smoothing factors from a
        synthetic outlier-channel statistic (1% of channels x100), W s
        quantized per output row on device; router weights N(0, 1/d) plus a
        Zipf(s) logit bias over a seeded expert shuffle."""
        g = torch.Generator(device="cuda").manual_seed(seed)
        rng = np.random.default_rng(seed)

        def stat(n):
            s = np.abs(rng.normal(size=n)) + 1.0
            s[rng.choice(n, max(1, n // 100), replace=False)] *= 100.0
            return s ** smooth_exponent

        experts = []
        for _ in range(E):
            s13, s2 = stat(d), stat(F)
            ex = {"s13": s13, "s2": s2}
            for name, shape, s in (("w1", (F, d), s13), ("w3", (F, d), s13), ("w2", (d, F), s2)):
                w = torch.randn(shape, generator=g, device="cuda", dtype=torch.float32) * 0.02
                sm = torch.as_tensor(s, dtype=torch.float64).reshape(1, -1).cuda()
                q = ops.act_quant(w, smooth=sm, smooth_mode=L.SMOOTH_MULTIPLY, granularity=PER_OUTPUT_ROW,
                                  rowsum=False)
                ex[name] = QuantizedMatrix(q["codes"], q["scale"], q["zp"], 8, PER_OUTPUT_ROW)
                del w
            experts.append(ex)
        rr = np.random.default_rng(router_seed)
        gw = rr.normal(size=(E, d)) / np.sqrt(d)
        bias = np.log(1.0 / (np.arange(E) + 1.0) ** zipf_s)
        bias = bias - np.log(np.exp(bias).sum())
        gb = bias[np.argsort(rr.permutation(E))]          # rank r -> expert shuffle[r]
        return cls(gw.astype(np.float32), experts, top_k, out_dtype, gate_bias=gb.astype(np.float32))

    # ------------------------------------------------------------------
    def route(self, x: torch.Tensor, want_logits: bool = False):
        logits, idx, w = ops.router_gate(x, self.gate_w, self.k, want_logits=want_logits, gate_bias=self.gate_b)
        return logits, idx, w

    def forward(self, x: torch.Tensor, out_dtype=None, y_dtype=None, return_aux: bool = False, stats=None,
                timer=None, out: torch.Tensor | None = None, h_dtype=torch.bfloat16):
        """x [T, d] (bf16) on device -> [T, d]. ``timer`` (optional) gets a
        ``mark(stage)`` call after every kernel stage (CUDA events).

        ``h_dtype=torch.float32`` is the precise mode: the SwiGLU output h is
        stored in float32 (not bf16) before K1 re-quantizes it, so h's codes
        follow the float64 oracle's except where float32 SwiGLU arithmetic
        lands within ~1e-6 of a rounding boundary (measured flip rate in
        DESIGN.md); K1 on h then takes the exact kernel and GEMM2 / combine
        run in float32. The default bf16 h is the serving path."""
        if x.dim() != 2 or x.shape[1] != self.d:
            raise ValueError(f"expected input [T, {self.d}], got {tuple(x.shape)}")
        out_dtype = out_dtype or self.out_dtype
        y_dtype = y_dtype or (torch.float32 if out_dtype == torch.float32 else torch.bfloat16)
        mark = timer.mark if timer is not None else (lambda _n: None)
        T = x.shape[0]
        if T == 0:
            empty = out if out is not None else torch.empty((0, self.d), dtype=out_dtype, device=x.device)
            return (empty, {}) if return_aux else empty
        mark("start")
        fused_combine = (self.k == 2 and not return_aux and y_dtype == torch.bfloat16
                         and out_dtype == torch.bfloat16 and self.d % 32 == 0 and self.F % 16 == 0
                         and T * self.k > L.tune(L.TUNE_K1_SMALL_ROWS) and L.tune(L.TUNE_FUSED_COMBINE) > 0
                         and h_dtype == torch.bfloat16)
        # the fused combine's counters, zeroed first so no memset sits between
        # the PDL-chained kernels of the layer
        # ... and the SwiGLU epilogue's extreme records, both in one launch
        precise = h_dtype == torch.float32
        fuse = (not precise and self.d % 16 == 0 and self.d >= 128 and T * self.k > L.tune(L.TUNE_K1_SMALL_ROWS))
        cws, ext = ops.step_init(T, self.d, T * self.k, x.device,
                                 combine=fused_combine and L.tune(L.TUNE_FUSED_QUANT) == 0, records=fuse)
        logits, idx, w = self.route(x, want_logits=return_aux)
        mark("router")
        if stats is not None:
            stats.record(idx)
        perm = ops.route_permute(idx, w, self.E)
        mark("permute")
        if ops.act_quant_tokens_ok(x) and L.tune(L.TUNE_K1_TOKENS) > 0 and T * self.k > L.tune(L.TUNE_K1_SMALL_ROWS):
            # token-major K1: each token's x row read once for its k expert rows
            a1 = ops.act_quant_tokens(x, perm["token_pos"], perm["row_expert"], smooth=self.s13,
                                      smooth_recip=self.s13_recip, smooth_recip_f32=self.s13_recip32)
        else:
            a1 = ops.act_quant(x, smooth=self.s13, smooth_recip=self.s13_recip, smooth_recip_f32=self.s13_recip32,
                               row_group=perm["row_expert"], gather=perm["src_token"], rows=T * self.k)
        mark("quant_x")
        # the SwiGLU epilogue also emits each h row's (value, column) records
        # of the float32 min/max of h * RN32(1/s2), so the second K1 streams h once
        # (decode-size batches go through K1's CTA-per-row kernel, whose own
        # extreme pass is cheaper than initialising and filling the records)
        if not precise and h_dtype != torch.bfloat16:
            raise ValueError("h_dtype must be torch.bfloat16 or torch.float32")
        if precise and y_dtype != torch.float32:
            y_dtype = torch.float32
        h = ops.w8a8_gemm(a1, self.w13, epilogue=L.EPI_SWIGLU, out_dtype=h_dtype,
                          group_offsets=perm["offsets"], num_groups=self.E, n_per_group=2 * self.F,
                          next_smooth_recip_f32=self.s2_recip32 if fuse else None, row_ext=ext,
                          row_ext_ready=True)
        mark("gemm13_swiglu")
        if fuse and self.F % 8 == 0 and L.tune(L.TUNE_FUSED_QUANT) > 0 and y_dtype == torch.bfloat16:
            # K1 of h runs inside the second grouped GEMM (its epilogue warps
            # quantize rows while the tensor cores work; bit-identical)
            mark("quant_h")
            y, a2 = ops.w8a8_gemm_quant_a(h, self.w2, smooth=self.s2, smooth_recip=self.s2_recip,
                                          smooth_recip_f32=self.s2_recip32, row_group=perm["row_expert"],
                                          row_ext=ext, group_offsets=perm["offsets"], num_groups=self.E,
                                          n_per_group=self.d, out_dtype=y_dtype, row_weight=perm["row_weight"])
            mark("gemm2")
        else:
            # (decode-size batches keep the separate combine: the per-chunk
            # hand-off costs more than the 4 us kernel at a few dozen rows)
            if fused_combine and cws is None:
                cws = ops.combine_workspace(T, self.d, x.device)
            a2 = ops.act_quant(h, smooth=self.s2, smooth_recip=self.s2_recip, smooth_recip_f32=self.s2_recip32,
                               row_group=perm["row_expert"], row_ext=ext)
            mark("quant_h")
            if fused_combine:
                # the top-2 combine fused into GEMM2's epilogue (bit-identical)
                out = ops.w8a8_gemm_combine(a2, self.w2, row_weight=perm["row_weight"], group_offsets=perm["offsets"],
                                            num_groups=self.E, n_per_group=self.d, src_token=perm["src_token"],
                                            token_pos=perm["token_pos"], T=T, out=out, workspace=cws)
                mark("gemm2")
                mark("combine")
                return out
            y = ops.w8a8_gemm(a2, self.w2, epilogue=L.EPI_DEQUANT, out_dtype=y_dtype, row_weight=perm["row_weight"],
                              group_offsets=perm["offsets"], num_groups=self.E, n_per_group=self.d)
            mark("gemm2")
        out = ops.combine(y, perm["token_pos"], T, self.k, out_dtype=out_dtype, out=out)
        mark("combine")
        if return_aux:
            return out, {"logits": logits, "idx": idx, "w": w, "perm": perm, "a1": a1, "h": h, "a2": a2, "y": y}
        return out

    __call__ = forward

    @staticmethod
    def chunk_plan(T: int, chunk_tokens: int = 4096, ramp: int | None = None) -> list:
        """Token chunk sizes for the host pipeline: optionally smaller chunks
        at both ends (``ramp``: the first H2D and the last D2H are not
        overlapped with compute), ``chunk_tokens`` in the middle. Every chunk
        re-streams all expert weights (1.41 GB at the Mixtral shape, ~0.22 ms
        of HBM time), so below ~4096 tokens a chunk costs more than the
        copy time it hides: measured on B200, uniform 4096-token chunks are
        the fastest plan at T = 16384 (tools/e2e_probe.py)."""
        ramp = chunk_tokens if ramp is None else ramp
        sizes, head = [], []
        c = ramp
        while c < chunk_tokens and 2 * (sum(head) + c) <= T:
            head.append(c)
            c *= 2
        mid = T - 2 * sum(head)
        body = [chunk_tokens] * (mid // chunk_tokens)
        if mid % chunk_tokens:
            body.append(mid % chunk_tokens)
        sizes = head + body + head[::-1]
        return [s for s in sizes if s > 0]

    def forward_host(self, x_host: torch.Tensor, out_host: torch.Tensor | None = None,
                     chunk_tokens: int = 4096, chunks: list | None = None) -> torch.Tensor:
        """Host (pinned) tokens in, host tokens out: the end-to-end public
        call. Token chunks are pipelined over three streams so the H2D copy
        of chunk i+1 and the D2H copy of chunk i-1 overlap the forward of
        chunk i (the MoE layer is token-parallel, so chunking is exact)."""
        T = x_host.shape[0]
        if out_host is None:
            out_host = torch.empty((T, self.d), dtype=self.out_dtype, pin_memory=True)
        cur = torch.cuda.current_stream()
        # persistent copy streams and device staging buffer: per-call streams
        # would defeat the caching allocator (fresh cudaMalloc = device sync)
        if getattr(self, "_io", None) is None or self._io["xbuf"].shape[0] < T:
            self._io = {"h2d": torch.cuda.Stream(), "d2h": torch.cuda.Stream(),
                        "xbuf": torch.empty((T, self.d), dtype=x_host.dtype, device="cuda")}
        h2d, d2h, xbuf = self._io["h2d"], self._io["d2h"], self._io["xbuf"]
        h2d.wait_stream(cur)      # previous users of xbuf on the compute stream are done
        sizes = chunks if chunks is not None else self.chunk_plan(T, chunk_tokens)
        if sum(sizes) != T:
            raise ValueError(f"chunk sizes sum to {sum(sizes)}, expected {T}")
        starts = np.concatenate([[0], np.cumsum(sizes)]).tolist()
        bounds = list(zip(starts[:-1], starts[1:]))
        loaded = []
        with torch.cuda.stream(h2d):
            for lo, hi in bounds:
                xbuf[lo:hi].copy_(x_host[lo:hi], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(h2d)
                loaded.append(ev)
        for i, (lo, hi) in enumerate(bounds):
            cur.wait_event(loaded[i])
            y = self.forward(xbuf[lo:hi])
            ev = torch.cuda.Event()
            ev.record(cur)
            d2h.wait_event(ev)
            with torch.cuda.stream(d2h):
                out_host[lo:hi].copy_(y, non_blocking=True)
            y.record_stream(d2h)
        d2h.synchronize()
        return out_host

    def graphed(self, T: int, out_dtype=None) -> "GraphedForward":
        """Capture one forward over a fixed token count into a CUDA graph
        (static input / output buffers): the 10 kernel launches of a step
        replay as one graph launch — for small, launch-bound batches."""
        xs = torch.zeros((T, self.d), dtype=torch.bfloat16, device="cuda")
        cur = torch.cuda.current_stream()
        side = torch.cuda.Stream()
        side.wait_stream(cur)
        with torch.cuda.stream(side):          # warm-up outside the capture (kernel attributes, pools)
            for _ in range(2):
                self.forward(xs, out_dtype=out_dtype)
        cur.wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            ys = self.forward(xs, out_dtype=out_dtype)
        return GraphedForward(graph, xs, ys)

    def forward_host_stream(self, batches: list, depth: int = 2) -> list:
        """Serving loop over several host batches [(x_host, out_host), ...]:
        the same per-batch work as ``forward_host`` (H2D of the batch's
        tokens, forward, D2H of its result), software-pipelined ACROSS
        batches on three streams with ``depth`` device staging buffers for
        the inputs and ``depth`` for the outputs, so the H2D of batch b+1 and
        the D2H of batch b-1 overlap the forward of batch b. Every batch is
        forwarded whole (no per-chunk weight re-streaming); the staging ring
        keeps the allocator out of the loop (no cross-stream frees).
        Returns the out_host tensors after the last D2H."""
        from .hostio import stream_batches
        # the layer is token-parallel: the first and last batches go in 4
        # chunks, so the pipeline fill / drain expose a quarter of a copy
        return stream_batches(self, self.forward, self.d, self.out_dtype, batches, depth, split_ends=4)

    # ------------------------------------------------------------------
    def save(self, out_dir) -> None:
        """Persist the layer in the reference's own formats: every expert
        matrix as a MOEP ``gpu_int`` blob (quant.py:506-538; byte-identical to
        precision_pack), the smoothing vectors and router as MOEK float64
        matrices (numkit.py:110-157), plus a small layer.json."""
        import json
        from pathlib import Path

        from . import formats
        from .quant import precision_pack

        out = Path(out_dir)
        out.mkdir(parents=True, exist_ok=True)
        for e in range(self.E):
            ex = self.host_experts[e]
            for name in ("w1", "w3", "w2"):
                (out / f"expert{e}_{name}.moep").write_bytes(precision_pack(ex[name], "gpu_int").blob)
            for name in ("s13", "s2"):
                (out / f"expert{e}_{name}.moek").write_bytes(
                    formats.moek_encode(np.asarray(_np(ex[name]), np.float64).reshape(1, -1)))
        (out / "gate.moek").write_bytes(formats.moek_encode(self.gate_w.cpu().numpy().astype(np.float64)))
        if self.gate_b is not None:
            (out / "gate_bias.moek").write_bytes(
                formats.moek_encode(self.gate_b.cpu().numpy().astype(np.float64).reshape(1, -1)))
        (out / "layer.json").write_text(json.dumps({"experts": self.E, "top_k": self.k, "d": self.d, "ffn": self.F,
                                                    "out_dtype": str(self.out_dtype).replace("torch.", "")}))

    @classmethod
    def load(cls, in_dir) -> "MoELayer":
        """Inverse of ``save``: 8-bit MOEP payloads go straight to the device
        as the u8 GEMM operand (formats.moep_to_device, no repacking)."""
        import json
        from pathlib import Path

        from . import formats

        src = Path(in_dir)
        meta = json.loads((src / "layer.json").read_text())
        experts = []
        for e in range(meta["experts"]):
            ex = {}
            for name in ("w1", "w3", "w2"):
                t = formats.moep_to_device((src / f"expert{e}_{name}.moep").read_bytes())
                ex[name] = QuantizedMatrix(t["codes"], t["scale"], t["zp"], t["bits"], t["granularity"])
            for name in ("s13", "s2"):
                ex[name] = formats.moek_decode((src / f"expert{e}_{name}.moek").read_bytes()).ravel()
            experts.append(ex)
        gate = formats.moek_decode((src / "gate.moek").read_bytes()).astype(np.float32)
        gb = src / "gate_bias.moek"
        bias = formats.moek_decode(gb.read_bytes()).ravel().astype(np.float32) if gb.exists() else None
        return cls(gate, experts, top_k=meta["top_k"], out_dtype=getattr(torch, meta["out_dtype"]),
                   gate_bias=bias)

    # ------------------------------------------------------------------
    def expert_host(self, e: int) -> dict:
        """Host copies of expert e in the oracle's layout (codes/scales/zps of
        w1, w3, w2 and the smoothing vectors) — for parity tests and the CPU
        baseline."""
        ex = self.host_experts[e]
        out = {"s13": np.asarray(_np(ex["s13"]), dtype=np.float64), "s2": np.asarray(_np(ex["s2"]), dtype=np.float64)}
        for name in ("w1", "w3", "w2"):
            q = ex[name]
            out[f"{name}_codes"] = _np(q.codes).astype(np.int32)
            out[f"{name}_scale"] = _np(q.scales).astype(np.float64)
            out[f"{name}_zp"] = _np(q.zero_points).astype(np.int32)
        return out


def _np(a):
    return a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)


class MoEStack:
    """A stack of W8A8 Mixtral blocks with pre-norm residual connections,
    x = x + Attn_l(RMSNorm(x)); x = x + MoE_l(RMSNorm(x)) (bf16) — the token
    path of SURVEY.md C5; with ``attn=None`` the blocks are MoE-only. Every
    residual add is fused with the next RMSNorm (``moe_rmsnorm_residual``).
    ``forward(x, stats=RoutingStats(L, E, k))`` records every layer's
    routing, so ``stats.to_trace()`` is a reference trace whose events are
    the tokens' full activation paths (trace.py:40-44) — the input of
    placement.plan_path / plan_two_stage. Attention runs on packed
    sequences of ``seq_len`` tokens (causal)."""

    def __init__(self, layers: list, attn: list | None = None, seq_len: int | None = None):
        if not layers:
            raise ValueError("empty stack")
        if attn is not None and (len(attn) != len(layers) or not seq_len):
            raise ValueError("one attention block per layer and a seq_len are needed")
        self.layers = layers
        self.attn = attn
        self.seq_len = seq_len
        self.E, self.k, self.d = layers[0].E, layers[0].k, layers[0].d

    @classmethod
    def random(cls, L: int, E: int, d: int, F: int, top_k: int = 2, seed: int = 1, attention: bool = False,
               seq_len: int = 4096, heads: int = 32, kv_heads: int = 8, **kw) -> "MoEStack":
        layers = [MoELayer.random(E, d, F, top_k=top_k, seed=seed + 17 * l, router_seed=2 + 17 * l, **kw)
                  for l in range(L)]
        attn = None
        if attention:
            from .attention import W8A8Attention
            attn = [W8A8Attention.random(d, heads, kv_heads, d // heads, seed=seed + 17 * l + 5,
                                         max_pos=max(seq_len, 1)) for l in range(L)]
        return cls(layers, attn, seq_len if attention else None)

    @staticmethod
    def norm(x: torch.Tensor, eps: float = 1e-5) -> torch.Tensor:
        """RMSNorm without a learned gain (random-weight stacks): keeps the
        residual stream's scale bounded across layers (moe_rmsnorm_residual)."""
        return ops.rmsnorm_residual(x, None, eps)[1]

    @staticmethod
    def residual(x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
        """bf16(x + y), the block's residual add (same kernel)."""
        return ops.rmsnorm_residual(x, y, want_norm=False)[0]

    def forward(self, x: torch.Tensor, stats=None, timer=None, out: torch.Tensor | None = None) -> torch.Tensor:
        # one fused pass per block boundary: residual add + next block's norm
        if timer is not None:
            timer.mark("start")
        n = self.norm(x)
        for l, layer in enumerate(self.layers):
            if self.attn is not None:
                x, n = ops.rmsnorm_residual(x, self.attn[l](n, self.seq_len))
            y = layer.forward(n, stats=_LayerStats(stats, l) if stats is not None else None)
            if l + 1 < len(self.layers):
                x, n = ops.rmsnorm_residual(x, y)
            else:
                x = self.residual(x, y)
        if timer is not None:
            timer.mark("stack")
        if out is not None:
            out.copy_(x)
            return out
        return x

    __call__ = forward

    def forward_host(self, x_host: torch.Tensor, out_host: torch.Tensor | None = None) -> torch.Tensor:
        """Pinned host tokens in, host tokens out (one synchronous call)."""
        y = self.forward(x_host.to("cuda", non_blocking=True))
        if out_host is None:
            out_host = torch.empty(tuple(y.shape), dtype=y.dtype, pin_memory=True)
        out_host.copy_(y, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return out_host

    def forward_host_stream(self, batches: list, depth: int = 2) -> list:
        """Serving loop over host batches (hostio.stream_batches)."""
        from .hostio import stream_batches
        return stream_batches(self, self.forward, self.d, torch.bfloat16, batches, depth, split_ends=4,
                              quantum=self.seq_len or 1)


class _LayerStats:
    """Binds a RoutingStats to one layer index for MoELayer.forward."""

    def __init__(self, stats, layer: int):
        self.stats, self.layer = stats, layer

    def record(self, idx):
        self.stats.record(idx, self.layer)


class GraphedForward:
    """A captured ``MoELayer.forward``: call with [T, d] bf16 tokens; returns
    the static output buffer (overwritten by the next call)."""

    def __init__(self, graph, x_static: torch.Tensor, y_static: torch.Tensor):
        self.graph, self.x, self.y = graph, x_static, y_static

    def __call__(self, x: torch.Tensor) -> torch.Tensor:
        if x.shape != self.x.shape:
            raise ValueError(f"graph captured for {tuple(self.x.shape)}, got {tuple(x.shape)}")
        if x.data_ptr() != self.x.data_ptr():
            self.x.copy_(x)
        self.graph.replay()
        return self.y
