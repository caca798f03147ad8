"""HAQ calibration of one linear layer with the calibration tokens sharded
over the ranks of a process group ("Calibration Hessian —
token-sharded partial H plus an all-reduce; GPTQ column loop — shard R
across GPUs with U replicated").

The reference's quantize_layer (quant.py:437-490) is decomposed into the
steps a token shard can do alone and the reductions between them:

Per-token activation quantization (the W8A8 forward's configuration): a
token's parameters depend on that token alone.

1. per-channel max |x| (smoothing statistic, quant.py:303)  -> all-reduce MAX
   (exact: the same statistic as on one GPU);
2. the 21 grid-point losses ||Q(W f) Q(X/f) - W X||^2 of the shard
   (quant.py:286-311; per-token activation params are per shard row)     -> all-reduce SUM;
   every rank then picks the same exponent (strict '<': ties keep the
   smaller one);
3. the partial Hessian 2 Xs Xs^T of the shard (K7, quant.py:327-343)     -> all-reduce SUM,
   then the damping and the inverse factor U on every rank (identical
   input, identical U);
4. the GPTQ column loop (K8, quant.py:388-434) on this rank's slice of
   the weight rows with the replicated U -> all-gather of the codes. Rows are
   independent, so a slice's codes are bit-identical to the same rows of a
   single-GPU run given the same U.

Only the order of the float sums in steps 2-3 differs from one GPU (the
loss and H are equal to ~1e-15 relative), so the exponent and the codes can
differ from a single-GPU run only at exact near-ties.

``quantize_layer_sharded`` drives it over torch.distributed (NCCL on
GPUs); ``run_loopback_calibration`` drives W shards in one process (tests,
single-GPU emulation).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from . import ops
from .quant import (DEFAULT_DAMPING, DEFAULT_GRID_STEPS, PER_OUTPUT_ROW, PER_TOKEN, STAT_FLOOR, LayerQuantResult,
                    QuantConfig, QuantizedMatrix, SmoothingResult, _inverse_upper_factor_device, _k1,
                    _LossContext)


class ShardedLayerCalibration:
    """One rank's part of quantize_layer: w [R, n] (every rank holds all of
    it), x_shard [n, T_rank] (this rank's calibration tokens, reference
    layout). Call the steps in order, feeding each the reduced result of the
    previous one."""

    def __init__(self, w, x_shard, cfg: QuantConfig | None = None, grid_steps: int = DEFAULT_GRID_STEPS,
                 rank: int = 0, world: int = 1):
        self.cfg = cfg or QuantConfig(bits=8, symmetric=False, granularity=PER_TOKEN)
        if self.cfg.granularity != PER_TOKEN:
            # per_tensor activation params span every token: they would need one more
            # reduction per grid point; the W8A8 forward path quantizes per token
            raise ValueError("token-sharded calibration needs per_token activation quantization")
        if grid_steps < 2:
            raise ValueError(f"grid_steps must be at least 2, got {grid_steps}")
        self.ctx = _LossContext(w, x_shard, self.cfg)
        self.grid = np.linspace(0.0, 1.0, grid_steps)
        self.rank, self.world = rank, world
        R = self.ctx.wd.shape[0]
        per = (R + world - 1) // world
        self.r0, self.r1 = min(R, rank * per), min(R, (rank + 1) * per)

    # 1. smoothing statistic
    def local_stat(self) -> torch.Tensor:
        return ops.channel_stats(self.ctx.xt.T.contiguous(), L.ORDER_MAX_ABS)

    # 2. grid-point losses of this shard
    def local_losses(self, stat: torch.Tensor) -> torch.Tensor:
        s = np.maximum(stat.cpu().numpy(), STAT_FLOOR)
        self.factors = [s ** e for e in self.grid]            # numpy pow, as quant.search_smoothing
        return torch.stack([self.ctx.sq_error_dev(torch.from_numpy(f).cuda()).reshape(()) for f in self.factors])

    def choose(self, sq_total: torch.Tensor) -> SmoothingResult:
        best = None
        for e, f, v in zip(self.grid, self.factors, sq_total.cpu().numpy()):
            loss = float(np.sqrt(float(v)))
            if best is None or loss < best.loss:
                best = SmoothingResult(float(e), f, loss)
        self.smoothing = best
        return best

    # 3. partial Hessian of the smoothed shard
    def local_hessian(self) -> tuple[torch.Tensor, torch.Tensor]:
        f = torch.from_numpy(self.smoothing.factors).cuda()
        self.ws, xs = ops.apply_smoothing(self.ctx.wd, self.ctx.xt.T.contiguous(), f)
        nonzero = torch.zeros(1, dtype=torch.int64, device=self.ws.device)
        H = ops.hessian(xs.T.contiguous(), finalize=False, nonzero=nonzero)
        return H, nonzero

    def finish_hessian(self, H_total: torch.Tensor, nonzero_total: torch.Tensor,
                       damping_fraction: float = DEFAULT_DAMPING) -> torch.Tensor:
        n = H_total.shape[0]
        L.call("moe_hessian_finalize", L.ptr(H_total), n, float(damping_fraction), L.ptr(nonzero_total),
               ops._s())
        self.U = _inverse_upper_factor_device(H_total)
        self.params = _k1(self.ws, self.cfg, PER_OUTPUT_ROW)    # per-row params of the whole (unpermuted) W
        return self.U

    # 4. this rank's rows of the compensated quantization
    def local_codes(self) -> torch.Tensor:
        if self.r1 <= self.r0:
            return torch.empty((0, self.ws.shape[1]), dtype=torch.uint8, device=self.ws.device)
        return ops.gptq_columns(self.ws[self.r0:self.r1].contiguous(), self.U,
                                self.params["scale"][self.r0:self.r1].contiguous(),
                                self.params["zp"][self.r0:self.r1].contiguous(), self.cfg.bits)

    def result(self, codes: torch.Tensor) -> LayerQuantResult:
        p = self.params
        q = QuantizedMatrix(codes.cpu().numpy().astype(np.int32), p["scale"].cpu().numpy(), p["zp"].cpu().numpy(),
                            self.cfg.bits, PER_OUTPUT_ROW)
        # output_mse / rtn_baseline_mse need every token: reported by the driver
        return LayerQuantResult(q, self.smoothing, None, float("nan"), float("nan"))

    def local_mse_terms(self, codes: torch.Tensor) -> torch.Tensor:
        """This shard's squared errors of the calibrated and of the RTN layer (quant.py:475-482)."""
        wq = {"codes": codes, "scale": self.params["scale"], "scale_f32": self.params["scale_f32"],
              "zp": self.params["zp"], "rowsum": codes.sum(dim=1, dtype=torch.int32)}
        f = torch.from_numpy(self.smoothing.factors).cuda()
        return torch.stack([self.ctx.sq_error_dev(f, w_codes=wq).reshape(()),
                            self.ctx.sq_error_dev(None).reshape(())])


def quantize_layer_sharded(w, x_shard, cfg: QuantConfig | None = None, grid_steps: int = DEFAULT_GRID_STEPS,
                           group=None) -> LayerQuantResult:
    """quantize_layer with this rank's calibration tokens x_shard [n, T_rank];
    every rank returns the same result."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    c = ShardedLayerCalibration(w, x_shard, cfg, grid_steps, rank, world)
    stat = c.local_stat()
    dist.all_reduce(stat, op=dist.ReduceOp.MAX, group=group)
    sq = c.local_losses(stat)
    dist.all_reduce(sq, group=group)
    c.choose(sq)
    H, nz = c.local_hessian()
    dist.all_reduce(H, group=group)
    dist.all_reduce(nz, group=group)
    c.finish_hessian(H, nz)
    mine = c.local_codes()
    R, n = c.ws.shape
    per = (R + world - 1) // world
    buf = torch.zeros((per, n), dtype=torch.uint8, device=c.ws.device)
    buf[: mine.shape[0]] = mine
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    codes = torch.cat(parts)[:R].contiguous()
    terms = c.local_mse_terms(codes)
    dist.all_reduce(terms, group=group)
    tokens = torch.tensor([c.ctx.xt.shape[0]], dtype=torch.int64, device=c.ws.device)
    dist.all_reduce(tokens, group=group)
    res = c.result(codes)
    numel = float(R * int(tokens.item()))
    t = terms.cpu().numpy()
    res.output_mse, res.rtn_baseline_mse = float(t[0]) / numel, float(t[1]) / numel
    return res


def run_loopback_calibration(w, x_shards: list, cfg: QuantConfig | None = None,
                             grid_steps: int = DEFAULT_GRID_STEPS) -> tuple[LayerQuantResult, list]:
    """Drive len(x_shards) ranks in one process (the reductions are sums /
    maxima of the ranks' tensors in rank order). Returns the result and the
    per-rank contexts (for inspection)."""
    W = len(x_shards)
    cs = [ShardedLayerCalibration(w, xs, cfg, grid_steps, r, W) for r, xs in enumerate(x_shards)]
    stat = torch.stack([c.local_stat() for c in cs]).amax(dim=0)
    sqs = [c.local_losses(stat) for c in cs]
    sq = sqs[0].clone()
    for s in sqs[1:]:
        sq += s
    for c in cs:
        c.choose(sq)
    parts = [c.local_hessian() for c in cs]
    H = parts[0][0].clone()
    nz = parts[0][1].clone()
    for h, z in parts[1:]:
        H += h
        nz += z
    for c in cs:
        c.finish_hessian(H.clone(), nz.clone())
    codes = torch.cat([c.local_codes() for c in cs]).contiguous()
    terms = torch.stack([c.local_mse_terms(codes) for c in cs]).sum(dim=0).cpu().numpy()
    res = cs[0].result(codes)
    numel = float(codes.shape[0] * sum(c.ctx.xt.shape[0] for c in cs))
    res.output_mse, res.rtn_baseline_mse = float(terms[0]) / numel, float(terms[1]) / numel
    return res, cs
