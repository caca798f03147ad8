"""The attention half of a Mixtral block for the 32-layer token path
(SURVEY.md §8 f4, config C5), W8A8 like the experts.

The reference has no forward at all (its only W8A8 product is the
fake-quant loss, quant.py:281-283); this block exists so that
``bench.py --layers 32`` runs the whole Mixtral token path:

    n = RMSNorm(x);  q, k, v = split(W8A8(n; W_qkv));  RoPE(q, k)
    a = causal GQA attention(q, k, v);  x = x + W8A8(a; W_o)

* the three projections share their input, so they are ONE W8A8 linear
  (``W8A8Linear``: K1 with the HAQ smoothing division fused in, then the
  tcgen05 kind::i8 GEMM with the dequant epilogue) over the stacked
  [W_q; W_k; W_v] — one activation quantization, one GEMM;
* rotary embedding: ``moe_rope_bf16`` in place on the q and k heads of the
  bf16 QKV rows (float64-built cos / sin tables, float32 products);
* attention: the library's scaled-dot-product attention on bf16 (cuDNN /
  flash kernels — a library call, like cuBLAS), causal per sequence,
  grouped-query (8 KV heads for 32 query heads at the Mixtral shape);
* the output projection: a second W8A8 linear.

Expert parallelism does not touch this block: tokens stay on their home
rank and every rank holds the (replicated) attention weights — SURVEY.md
§8e: "Dense W8A8 linears ... attention projections in C5: replicas only".
"""

from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F

from . import _lib as L
from . import ops
from .linear import W8A8Linear
from .quant import PER_OUTPUT_ROW, QuantizedMatrix


class W8A8Attention:
    def __init__(self, qkv: W8A8Linear, o: W8A8Linear, heads: int, kv_heads: int, head_dim: int,
                 theta: float = 1e6, max_pos: int = 32768):
        if qkv.out_features != (heads + 2 * kv_heads) * head_dim:
            raise ValueError("qkv projection must produce (heads + 2 kv_heads) * head_dim features")
        if o.in_features != heads * head_dim or o.out_features != qkv.in_features:
            raise ValueError("output projection must map heads * head_dim back to d")
        if heads % kv_heads:
            raise ValueError("heads must be a multiple of kv_heads")
        self.qkv, self.o = qkv, o
        self.d = qkv.in_features
        self.heads, self.kv_heads, self.head_dim = heads, kv_heads, head_dim
        self.theta, self.max_pos = theta, max_pos
        self.cos, self.sin = ops.rope_tables(max_pos, head_dim, theta)
        self._pos = {}

    @classmethod
    def random(cls, d: int = 4096, heads: int = 32, kv_heads: int = 8, head_dim: int = 128, seed: int = 1,
               smooth_exponent: float = 0.5, **kw) -> "W8A8Attention":
        """Random-init Mixtral-shape attention (W ~ N(0, 0.02^2)), W s
        quantized per output row on device with synthetic smoothing factors
        (1 % of channels x100 in the statistic, as MoELayer.random)."""
        g = torch.Generator(device="cuda").manual_seed(seed)
        rng = np.random.default_rng(seed)

        def stat(n):
            s = np.abs(rng.normal(size=n)) + 1.0
            s[rng.choice(n, max(1, n // 100), replace=False)] *= 100.0
            return s ** smooth_exponent

        def lin(rows, cols):
            s = stat(cols)
            w = torch.randn((rows, cols), generator=g, device="cuda", dtype=torch.float32) * 0.02
            sm = torch.as_tensor(s, dtype=torch.float64).reshape(1, -1).cuda()
            q = ops.act_quant(w, smooth=sm, smooth_mode=L.SMOOTH_MULTIPLY, granularity=PER_OUTPUT_ROW,
                              rowsum=False)
            return W8A8Linear(QuantizedMatrix(q["codes"], q["scale"], q["zp"], 8, PER_OUTPUT_ROW), s)

        return cls(lin((heads + 2 * kv_heads) * head_dim, d), lin(d, heads * head_dim), heads, kv_heads, head_dim,
                   **kw)

    def positions(self, T: int, seq_len: int) -> torch.Tensor:
        """Position of every row of a batch of T / seq_len packed sequences."""
        key = (T, seq_len)
        if key not in self._pos:
            if T % seq_len or seq_len > self.max_pos:
                raise ValueError(f"{T} tokens are not whole sequences of {seq_len} (max_pos {self.max_pos})")
            self._pos[key] = (torch.arange(T, device="cuda", dtype=torch.int32) % seq_len).contiguous()
        return self._pos[key]

    def project_qkv(self, x: torch.Tensor, seq_len: int) -> torch.Tensor:
        """The fused W8A8 QKV projection with RoPE applied to q and k: [T, (H + 2 Hkv) hd] bf16."""
        qkv = self.qkv(x, out_dtype=torch.bfloat16)
        pos = self.positions(x.shape[0], seq_len)
        H, Hk, hd = self.heads, self.kv_heads, self.head_dim
        ops.rope_(qkv, H, hd, self.cos, self.sin, pos)
        ops.rope_(qkv[:, H * hd:], Hk, hd, self.cos, self.sin, pos)
        return qkv

    def attend(self, qkv: torch.Tensor, seq_len: int) -> torch.Tensor:
        """Causal grouped-query attention of the packed sequences: [T, H hd] bf16."""
        T = qkv.shape[0]
        B, H, Hk, hd = T // seq_len, self.heads, self.kv_heads, self.head_dim
        q = qkv[:, : H * hd].view(B, seq_len, H, hd).transpose(1, 2)
        k = qkv[:, H * hd:(H + Hk) * hd].view(B, seq_len, Hk, hd).transpose(1, 2)
        v = qkv[:, (H + Hk) * hd:].view(B, seq_len, Hk, hd).transpose(1, 2)
        a = F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=(Hk != H))
        return a.transpose(1, 2).reshape(T, H * hd)

    def forward(self, x: torch.Tensor, seq_len: int) -> torch.Tensor:
        if x.dim() != 2 or x.shape[1] != self.d:
            raise ValueError(f"expected input [T, {self.d}], got {tuple(x.shape)}")
        return self.o(self.attend(self.project_qkv(x, seq_len), seq_len), out_dtype=torch.bfloat16)

    __call__ = forward
