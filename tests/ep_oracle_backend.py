"""Float64 CPU compute backend for the expert-parallel runtime (TEST
INFRASTRUCTURE ONLY). It plugs the oracle's per-row arithmetic
(oracle/moe_ref.py) into ``paper_2508_07329_b200.ep.ExpertParallelMoE`` so
that the runtime's host logic — placement, route keys, send/receive counts,
regrouping, the gloo all-to-all exchanges and the return trip — can be
checked at world size 2 on CPU against ``moe_ref.moe_forward``.
"""

from __future__ import annotations

import numpy as np
import torch

from oracle import moe_ref as M


def random_experts(rng, E: int, d: int, F: int) -> list:
    out = []
    for _ in range(E):
        ex = {"s13": np.exp(rng.normal(size=d) * 0.5), "s2": np.exp(rng.normal(size=F) * 0.5)}
        for name, shape, s in (("w1", (F, d), "s13"), ("w3", (F, d), "s13"), ("w2", (d, F), "s2")):
            w = rng.normal(size=shape) * 0.02 * ex[s][None, :]
            c, sc, z = M.quantize_weight_rows(w)
            ex[f"{name}_codes"], ex[f"{name}_scale"], ex[f"{name}_zp"] = c, sc, z
        out.append(ex)
    return out


class OracleBackend:
    def __init__(self, wg, experts: list, local_experts, k: int = 2):
        self.wg = np.asarray(wg, dtype=np.float64)
        self.expert_params = experts
        self.local_experts = tuple(local_experts)
        self.k = k
        self.s13 = np.stack([e["s13"] for e in experts])

    @staticmethod
    def to_index_tensor(a):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32))

    @staticmethod
    def to_host(t):
        return t.numpy()

    def route(self, x):
        logits = M.gate_logits(x.numpy(), self.wg).astype(np.float32)
        idx, w, _ = M.router_topk(logits, self.k)
        return torch.from_numpy(idx.astype(np.int32)), torch.from_numpy(np.asarray(w, np.float64))

    def route_keys(self, idx, dest, E):
        return dest[idx.long()] * E + idx

    def permute(self, keys, w, G):
        off, src_token, src_slot, token_pos = M.permute(keys.numpy(), G)
        flat = keys.numpy().ravel()
        order = src_token.astype(np.int64) * self.k + src_slot
        return {"offsets": torch.from_numpy(off), "src_token": torch.from_numpy(src_token),
                "row_key": torch.from_numpy(flat[order].astype(np.int32)),
                "row_weight": torch.from_numpy(w.numpy()[src_token, src_slot]),
                "token_pos": torch.from_numpy(token_pos)}

    def quantize_pack(self, x, perm, E):
        rows = x.numpy()[perm["src_token"].numpy()]
        e = perm["row_key"].numpy() % E
        codes, scale, zp, rs = M.quantize_rows_grouped(rows, e, self.s13)
        params = np.stack([scale, zp.astype(np.float64), rs.astype(np.float64), perm["row_weight"].numpy()], 1)
        return [torch.from_numpy(codes.astype(np.int64)), torch.from_numpy(params)]

    def experts(self, recv, index, group_counts, mark=None):
        codes = recv[0].numpy()[index]
        prm = recv[1].numpy()[index]
        d = self.s13.shape[1]
        y = np.zeros((index.size, d))
        lo = 0
        for slot, e in enumerate(self.local_experts):
            hi = lo + int(group_counts[slot])
            if hi > lo:
                ex = self.expert_params[e]
                c, s, z = codes[lo:hi], prm[lo:hi, 0], prm[lo:hi, 1].astype(np.int64)
                g, _ = M.w8a8_linear(c, s, z, ex["w1_codes"], ex["w1_scale"], ex["w1_zp"])
                u, _ = M.w8a8_linear(c, s, z, ex["w3_codes"], ex["w3_scale"], ex["w3_zp"])
                ch, sh, zh, _ = M.quantize_rows(M.silu(g) * u, ex["s2"])
                ye, _ = M.w8a8_linear(ch, sh, zh, ex["w2_codes"], ex["w2_scale"], ex["w2_zp"])
                y[lo:hi] = prm[lo:hi, 3][:, None] * ye
            lo = hi
        out = np.empty_like(y)
        out[index] = y
        return torch.from_numpy(out)

    def combine(self, y_home, perm, T, out=None):
        y = y_home.numpy()
        pos = perm["token_pos"].numpy()
        acc = np.zeros((T, y.shape[1]))
        for j in range(self.k):
            acc = acc + y[pos[:, j]]
        if out is not None:
            out.copy_(torch.from_numpy(acc))
            return out
        return torch.from_numpy(acc)
