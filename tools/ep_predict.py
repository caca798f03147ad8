"""Predicted expert-parallel step time at W = 2/4/8 GPUs from W ranks
emulated on ONE B200 at the Mixtral shape (bench routing, T tokens per
rank, weak scaling): every rank's three phases of the peer-memory forward
run for real (same kernels, device-side plan; the peers are other buffers
on the one GPU, ranks run phase by phase) and are timed with CUDA events:

  send     router, permutation, plan, K1 dispatch into the owners' buffers
  compute  grouped GEMM13 + SwiGLU, K1 on h, GEMM2 scattering to home ranks
  combine  the home rank's top-2 combine

Ranks synchronise between phases (two device barriers), so the predicted
step is sum over phases of the slowest rank; NVLink transfer time is not
modelled beyond the dispatch writes landing in local HBM (the dispatch
moves d + 16 bytes per remote row, ~14 ns per row at 900 GB/s, overlapped
with K1). Placements: `balanced` (plan_two_stage residents + load split,
the default) and `round1` (residents + one holder per expert).

    python tools/ep_predict.py [T] [out.json]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_07329_b200.ep import (CudaExpertBackend, ExpertPlacement, PeerBuffers,  # noqa: E402
                                      PeerExpertParallelMoE, plan_placement)
from paper_2508_07329_b200.moe import MoELayer  # noqa: E402


class _Local:
    def __init__(self, world, rank):
        self.world, self.rank = world, rank


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


def run(layer, xs, pl, reps=4):
    W, T = len(xs), xs[0].shape[0]
    cap_home = T * 2
    bufs = PeerBuffers.loopback(W, 4096, 2 * cap_home, cap_home)
    ranks = [PeerExpertParallelMoE(CudaExpertBackend.from_layer_spec(layer, pl.local_experts(r)), pl, bufs[r],
                                   rank=r, exchange=_Local(W, r)) for r in range(W)]
    best = None
    for rep in range(reps):
        t = {"send": [0.0] * W, "compute": [0.0] * W, "combine": [0.0] * W}
        sts, prep, snd, cb, plans, outs = [], [], [], [], [], []
        for r, m in enumerate(ranks):
            a = ev()
            sts.append(m.peer_prepare(xs[r]))
            prep.append((a, ev()))
        offs = torch.stack([st.perm["offsets"] for st in sts])     # the all-gather
        for m, st in zip(ranks, sts):
            a = ev()
            p = m.peer_plan(offs)
            m.peer_send(st, p)
            snd.append((a, ev()))
            plans.append(p)
        order = list(range(W)) if rep % 2 == 0 else list(range(W))[::-1]   # position effects show up
        cp = [None] * W
        for r in order:
            a = ev()
            ranks[r].peer_compute(plans[r])
            cp[r] = (a, ev())
        for m, st in zip(ranks, sts):
            a = ev()
            outs.append(m.peer_finish(st))
            cb.append((a, ev()))
        torch.cuda.synchronize()
        for r in range(W):
            t["send"][r] = prep[r][0].elapsed_time(prep[r][1]) + snd[r][0].elapsed_time(snd[r][1])
            t["compute"][r] = cp[r][0].elapsed_time(cp[r][1])
            t["combine"][r] = cb[r][0].elapsed_time(cb[r][1])
        t["received_rows"] = [int(p[1].item()) for p in plans]
        step = sum(max(v) for k, v in t.items() if k != "received_rows")
        if best is None or step < best[0]:
            best = (step, t, outs)
    for m in ranks:
        m.check(wait=True)
    return best


def main():
    T = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 8192
    out_path = next((a for a in sys.argv[1:] if a.endswith(".json")), None)
    layer = MoELayer.random(8, 4096, 14336, top_k=2, seed=1)
    x1 = torch.from_numpy(bench.synth_tokens(T, 4096, 100)).to(torch.bfloat16).cuda()
    for _ in range(3):
        layer.forward(x1)
    torch.cuda.synchronize()
    a = ev()
    for _ in range(5):
        layer.forward(x1)
    b = ev()
    torch.cuda.synchronize()
    single = a.elapsed_time(b) / 5
    res = {"tokens_per_rank": T, "single_gpu_ms": single, "worlds": {}}
    print(f"single GPU, {T} tokens: {single:.3f} ms", flush=True)
    for W in (2, 4, 8):
        xs = [torch.from_numpy(bench.synth_tokens(T, 4096, 100 + r)).to(torch.bfloat16).cuda() for r in range(W)]
        idx = layer.route(torch.cat(xs))[1]
        counts = np.bincount(idx.cpu().numpy().ravel(), minlength=8)
        bal = plan_placement(idx, 8, 2, W)
        r1 = ExpertPlacement.from_counts(counts, W, bal.replicated)
        row = {}
        for name, pl in (("balanced", bal), ("round1", r1)):
            step, t, outs = run(layer, xs, pl)
            exact = all(torch.equal(o, layer.forward(x)) for o, x in zip(outs, xs))
            row[name] = {"predicted_step_ms": step, "weak_scaling_efficiency": single / step,
                         "phase_max_ms": {k: max(v) for k, v in t.items() if k != "received_rows"},
                         "compute_ms_per_rank": t["compute"], "received_rows": t["received_rows"],
                         "bit_identical": exact,
                         "holders": [list(pl.holders(e)) for e in range(8)], "replicated": list(pl.replicated),
                         "predicted_load_max_over_mean": float(pl.rank_loads(counts).max()
                                                               / pl.rank_loads(counts).mean())}
            print(W, name, json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in row[name].items()
                                       if k not in ("holders", "compute_ms_per_rank")}), flush=True)
            del outs
            torch.cuda.empty_cache()
        res["worlds"][W] = row
        del xs
        torch.cuda.empty_cache()
    if out_path:
        json.dump(res, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main()
