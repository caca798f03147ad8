"""Predicted per-rank expert load of the EP forward at W = 2/4/8 under the
bench's routing (bench.synth_tokens per rank, MoELayer.random's router:
N(0, 1/d) gate + Zipf(1.2) logit bias), for four placements:
  sharded        one holder per expert, contiguous blocks
  from_counts    round-1 design: plan_two_stage residents replicated, the
                 rest bin-packed one holder each
  balanced       residents replicated, hot sharded experts split over
                 ceil(load / share) holders (ExpertPlacement.balanced)
  balanced_norep no residents, load split only
Routing is computed on the CPU in float32 (counts only; the GPU router's
exact ids are not needed for a load prediction).

    python tools/ep_load_table.py [tokens_per_rank] -> profiles/ep_load_r02.json
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import D, E, TOPK, synth_tokens  # noqa: E402
from paper_2508_07329_b200.ep import ExpertPlacement  # noqa: E402
from paper_2508_07329_b200.placement import plan_two_stage  # noqa: E402
from paper_2508_07329_b200.trace import PHASE_PREFILL, RoutingEvent, Trace, expert_freq, path_stats  # noqa: E402


def router():
    rr = np.random.default_rng(2)
    gw = rr.normal(size=(E, D)) / np.sqrt(D)
    bias = np.log(1.0 / (np.arange(E) + 1.0) ** 1.2)
    bias = bias - np.log(np.exp(bias).sum())
    return gw.astype(np.float32), bias[np.argsort(rr.permutation(E))].astype(np.float32)


def main():
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    gw, gb = router()
    out = {"tokens_per_rank": T, "experts": E, "top_k": TOPK, "worlds": {}}
    sel_all = []
    for r in range(8):
        x = synth_tokens(T, D, seed=100 + r)
        x = (x.view(np.uint32) & 0xFFFF0000).view(np.float32)        # bf16 truncation (approximate)
        logits = x @ gw.T + gb
        sel_all.append(np.argsort(-logits, axis=1, kind="stable")[:, :TOPK])
    for W in (2, 4, 8):
        sel = np.concatenate(sel_all[:W])
        counts = np.bincount(sel.ravel(), minlength=E)
        paths = [tuple(sorted(map(int, s))) for s in sel]
        trace = Trace(1, E, TOPK, [RoutingEvent(i, PHASE_PREFILL, (p,)) for i, p in enumerate(paths)])
        freq = expert_freq(trace)
        plan = plan_two_stage(path_stats(trace), freq, 1, 1)
        res = plan.residents[0]
        pls = {"sharded": ExpertPlacement.sharded(E, W),
               "from_counts": ExpertPlacement.from_counts(counts, W, res),
               "balanced": ExpertPlacement.balanced(counts, W, res),
               "balanced_norep": ExpertPlacement.balanced(counts, W)}
        row = {"counts": counts.tolist(), "residents": list(res)}
        for name, pl in pls.items():
            ld = pl.rank_loads(counts)
            row[name] = {"max_over_mean": float(ld.max() / ld.mean()), "loads": [round(v) for v in ld],
                         "local_fraction": pl.local_fraction(counts),
                         "experts_held_max": max(len(pl.local_experts(r)) for r in range(W)),
                         "holders": [list(pl.holders(e)) for e in range(E)]}
        out["worlds"][W] = row
        print(W, {k: round(v["max_over_mean"], 3) for k, v in row.items() if isinstance(v, dict)},
              {k: round(v["local_fraction"], 3) for k, v in row.items() if isinstance(v, dict)})
    (ROOT / "profiles" / "ep_load_r02.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
