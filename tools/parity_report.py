"""Oracle parity numbers at the exact bench configuration (C4 Mixtral layer,
T = 4096 / 16384) -> profiles/parity_<tag>.json. The checks and their
definitions are in tests/parity_bench.py (shared with the -m gpu test)."""

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from bench import synth_tokens  # noqa: E402
from paper_2508_07329_b200.moe import MoELayer  # noqa: E402
from tests.parity_bench import D, E, F, K, check_bench_config  # noqa: E402


def main(tag="r02", per_expert=96):
    torch.cuda.set_device(0)
    layer = MoELayer.random(E, D, F, top_k=K, seed=1)
    res = {}
    for T in (4096, 16384):
        x = torch.from_numpy(synth_tokens(T, D, seed=100)).cuda().bfloat16()
        res[str(T)] = check_bench_config(layer, x, per_expert=per_expert, assert_ok=False)
        print(json.dumps(res[str(T)]), flush=True)
    out = ROOT / "profiles" / f"parity_{tag}.json"
    out.write_text(json.dumps({"config": "C4 Mixtral layer, bench.synth_tokens(seed=100), MoELayer.random(seed=1)",
                               "per_expert_sample": per_expert, "results": res}, indent=1))
    print("wrote", out)


if __name__ == "__main__":
    main(*sys.argv[1:2])
