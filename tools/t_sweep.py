"""Token-count sweep of the Mixtral-shape W8A8 MoE layer (SURVEY.md §8d C4:
T in {4096, 8192, 16384}, plus small serving/decode batches where the layer
is expert-weight-stream (HBM) bound).

    python tools/t_sweep.py [out.json]  ->  prints JSON lines, writes profiles/tsweep_r01.json

Per T: eager forward and CUDA-graph replay (CUDA events, mean of n steps
after warm-up), per-stage split, int8 TOPS over the layer, and the HBM
roofline of the weight stream (1.41 GB of u8 expert weights + activations
per step) against the measured HBM peak."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from bench import D, E, F, OPS_PER_TOKEN, TOPK, StageTimer, synth_tokens
from paper_2508_07329_b200.moe import MoELayer

PEAKS = json.load(open("MEASURED_PEAKS.json")) if os.path.exists("MEASURED_PEAKS.json") else {}
HBM = float(PEAKS.get("hbm_gbs", 6536.0))
INT8 = json.load(open("profiles/int8_peak.json"))["cublaslt_int8_burst"]


def timed(fn, n, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def main():
    layer = MoELayer.random(E, D, F, top_k=TOPK, seed=1)
    wbytes = sum(int(t.numel()) for t in (layer.w13["codes"], layer.w2["codes"]))
    x_all = torch.from_numpy(synth_tokens(16384, D, seed=100)).to(torch.bfloat16).cuda()
    rows = []
    for T in (16, 64, 256, 1024, 2048, 4096, 8192, 16384):
        x = x_all[:T].contiguous()
        n = 50 if T <= 2048 else 20
        ms = timed(lambda: layer.forward(x), n)
        g = layer.graphed(T)
        ms_g = timed(lambda: g(x), n)
        del g
        layer.forward(x, timer=StageTimer())     # allocations for this T outside the stage timing
        torch.cuda.synchronize()
        tm = StageTimer()
        for _ in range(5):
            layer.forward(x, timer=tm)
        torch.cuda.synchronize()
        stages = {k: round(v / 5, 4) for k, v in tm.stage_ms().items()}
        best = min(ms, ms_g)
        act = T * (D * 2) * 2 + T * TOPK * (D + F * 3 + F) + T * TOPK * D * 4   # x in/out, codes, h, y (approx.)
        r = {"T": T, "ms_eager": ms, "ms_graph": ms_g, "tokens_per_s": T / (best / 1e3),
             "int8_tops": T * OPS_PER_TOKEN / (best / 1e3) / 1e12, "int8_frac": T * OPS_PER_TOKEN / (best / 1e3) / 1e12 / INT8,
             "weight_stream_gbs": wbytes / (best / 1e3) / 1e9,
             "hbm_frac_weights_only": wbytes / (best / 1e3) / 1e9 / HBM,
             "hbm_floor_ms": (wbytes + act) / HBM / 1e6, "stages_ms": stages}
        rows.append(r)
        print(json.dumps(r), flush=True)
        torch.cuda.empty_cache()
    out = {"gpu": torch.cuda.get_device_name(), "weights_bytes": wbytes, "hbm_peak_gbs": HBM,
           "int8_peak_tops": INT8, "rows": rows}
    path = sys.argv[1] if len(sys.argv) > 1 else "profiles/tsweep_r01.json"
    os.makedirs(os.path.dirname(path) or ".", exist_ok=True)
    with open(path, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
