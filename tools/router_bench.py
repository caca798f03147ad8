"""Tensor-core router kernels at the Mixtral shape (d=4096, E=8, top-2):
cluster split-K vs persistent multi-accumulator, per token count. 20 calls
captured in a CUDA graph (no host overhead), CUDA-event timed.

    python tools/router_bench.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2508_07329_b200 import _lib as L
from paper_2508_07329_b200 import ops

d = 4096
x = torch.from_numpy(bench.synth_tokens(16384, d, 100)).to(torch.bfloat16).cuda()
wg = torch.randn(8, d, device="cuda") / d ** 0.5
for T in (1, 16, 128, 512, 1024, 2048, 4096, 8192, 16384):
    xs = x[:T].contiguous()
    res = {}
    for name, tiles in (("cluster", 1 << 40), ("persistent", 0)):
        with L.tuned(L.TUNE_ROUTER_CLUSTER_TILES, tiles):
            for _ in range(2):
                ops.router_gate(xs, wg, 2, want_logits=False, tensor_cores=True)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(20):
                    ops.router_gate(xs, wg, 2, want_logits=False, tensor_cores=True)
            g.replay()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(5):
                g.replay()
            b.record()
            torch.cuda.synchronize()
            res[name] = a.elapsed_time(b) / 100 * 1e3
    print(f"T={T:6d}  cluster {res['cluster']:7.1f} us  persistent {res['persistent']:7.1f} us", flush=True)
