"""GPU: oracle parity at the exact configuration bench.py times (C4 Mixtral
layer, default knobs: CTA-pair grouped GEMMs, banded W2 raster, row-ext
speculation, GEMM2 with the fused top-2 combine) at T = 4096 and 16384
tokens. The checks live in tests/parity_bench.py; tools/parity_report.py
writes the same numbers to profiles/."""

import pytest
import torch

from .parity_bench import D, E, F, K, check_bench_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bench_layer(cuda):
    from paper_2508_07329_b200.moe import MoELayer
    return MoELayer.random(E, D, F, top_k=K, seed=1)       # == bench.py's layer


@pytest.mark.parametrize("T", [4096, 16384])
def test_bench_config_parity(cuda, bench_layer, T):
    from bench import synth_tokens
    x = torch.from_numpy(synth_tokens(T, D, seed=100)).to(cuda).bfloat16()
    rep = check_bench_config(bench_layer, x, per_expert=48)
    e2e = rep["end_to_end_from_x"]
    # precise mode (float32 h): within the north star's 1e-3 of the float64 oracle from x
    assert e2e["f32_h_precise"]["normwise_rel_err"] < 1e-3, e2e
    assert e2e["f32_h_precise"]["h_code_flip_rate"] < 1e-3, e2e
    # serving mode (bf16 h): bounded, documented deviation
    assert e2e["bf16_h"]["normwise_rel_err"] < 2e-2, e2e
