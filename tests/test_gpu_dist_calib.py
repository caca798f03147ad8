"""GPU: HAQ calibration with the calibration tokens sharded over ranks
(SURVEY.md §8e): statistic all-reduce MAX, grid losses and partial
Hessians all-reduce SUM, GPTQ rows sharded with the replicated U. One shard
reproduces quantize_layer bit for bit; several shards (emulated in one
process) agree with it up to float-sum order, and the row sharding of the
column loop is bit-exact given U. Also a real NCCL world of one."""

import os
import socket
import subprocess
import sys
import textwrap

import numpy as np
import pytest
import torch

from paper_2508_07329_b200 import ops, quant
from paper_2508_07329_b200.dist_calib import run_loopback_calibration

pytestmark = pytest.mark.gpu


def _problem(R=384, n=256, T=600, seed=0):
    rng = np.random.default_rng(seed)
    w = rng.normal(size=(R, n)) * 0.05
    x = rng.normal(size=(n, T))
    x[rng.choice(n, 4, replace=False)] *= 40.0
    return w, x


CFG = quant.QuantConfig(8, False, quant.PER_TOKEN)


def test_one_shard_is_quantize_layer(cuda):
    w, x = _problem()
    ref = quant.quantize_layer(w, x, CFG)
    res, _ = run_loopback_calibration(w, [x], CFG)
    assert res.smoothing.exponent == ref.smoothing.exponent
    np.testing.assert_array_equal(res.quantized.codes, ref.quantized.codes)
    np.testing.assert_array_equal(res.quantized.scales, ref.quantized.scales)
    assert res.output_mse == pytest.approx(ref.output_mse, rel=1e-12)


@pytest.mark.parametrize("W", [2, 3])
def test_sharded_tokens_agree(cuda, W):
    w, x = _problem(seed=W)
    ref = quant.quantize_layer(w, x, CFG)
    shards = np.array_split(x, W, axis=1)
    res, cs = run_loopback_calibration(w, shards, CFG)
    assert res.smoothing.exponent == ref.smoothing.exponent
    np.testing.assert_array_equal(res.smoothing.factors, ref.smoothing.factors)
    agree = np.mean(res.quantized.codes == ref.quantized.codes)
    assert agree > 0.999, agree                      # only float-sum-order near-ties may differ
    # the row-sharded column loop is bit-exact given the replicated U
    c = cs[0]
    full = ops.gptq_columns(c.ws, c.U, c.params["scale"], c.params["zp"], 8).cpu().numpy()
    np.testing.assert_array_equal(res.quantized.codes, full)
    for o in cs[1:]:
        assert torch.equal(o.U, c.U)
    assert res.output_mse == pytest.approx(ref.output_mse, rel=1e-3)
    with pytest.raises(ValueError):
        run_loopback_calibration(w, shards, quant.QuantConfig())          # per_tensor activations


def test_nccl_world_one(tmp_path):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    script = textwrap.dedent(f"""
        import os, sys, numpy as np, torch
        sys.path.insert(0, {repr(os.getcwd())})
        import torch.distributed as dist
        from paper_2508_07329_b200 import quant
        from paper_2508_07329_b200.dist_calib import quantize_layer_sharded
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="{port}")
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        rng = np.random.default_rng(1)
        w = rng.normal(size=(256, 128)) * 0.05
        x = rng.normal(size=(128, 300))
        cfg = quant.QuantConfig(8, False, quant.PER_TOKEN)
        a = quantize_layer_sharded(w, x, cfg)
        b = quant.quantize_layer(w, x, cfg)
        ok = np.array_equal(a.quantized.codes, b.quantized.codes) and a.smoothing.exponent == b.smoothing.exponent
        dist.destroy_process_group()
        print("EQUAL" if ok else "DIFFERENT")
    """)
    r = subprocess.run([sys.executable, "-c", script], capture_output=True, text=True, timeout=300)
    assert "EQUAL" in r.stdout, r.stdout + r.stderr[-3000:]
