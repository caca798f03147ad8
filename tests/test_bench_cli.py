"""bench.py contract on CPU: the reference arm prints one JSON line with the
driver's keys (value, e2e with zero copy bytes, cpu_baseline describing the
run) for the C4 layer and for the C5 stack, and a multi-GPU request that the
machine cannot serve fails loudly instead of measuring one GPU."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=600):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=timeout, cwd=ROOT)


@pytest.mark.parametrize("layers", [1, 32])
def test_reference_arm_line(layers):
    r = _run("--impl", "reference", "--steps", "1", "--warmup", "0", "--cpu-tokens", "4", "--layers", str(layers))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["runs"] == d["steps"] == 1 and d["cpu_baseline"]["warmup_runs"] == d["warmup"] == 0
    assert d["config"]["layers"] == layers and d["unit"] == "tokens/s"


def test_multi_gpu_request_fails_loudly():
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("machine has 2+ GPUs")
    r = _run("--gpus", "2", "--steps", "1", "--warmup", "3", timeout=300)
    assert r.returncode != 0
    assert "requested but only" in r.stderr
    assert not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
