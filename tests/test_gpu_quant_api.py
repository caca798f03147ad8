"""GPU: the moekit-compatible quantizer API (paper_2508_07329_b200.quant),
run through the CUDA kernels, against the unmodified reference's golden
vectors and the reference test suite's own known answers."""

import math

import numpy as np
import pytest

from oracle import quant_ref as Q
from paper_2508_07329_b200 import numkit, quant
from paper_2508_07329_b200.errors import DegenerateHessianError, NotPositiveDefiniteError, QuantizationFailedError
from paper_2508_07329_b200.quant import PER_OUTPUT_ROW, PER_TOKEN, QuantConfig

pytestmark = pytest.mark.gpu
GRANS = ("per_tensor", "per_token", "per_output_row")


def test_rtn_golden(cuda, golden):
    for i in range(int(golden["rtn_ncases"])):
        bits, sym, gran = golden[f"rtn{i}_cfg"]
        q = quant.rtn_quantize(golden[f"rtn{i}_x"], QuantConfig(int(bits), bool(sym), GRANS[int(gran)]))
        np.testing.assert_array_equal(q.codes, golden[f"rtn{i}_codes"])
        np.testing.assert_array_equal(q.scales, golden[f"rtn{i}_scales"])
        np.testing.assert_array_equal(q.zero_points, golden[f"rtn{i}_zps"])


def test_rtn_hand_cases(cuda):
    q = quant.rtn_quantize(np.array([[-1.0, 0.0, 3.0]]), QuantConfig(bits=8))
    assert q.scales[0] == pytest.approx(4.0 / 255.0) and q.zero_points[0] == 64
    assert q.codes[0, 0] == 0 and q.codes[0, 2] == 255
    q = quant.rtn_quantize(np.full((2, 3), 5.0), QuantConfig(bits=8))
    assert q.scales[0] == quant.SCALE_FLOOR
    q = quant.rtn_quantize(np.zeros((2, 3)), QuantConfig(bits=8))
    np.testing.assert_array_equal(quant.dequantize(q), np.zeros((2, 3)))
    rng = np.random.default_rng(5)
    for bits in (2, 4, 8):
        x = rng.normal(size=(6, 40))
        q = quant.rtn_quantize(x, QuantConfig(bits=bits))
        assert np.abs(quant.dequantize(q) - x).max() <= 0.5 * q.scales[0] + 1e-12


def test_quant_loss_and_search_golden(cuda, golden):
    for i in range(4):
        c = QuantConfig(8, False, GRANS[int(golden[f"ql{i}_gran"])])
        w, x, f = golden[f"ql{i}_w"], golden[f"ql{i}_x"], golden[f"ql{i}_f"]
        assert quant.quant_loss(w, x, f, c) == pytest.approx(float(golden[f"ql{i}_loss"]), rel=1e-9)
        sm = quant.search_smoothing(w, x, c)
        assert sm.exponent == float(golden[f"ss{i}_exp"])
        assert sm.loss == pytest.approx(float(golden[f"ss{i}_loss"]), rel=1e-9)


def test_search_smoothing_tie_and_validation(cuda):
    w = np.array([[0.3, -0.7], [1.1, 0.2]])
    assert quant.search_smoothing(w, np.ones((2, 9)), QuantConfig(bits=8)).exponent == 0.0
    with pytest.raises(ValueError):
        quant.search_smoothing(w, np.ones((2, 9)), QuantConfig(bits=8), grid_steps=1)
    with pytest.raises(ValueError):
        quant.quant_loss(w, np.ones((3, 9)), [1, 1], QuantConfig())
    with pytest.raises(ValueError):
        quant.apply_smoothing(w, np.ones((2, 4)), [1.0, -1.0])


def test_criterion_02_search_beats_identity(cuda):
    """test_acceptance.py:73-89 on the device path (25 seeds)."""
    cfg = QuantConfig(bits=8)
    strict = 0
    for i in range(25):
        rng = np.random.default_rng(1000 + i)
        w = rng.normal(size=(8, 16))
        x = rng.normal(size=(16, 64))
        x[3] *= 100.0
        best = quant.search_smoothing(w, x, cfg)
        ident = quant.quant_loss(w, x, np.ones(16), cfg)
        assert best.loss <= ident
        strict += best.loss < ident
    assert strict >= 23


def test_build_hessian_golden(cuda, golden):
    np.testing.assert_allclose(quant.build_hessian(golden["hs_x"]), golden["hs_h"], rtol=1e-12)
    with pytest.raises(DegenerateHessianError):
        quant.build_hessian(np.zeros((4, 16)))
    with pytest.raises(ValueError):
        quant.build_hessian(np.ones((2, 4)), damping_fraction=-0.1)


def test_inverse_factor_and_retries(cuda, golden):
    np.testing.assert_allclose(quant._inverse_upper_factor(golden["hs_h"]), golden["hs_u"], rtol=1e-8, atol=1e-12)
    v = np.array([[1.0], [2.0], [3.0]])
    assert np.isfinite(quant._inverse_upper_factor(v @ v.T)).all()
    with pytest.raises(QuantizationFailedError):
        quant._inverse_upper_factor(-np.eye(3))
    with pytest.raises(NotPositiveDefiniteError) as ei:
        numkit.cholesky(np.array([[1.0, 2.0], [2.0, 1.0]]))
    assert ei.value.pivot == 1 and ei.value.value == pytest.approx(-3.0)
    np.testing.assert_allclose(numkit.cholesky(np.array([[4.0, 2.0], [2.0, 5.0]])), [[2, 0], [1, 2]], atol=1e-14)


def test_hessian_quantize_golden(cuda, golden):
    for bits in (3, 4, 8):
        q = quant.hessian_quantize(golden["hs_w"], golden["hs_h"], QuantConfig(bits=bits))
        np.testing.assert_array_equal(q.codes, golden[f"hq{bits}_codes"])
        np.testing.assert_array_equal(q.scales, golden[f"hq{bits}_scales"])
    q = quant.hessian_quantize(golden["hs_w"], golden["hs_h"], QuantConfig(bits=4), order=golden["hq_order"])
    np.testing.assert_array_equal(q.codes, golden["hqo_codes"])


def test_hessian_quantize_diagonal_is_rtn(cuda):
    rng = np.random.default_rng(17)
    w = rng.normal(size=(6, 10))
    for c in (0.5, 1.0, 8.0):
        q = quant.hessian_quantize(w, c * np.eye(10), QuantConfig(bits=4))
        r = quant.rtn_quantize(w, QuantConfig(bits=4, granularity=PER_OUTPUT_ROW))
        np.testing.assert_array_equal(q.codes, r.codes)


def _round_ref(v):
    return int(math.copysign(math.floor(abs(v) + 0.5), v))


def test_hessian_quantize_matches_obs_reference(cuda):
    """test_quant.py:329-365's naive re-inversion reference."""
    for seed in range(4):
        rng = np.random.default_rng(200 + seed)
        w = rng.normal(size=(3, 5))
        h = quant.build_hessian(rng.normal(size=(5, 40)))
        q = quant.hessian_quantize(w, h, QuantConfig(bits=4))
        lo, hi = w.min(axis=1), w.max(axis=1)
        scale = np.maximum((hi - lo) / 15, quant.SCALE_FLOOR)
        zp = np.clip(np.array([_round_ref(v) for v in -lo / scale]), 0, 15)
        work = w.copy()
        codes = np.empty(w.shape, dtype=np.int64)
        for i in range(5):
            hinv = np.linalg.inv(h[i:, i:])
            c = np.clip(np.array([_round_ref(v) for v in work[:, i] / scale]) + zp, 0, 15)
            codes[:, i] = c
            err = (work[:, i] - (c - zp) * scale) / hinv[0, 0]
            work[:, i + 1:] -= np.outer(err, hinv[0, 1:])
        np.testing.assert_array_equal(q.codes, codes)


def test_quantize_layer_golden(cuda, golden):
    for j, ordering in enumerate(("none", "max_abs")):
        res = quant.quantize_layer(golden["ly_w"], golden["ly_x"], QuantConfig(8, False, PER_TOKEN),
                                   ordering=ordering)
        assert res.smoothing.exponent == float(golden[f"ly{j}_exp"])
        np.testing.assert_array_equal(res.quantized.codes, golden[f"ly{j}_codes"])
        np.testing.assert_array_equal(res.quantized.scales, golden[f"ly{j}_scales"])
        assert res.output_mse == pytest.approx(float(golden[f"ly{j}_mse"]), rel=1e-9)
        assert res.rtn_baseline_mse == pytest.approx(float(golden[f"ly{j}_rtn_mse"]), rel=1e-9)


def test_quantize_layer_behaviour(cuda, tmp_path):
    rng = np.random.default_rng(21)
    w = rng.normal(size=(8, 16))
    x = rng.normal(size=(16, 64))
    x[5] *= 100.0
    res = quant.quantize_layer(w, x, QuantConfig(bits=4))
    assert res.output_mse < res.rtn_baseline_mse
    with pytest.warns(UserWarning, match="calibration tokens"):
        quant.quantize_layer(w[:, :4], rng.normal(size=(4, 5)), QuantConfig(bits=8))
    with pytest.raises(DegenerateHessianError):
        quant.quantize_layer(np.ones((2, 3)), np.zeros((3, 16)), QuantConfig(bits=8))
    res = quant.quantize_layer(w, x, QuantConfig(bits=4), ordering="sum_squares")
    quant.save_layer_result(res, tmp_path)
    q, doc = quant.load_layer_result(tmp_path)
    np.testing.assert_array_equal(q.codes, res.quantized.codes)
    assert doc["ordering"] == res.ordering.tolist()


def test_apply_smoothing_and_pack(cuda):
    rng = np.random.default_rng(8)
    w, x, s = rng.normal(size=(4, 6)), rng.normal(size=(6, 10)), np.exp(rng.normal(size=6))
    ws, xs = quant.apply_smoothing(w, x, s)
    np.testing.assert_array_equal(ws, w * s[None, :])
    np.testing.assert_array_equal(xs, x / s[:, None])
    q = quant.rtn_quantize(rng.normal(size=(4, 10)), QuantConfig(bits=4, granularity=PER_OUTPUT_ROW))
    back = quant.unpack_expert(quant.precision_pack(q, quant.TARGET_GPU_INT))
    np.testing.assert_array_equal(back.codes, q.codes)
    cpu = quant.unpack_expert(quant.precision_pack(q, quant.TARGET_CPU_FP))
    np.testing.assert_allclose(cpu, quant.dequantize(q), rtol=1e-6)


def test_channel_order(cuda):
    x = np.array([[1.0, -1.0], [3.0, 0.0], [-2.0, 2.0]])
    np.testing.assert_array_equal(quant.channel_order(x, "max_abs"), [1, 2, 0])
    np.testing.assert_array_equal(quant.channel_order(x, "sum_squares"), [1, 2, 0])
    np.testing.assert_array_equal(quant.channel_order(np.array([[2.0], [2.0], [1.0]]), "max_abs"), [0, 1, 2])
    rng = np.random.default_rng(2)
    xr = rng.normal(size=(300, 50))
    for strat in ("max_abs", "sum_squares"):
        np.testing.assert_array_equal(quant.channel_order(xr, strat), Q.channel_order(xr, strat))
