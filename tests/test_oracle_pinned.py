"""CPU: the oracle restatement must reproduce the unmodified reference's
golden vectors (tests/golden/make_golden.py) bit-for-bit where the reference
is integer/byte work and to 1e-12 where it is float64 arithmetic."""

import numpy as np
import pytest

from oracle import moe_ref as M
from oracle import numkit_ref as N
from oracle import quant_ref as Q
from oracle import routing_ref as R

GRANS = ("per_tensor", "per_token", "per_output_row")


def test_rounding_kat(golden):
    np.testing.assert_array_equal(Q.rha(golden["rha_in"]), golden["rha_out"])
    # test_quant.py:32-35 known answers
    np.testing.assert_array_equal(Q.rha(np.array([0.5, -0.5, 1.5, 2.5, -2.5, 0.49, -0.49, 3.0])),
                                  [1, -1, 2, 3, -3, 0, 0, 3])
    assert Q.rha(np.array([0.49999999999999994]))[0] == 1.0


def test_rtn_cases(golden):
    for i in range(int(golden["rtn_ncases"])):
        bits, sym, gran = golden[f"rtn{i}_cfg"]
        c = Q.cfg(int(bits), bool(sym), GRANS[int(gran)])
        codes, s, z = Q.rtn(golden[f"rtn{i}_x"], c)
        np.testing.assert_array_equal(codes, golden[f"rtn{i}_codes"])
        np.testing.assert_array_equal(s, golden[f"rtn{i}_scales"])
        np.testing.assert_array_equal(z, golden[f"rtn{i}_zps"])


def test_rtn_hand_cases():
    # test_quant.py:44-52 and :74-78
    codes, s, z = Q.rtn(np.array([[-1.0, 0.0, 3.0]]), Q.cfg(8))
    assert s[0] == pytest.approx(4.0 / 255.0) and z[0] == 64
    assert codes[0, 0] == 0 and codes[0, 2] == 255
    codes, s, z = Q.rtn(np.array([[0.0, 1.0]]), Q.cfg(8))
    assert z[0] == 0 and list(codes[0]) == [0, 255]
    _, s, z = Q.rtn(np.array([[-2.0, 1.0, 0.5]]), Q.cfg(8, True))
    assert z[0] == 128 and s[0] == pytest.approx(2.0 / 127.0)


def test_k1_semantics(golden):
    codes, s, z, rs = M.quantize_rows(golden["k1_x_bf16"], golden["k1_smooth"])
    np.testing.assert_array_equal(codes, golden["k1_codes"])
    np.testing.assert_array_equal(s, golden["k1_scales"])
    np.testing.assert_array_equal(z, golden["k1_zps"])
    np.testing.assert_array_equal(rs, golden["k1_codes"].astype(np.int64).sum(axis=1))


def test_quant_loss_and_search(golden):
    for i in range(4):
        c = Q.cfg(8, False, GRANS[int(golden[f"ql{i}_gran"])])
        w, x, f = golden[f"ql{i}_w"], golden[f"ql{i}_x"], golden[f"ql{i}_f"]
        assert Q.quant_loss(w, x, f, c) == pytest.approx(float(golden[f"ql{i}_loss"]), rel=1e-12)
        e, fac, loss = Q.search_smoothing(w, x, c)
        assert e == float(golden[f"ss{i}_exp"])
        assert loss == pytest.approx(float(golden[f"ss{i}_loss"]), rel=1e-12)
        np.testing.assert_array_equal(fac, golden[f"ss{i}_factors"])


def test_hessian_factor_gptq(golden):
    h = Q.build_hessian(golden["hs_x"])
    np.testing.assert_allclose(h, golden["hs_h"], rtol=1e-12)
    u = Q.inverse_upper_factor(golden["hs_h"])
    np.testing.assert_allclose(u, golden["hs_u"], rtol=1e-10, atol=1e-14)
    for bits in (3, 4, 8):
        codes, s, z = Q.hessian_quantize(golden["hs_w"], golden["hs_h"], Q.cfg(bits))
        np.testing.assert_array_equal(codes, golden[f"hq{bits}_codes"])
        np.testing.assert_array_equal(s, golden[f"hq{bits}_scales"])
        np.testing.assert_array_equal(z, golden[f"hq{bits}_zps"])
    codes, _, _ = Q.hessian_quantize(golden["hs_w"], golden["hs_h"], Q.cfg(4), golden["hq_order"])
    np.testing.assert_array_equal(codes, golden["hqo_codes"])


def test_quantize_layer(golden):
    for j, ordering in enumerate(("none", "max_abs")):
        res = Q.quantize_layer(golden["ly_w"], golden["ly_x"], Q.cfg(8, False, "per_token"),
                               ordering=ordering)
        np.testing.assert_array_equal(res["codes"], golden[f"ly{j}_codes"])
        np.testing.assert_array_equal(res["scales"], golden[f"ly{j}_scales"])
        assert res["exponent"] == float(golden[f"ly{j}_exp"])
        assert res["output_mse"] == pytest.approx(float(golden[f"ly{j}_mse"]), rel=1e-10)
        assert res["rtn_baseline_mse"] == pytest.approx(float(golden[f"ly{j}_rtn_mse"]), rel=1e-10)


def test_cholesky_kat():
    # test_numkit.py:64-68 and the failing-pivot case :79-84
    np.testing.assert_allclose(N.cholesky_lower(np.array([[4.0, 2.0], [2.0, 5.0]])),
                               [[2.0, 0.0], [1.0, 2.0]], atol=1e-14)
    with pytest.raises(N.OracleNotPD) as ei:
        N.cholesky_lower(np.array([[1.0, 2.0], [2.0, 1.0]]))
    assert ei.value.pivot == 1 and ei.value.value == pytest.approx(-3.0)


def test_routing_stats_and_placement(golden):
    for j in range(2):
        paths = golden[f"tr{j}_paths"]
        np.testing.assert_array_equal(R.expert_freq(paths, 8), golden[f"tr{j}_freq"])
        st = R.path_stats(paths)
        assert len(st) == int(golden[f"tr{j}_stat_n"])
        top = st[:50]
        np.testing.assert_array_equal(np.array([p for p, _ in top]), golden[f"tr{j}_stat_paths"])
        np.testing.assert_array_equal(np.array([c for _, c in top]), golden[f"tr{j}_stat_counts"])
        counts = golden[f"tr{j}_freq"]
        plans = {"two": R.plan_two_stage(st, counts, 2, 2),
                 "two23": R.plan_two_stage(st, counts, 2, 3),
                 "freq": R.plan_frequency(counts, 128),
                 "path": R.plan_path(st, 32, 8, 128)}
        for name, res in plans.items():
            mask = np.zeros((32, 8), dtype=np.int8)
            for layer, r in enumerate(res):
                mask[layer, sorted(r)] = 1
            np.testing.assert_array_equal(mask, golden[f"tr{j}_{name}_mask"])
            _, mean, std, gap = R.evaluate_plan(res, paths, 2)
            np.testing.assert_allclose([mean, std, gap], golden[f"tr{j}_{name}_eval"], rtol=1e-12)


def test_pack_layout(golden):
    for bits in (3, 8):
        blob = Q.pack_gpu_int(golden[f"pk{bits}_codes"], golden[f"pk{bits}_scales"],
                              golden[f"pk{bits}_zps"], bits, "per_output_row")
        assert blob == golden[f"pk{bits}_blob"].tobytes()
    # 8-bit payload is the raw row-major u8 code matrix
    c = golden["pk8_codes"]
    body = golden["pk8_blob"].tobytes()[20 + 16 * c.shape[0]:]
    assert body == c.astype(np.uint8).tobytes()


def test_moe_oracle_small_consistency():
    """The exact-accumulator MoE oracle and the reference-style fake-quant
    path must agree to float64 rounding (they differ only in summation
    order)."""
    rng = np.random.default_rng(0)
    t, d, ffn, e = 24, 32, 48, 4
    x = rng.normal(size=(t, d))
    wg = rng.normal(size=(e, d)) / np.sqrt(d)
    experts, deq = [], []
    for _ in range(e):
        ex = {"s13": np.exp(rng.normal(size=d) * 0.3), "s2": np.exp(rng.normal(size=ffn) * 0.3)}
        dq = {"s13": ex["s13"], "s2": ex["s2"]}
        for name, shape, s in (("w1", (ffn, d), "s13"), ("w3", (ffn, d), "s13"), ("w2", (d, ffn), "s2")):
            w = rng.normal(size=shape) * 0.05 * ex[s][None, :]
            c, sc, z = M.quantize_weight_rows(w)
            ex[f"{name}_codes"], ex[f"{name}_scale"], ex[f"{name}_zp"] = c, sc, z
            dq[name] = Q.dequant(c, sc, z, "per_output_row")
        experts.append(ex)
        deq.append(dq)
    out, idx, w = M.moe_forward(x, wg, experts)
    ref = M.moe_forward_fakequant(x, wg, deq)
    np.testing.assert_allclose(out, ref, rtol=1e-9, atol=1e-12)
    # permutation invariants
    offs, tok, slot, pos = M.permute(idx, e)
    assert offs[-1] == t * 2
    np.testing.assert_array_equal(idx[tok, slot], np.repeat(np.arange(e), np.diff(offs)))
    assert (np.diff(tok[offs[0]:offs[1]]) >= 0).all()
