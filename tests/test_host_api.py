"""CPU: host-side logic of the product package (trace model, placement,
formats, config validation) against the reference's golden vectors, and the
C-ABI library's symbol table (loads without a GPU, no compute calls)."""

import re
import struct
from pathlib import Path

import numpy as np
import pytest

from paper_2508_07329_b200 import _lib, formats, placement, quant, trace
from paper_2508_07329_b200.errors import FormatError

ROOT = Path(__file__).resolve().parents[1]


def _gen(seed):
    return trace.generate_trace(trace.GenConfig(layers=32, experts_per_layer=8, top_k=2, n_prefill_tokens=300,
                                                hot_path_prob=0.3, zipf_s=1.2, seed=seed))


def test_generator_matches_reference(golden):
    for j, seed in enumerate((0, 7)):
        np.testing.assert_array_equal(_gen(seed).paths_array(), golden[f"tr{j}_paths"])


def test_generator_golden_snapshot():
    # test_trace.py:79-103 frozen draw
    cfg = trace.GenConfig(layers=3, experts_per_layer=4, top_k=2, n_prefill_tokens=4, n_decode_tokens=3,
                          hot_path_prob=0.5, zipf_s=1.0, seed=123)
    want = [
        (0, "prefill", ((2, 3), (0, 1), (0, 3))),
        (1, "prefill", ((2, 3), (1, 3), (1, 3))),
        (2, "prefill", ((0, 2), (0, 3), (0, 3))),
        (3, "prefill", ((2, 3), (1, 3), (1, 3))),
        (4, "decode", ((0, 2), (0, 3), (0, 3))),
        (5, "decode", ((1, 3), (2, 3), (0, 2))),
        (6, "decode", ((1, 3), (1, 2), (1, 3))),
    ]
    assert [(ev.token_index, ev.phase, ev.path) for ev in trace.generate_trace(cfg).events] == want


def test_stats_and_plans(golden):
    for j, seed in enumerate((0, 7)):
        tr = _gen(seed)
        fq = trace.expert_freq(tr)
        np.testing.assert_array_equal(fq.counts, golden[f"tr{j}_freq"])
        st = trace.path_stats(tr)
        assert len(st.entries) == int(golden[f"tr{j}_stat_n"])
        np.testing.assert_array_equal(np.array([p for p, _ in st.entries[:50]]), golden[f"tr{j}_stat_paths"])
        plans = {"two": placement.plan_two_stage(st, fq, 2, 2), "two23": placement.plan_two_stage(st, fq, 2, 3),
                 "freq": placement.plan_frequency(fq, 128), "path": placement.plan_path(st, 128)}
        for name, plan in plans.items():
            mask = np.zeros((32, 8), dtype=np.int8)
            for layer, r in enumerate(plan.residents):
                mask[layer, sorted(r)] = 1
            np.testing.assert_array_equal(mask, golden[f"tr{j}_{name}_mask"], err_msg=name)
            rep = placement.evaluate_plan(plan, tr)
            np.testing.assert_allclose([rep.mean, rep.std, rep.gap], golden[f"tr{j}_{name}_eval"], rtol=1e-12)
        assert all(len(r) == 4 for r in plans["two"].residents)


def test_trace_and_plan_files(tmp_path):
    tr = _gen(3)
    trace.write_trace(tmp_path / "t.txt", tr)
    back = trace.read_trace(tmp_path / "t.txt")
    assert back.events == tr.events
    plan = placement.plan_two_stage(trace.path_stats(tr), trace.expert_freq(tr), 2, 2)
    placement.write_plan(tmp_path / "p.txt", plan)
    assert placement.read_plan(tmp_path / "p.txt") == plan
    (tmp_path / "bad.txt").write_text("trace layers=2 experts=4 top_k=2\n0 prefill 1,0|2,3\n")
    with pytest.raises(FormatError):
        trace.read_trace(tmp_path / "bad.txt")


def test_moep_formats(golden):
    for bits in (3, 8):
        blob = formats.moep_encode(golden[f"pk{bits}_codes"], golden[f"pk{bits}_scales"], golden[f"pk{bits}_zps"],
                                   bits, "per_output_row", "gpu_int")
        assert blob == golden[f"pk{bits}_blob"].tobytes()
        codes, sc, zp, b, gran = formats.moep_decode(blob)
        np.testing.assert_array_equal(codes, golden[f"pk{bits}_codes"])
        np.testing.assert_array_equal(sc, golden[f"pk{bits}_scales"])
        assert b == bits and gran == "per_output_row"
        # size formula (test_quant.py:521-529)
        r, c = golden[f"pk{bits}_codes"].shape
        assert len(blob) == 20 + 16 * r + (r * c * bits + 7) // 8
    with pytest.raises(ValueError):
        formats.moep_decode(b"XXXX" + b"\0" * 32)


def test_moek_round_trip(tmp_path):
    from paper_2508_07329_b200 import numkit
    a = np.random.default_rng(3).normal(size=(5, 7))
    numkit.write_matrix(tmp_path / "a.mat", a)
    back = numkit.read_matrix(tmp_path / "a.mat")
    np.testing.assert_array_equal(back, a)
    back[0, 0] = 1.0
    raw = (tmp_path / "a.mat").read_bytes()
    assert raw[:4] == b"MOEK" and struct.unpack("<III", raw[4:16]) == (5, 7, 1)
    (tmp_path / "b.mat").write_bytes(raw[:20])
    with pytest.raises(FormatError):
        numkit.read_matrix(tmp_path / "b.mat")


def test_quant_config_and_matrix_validation():
    with pytest.raises(ValueError):
        quant.QuantConfig(bits=1)
    with pytest.raises(ValueError):
        quant.QuantConfig(granularity="per_block")
    assert quant.QuantConfig().qmax == 255
    with pytest.raises(ValueError):
        quant.QuantizedMatrix(np.array([[300]]), [1.0], [0], 8, "per_tensor")
    with pytest.raises(ValueError):
        quant.QuantizedMatrix(np.array([[1], [2]]), [1.0], [0], 8, "per_token")
    q = quant.QuantizedMatrix(np.array([[1, 2]]), [0.5], [1], 8, "per_tensor")
    assert q.group_params()[0].zero_point == 1


def test_library_exports_every_header_symbol():
    header = (ROOT / "include" / "moe_b200.h").read_text()
    declared = set(re.findall(r"^\s*(?:const char\*|uint64_t|int64_t|int|moe_status)\s+(moe_\w+)\s*\(", header, re.M))
    assert declared, "no declarations parsed"
    assert declared == set(_lib.exported_symbols())
    if not _lib.LIB_PATH.exists():
        pytest.skip("library not built (run __graft_entry__.build())")
    lib = _lib.load_library()
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.moe_abi_version() == 1
    assert lib.moe_act_quant_workspace(4, 4, 0) == 16


def test_abi_argument_errors_without_gpu():
    """The C ABI's error contract (status code + thread-local message) for
    invalid arguments: checked before any device work, so it runs here."""
    if not _lib.LIB_PATH.exists():
        pytest.skip("library not built (run __graft_entry__.build())")
    lib = _lib.load_library()
    P = None
    # act_quant: empty matrix, unsupported bits
    D = 16   # dummy (never dereferenced) device addresses: validation runs before any launch
    st = lib.moe_act_quant(D, _lib.DT_BF16, 0, 8, 8, P, P, P, P, _lib.SMOOTH_NONE, P, 8, 0, 1, D, 8, D, D, D, D, P,
                           P, 0, P)
    assert st == _lib.EINVAL and b"non-empty" in lib.moe_last_error()
    st = lib.moe_act_quant(P, _lib.DT_BF16, 4, 8, 8, P, P, P, P, _lib.SMOOTH_NONE, P, 8, 0, 1, D, 8, D, D, D, D, P,
                           P, 0, P)
    assert st == _lib.EINVAL and b"null" in lib.moe_last_error()
    # GEMM: K beyond the exact-int32 bound
    st = lib.moe_w8a8_gemm(1, 4, 40000, 40000, 1, 1, 1, 1, 4, 40000, 1, 1, 1, P, P, P, 1, _lib.EPI_DEQUANT, 1,
                           _lib.DT_F32, 4, P, 0, P, 0, P, P)
    assert st == _lib.EINVAL and b"K too large" in lib.moe_last_error()
    # fused combine needs top-2 rows (M == 2 T)
    st = lib.moe_w8a8_gemm_combine(1, 6, 128, 128, 1, 1, 1, 1, 64, 128, 1, 1, 1, P, P, 1, _lib.EPI_DEQUANT, 16, 64,
                                   1, 1, 4, 16, 64, 16, 1 << 20, P)
    assert st == _lib.EINVAL and b"top-2" in lib.moe_last_error()
    # tuning knobs: query, set/restore, unknown key
    import ctypes
    old = ctypes.c_int64(0)
    assert lib.moe_tune(_lib.TUNE_K1_SMALL_ROWS, -1, ctypes.byref(old)) == _lib.OK and old.value >= 0
    assert lib.moe_tune(99, 1, P) == _lib.EINVAL and b"unknown key" in lib.moe_last_error()
    # rmsnorm: d must be a multiple of 8
    assert lib.moe_rmsnorm_residual(16, P, P, 16, 4, 12, 1e-5, P) == _lib.EINVAL


def test_hostio_split_ends():
    """The serving loop cuts only the first and last batch into chunks
    (multiples of the quantum rows) and returns the callers' outputs."""
    import torch
    from paper_2508_07329_b200.hostio import _split_ends
    xs = [torch.zeros((n, 4)) for n in (16384, 100, 8192)]
    outs = [torch.empty((n, 4)) for n in (16384, 100, 8192)]
    items, final = _split_ends(list(zip(xs, outs)), 4, torch.float32, 4, 1)
    assert [it[0].shape[0] for it in items] == [4096] * 4 + [100] + [2048] * 4
    assert all(a is b for a, b in zip(final, outs))
    assert items[1][1].data_ptr() == outs[0][4096:].data_ptr()          # views into the caller's buffer
    items, _ = _split_ends(list(zip(xs, outs)), 4, torch.float32, 4, 4096)
    assert [it[0].shape[0] for it in items] == [4096] * 4 + [100] + [8192]   # 8192 / 4 < quantum: whole
    items, _ = _split_ends(list(zip(xs, outs)), 4, torch.float32, 1, 1)
    assert len(items) == 3
