"""ctypes binding of the C ABI in include/moe_b200.h (lib/libmoe_b200.so).

There is deliberately no fallback: if the library is missing or the device
is not an sm_100 part, load() raises and every GPU entry point fails loudly.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import DegenerateHessianError, NotPositiveDefiniteError, QuantizationFailedError

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libmoe_b200.so"
if os.environ.get("MOE_B200_LIB"):     # experiment builds (tools/build_variant.sh); default: the in-tree build
    LIB_PATH = Path(os.environ["MOE_B200_LIB"]).resolve()

OK, EINVAL, ENOTPD, EDEGENERATE, EQUANTFAIL, ECUDA, EUNSUPPORTED = range(7)
DT_F32, DT_F64, DT_BF16, DT_F16, DT_U8, DT_I32 = range(6)
GRAN = {"per_tensor": 0, "per_token": 1, "per_output_row": 2}
SMOOTH_NONE, SMOOTH_DIVIDE, SMOOTH_MULTIPLY = 0, 1, 2
EPI_DEQUANT, EPI_SWIGLU, EPI_ACC_I32 = 0, 1, 2
EPI_FLAG_WCORR = 0x100
EPI_FLAG_WS_ZEROED = 0x200
EPI_FLAG_EXT_READY = 0x400
TUNE_K1_SMALL_ROWS = 1
TUNE_ROUTER_CLUSTER_TILES = 2
TUNE_FUSED_QUANT = 3
TUNE_FUSED_COMBINE = 4
TUNE_K1_TOKENS = 5
TUNE_GPTQ_LANES = 6
TUNE_BAND_MB = 7
ORDER_MAX_ABS, ORDER_SUM_SQUARES = 1, 2

_P, _I64, _I, _D = C.c_void_p, C.c_int64, C.c_int, C.c_double

# name -> (restype, argtypes)
_SIGS = {
    "moe_last_error": (C.c_char_p, []),
    "moe_last_error_detail": (_I, [_P, _P]),
    "moe_abi_version": (_I, []),
    "moe_launch_count": (C.c_uint64, []),
    "moe_device_check": (_I, [_I]),
    "moe_tune": (_I, [_I, _I64, _P]),
    "moe_act_quant_workspace": (_I64, [_I64, _I64, _I]),
    "moe_act_quant": (_I, [_P, _I, _I64, _I64, _I64, _P, _P, _P, _P, _I, _P, _I, _I, _I, _P, _I64, _P, _P,
                           _P, _P, _P, _P, _I64, _P]),
    "moe_act_quant_tokens": (_I, [_P, _I, _I64, _I64, _I64, _I, _P, _P, _P, _P, _P, _I, _I, _P, _I64, _P, _P, _P,
                                  _P, _P]),
    "moe_reciprocal_f64": (_I, [_P, _I64, _P, _P, _P]),
    "moe_dequantize": (_I, [_P, _I64, _I64, _I64, _P, _P, _I, _P, _P]),
    "moe_apply_smoothing": (_I, [_P, _I64, _I64, _P, _I64, _P, _P, _P, _P]),
    "moe_channel_stats": (_I, [_P, _I64, _I64, _I, _P, _P]),
    "moe_w8a8_gemm": (_I, [_P, _I64, _I64, _I64, _P, _P, _P, _P, _I64, _I64, _P, _P, _P, _P, _P, _P, _I, _I,
                           _P, _I, _I64, _P, _I64, _P, _I64, _P, _P]),
    "moe_w8a8_gemm_quant_a_workspace": (_I64, [_I64]),
    "moe_w8a8_gemm_quant_a": (_I, [_P, _I64, _P, _P, _P, _P, _P, _P, _I64, _P, _P, _P, _P, _I64, _I64, _P, _I64,
                                   _I64, _P, _P, _P, _P, _P, _P, _I, _I, _P, _I, _I64, _P, _I64, _P]),
    "moe_w8a8_gemm_combine_workspace": (_I64, [_I64, _I64]),
    "moe_step_init": (_I, [_P, _I64, _P, _I64, _P]),
    "moe_w8a8_gemm_combine": (_I, [_P, _I64, _I64, _I64, _P, _P, _P, _P, _I64, _I64, _P, _P, _P, _P, _P, _I, _I,
                                   _P, _I64, _P, _P, _I64, _P, _I64, _P, _I64, _P]),
    "moe_rmsnorm_residual": (_I, [_P, _P, _P, _P, _I64, _I64, C.c_float, _P]),
    "moe_quant_sq_error": (_I, [_P, _I64, _I64, _P, _I, _P, _P, _P, _P, _I64, _P]),
    "moe_quant_sq_error_workspace": (_I64, [_I64, _I64]),
    "moe_router_gate": (_I, [_P, _I, _I64, _I64, _I64, _P, _P, _I, _I, _P, _P, _P, _P]),
    "moe_router_tc_workspace": (_I64, [_I64]),
    "moe_router_prepare": (_I, [_P, _I, _I64, _P, _P]),
    "moe_router_gate_tc": (_I, [_P, _I64, _I64, _I64, _P, _P, _I, _I, _P, _P, _P, _P]),
    "moe_router_topk": (_I, [_P, _I64, _I, _I, _P, _P, _P]),
    "moe_route_permute_workspace": (_I64, [_I64, _I, _I]),
    "moe_route_permute": (_I, [_P, _P, _I64, _I, _I, _P, _P, _P, _P, _P, _P, _I64, _P]),
    "moe_combine": (_I, [_P, _I, _P, _I64, _I, _I64, _P, _I, _I64, _P]),
    "moe_expert_histogram": (_I, [_P, _I64, _I, _I, _I, _P, _P, _P]),
    "moe_hessian_accum": (_I, [_P, _I, _I64, _I64, _I64, _P, _P, _P, _P, _P]),
    "moe_hessian_finalize": (_I, [_P, _I64, _D, _P, _P]),
    "moe_gptq_workspace": (_I64, [_I64, _I64]),
    "moe_gptq_columns": (_I, [_P, _I64, _I64, _I64, _P, _P, _P, _P, _I, _P, _I64, _P, _I64, _P]),
    "moe_route_keys": (_I, [_P, _I64, _P, _I, _P, _P]),
    "moe_act_quant_dispatch": (_I, [_P, _I, _I64, _I64, _I64, _P, _P, _I, _P, _P, _P, _P, _I, _I, _P, _P, _P, _P,
                                    _P, _I64, _P]),
    "moe_act_quant_given_dev": (_I, [_P, _I, _I64, _P, _I64, _I64, _P, _P, _P, _P, _I, _I, _P, _I64, _P, _P, _P, _P,
                                     _P, _P]),
    "moe_w8a8_gemm_scatter": (_I, [_P, _I64, _I64, _I64, _P, _P, _P, _P, _I64, _I64, _P, _P, _P, _P, _P, _P, _I,
                                   _I, _P, _P, _P, _I, _I64, _P]),
    "moe_block_map": (_I, [_I64, _P, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "moe_ep_peer_plan_size": (_I64, [_I, _I, _I]),
    "moe_rope_bf16": (_I, [_P, _I64, _I, _I, _I64, _P, _P, _P, _P]),
    "moe_ep_peer_plan": (_I, [_P, _I, _I, _I, _P, _I, _I64, _I64, _P, _P, _P]),
    "moe_gather_rows": (_I, [_P, _I64, _P, _I64, _I64, _P, _I64, _P]),
    "moe_ep_pack_params": (_I, [_P, _P, _P, _P, _I64, _P, _P]),
    "moe_ep_unpack_params": (_I, [_P, _P, _I64, _P, _P, _P, _P, _P, _P]),
}

_lib = None


def exported_symbols() -> list[str]:
    return list(_SIGS)


def load_library():
    """dlopen the library and bind every declared symbol (works without a GPU)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"CUDA library {LIB_PATH} is missing; build it with `python -m paper_2508_07329_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


_checked = False


def load():
    """Library + device check: the entry point every GPU op goes through."""
    global _checked
    lib = load_library()
    if not _checked:
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2508_07329_b200 needs a CUDA device (sm_100a); no CPU fallback exists")
        dev = torch.cuda.current_device()
        st = lib.moe_device_check(dev)
        if st != OK:
            raise RuntimeError(f"device check failed: {lib.moe_last_error().decode()}")
        _checked = True
    return lib


def check(status: int, what: str = "") -> None:
    if status == OK:
        return
    msg = _lib.moe_last_error().decode() if _lib is not None else "unknown error"
    if what:
        msg = f"{what}: {msg}"
    if status == EINVAL:
        raise ValueError(msg)
    if status == ENOTPD:
        piv, val = C.c_int64(-1), C.c_double(float("nan"))
        if _lib is not None:
            _lib.moe_last_error_detail(C.byref(piv), C.byref(val))
        raise NotPositiveDefiniteError(int(piv.value), float(val.value))
    if status == EDEGENERATE:
        raise DegenerateHessianError(msg)
    if status == EQUANTFAIL:
        raise QuantizationFailedError(msg)
    raise RuntimeError(msg)


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t) -> int | None:
    """Device pointer of a tensor (None for None)."""
    return None if t is None else int(t.data_ptr())


def call(name: str, *args, what: str | None = None):
    lib = load()
    st = getattr(lib, name)(*args)
    check(st, what or name)
    if _SYNC:
        import torch
        try:
            torch.cuda.synchronize()
        except RuntimeError as exc:
            raise RuntimeError(f"{name}: device error after launch: {exc}") from None


_SYNC = os.environ.get("MOE_B200_SYNC", "0") == "1"   # debug: synchronize after every entry point


def tune(key: int, value: int = -1) -> int:
    """Set a kernel-selection knob (``moe_tune``); returns the previous
    value (value < 0 only queries). Results never depend on the knobs."""
    lib = load_library()
    old = C.c_int64(0)
    check(lib.moe_tune(key, value, C.byref(old)), "moe_tune")
    return int(old.value)


class tuned:
    """Context manager: ``with tuned(TUNE_K1_SMALL_ROWS, 0): ...``."""

    def __init__(self, key: int, value: int):
        self.key, self.value = key, value

    def __enter__(self):
        self.old = tune(self.key, self.value)
        return self

    def __exit__(self, *exc):
        tune(self.key, self.old)
