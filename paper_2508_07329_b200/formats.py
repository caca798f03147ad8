"""On-disk formats of the reference and their zero-copy path into HBM.

* MOEK matrix container (numkit.py:12-14, 110-157): 16-byte header
  ``b"MOEK" | rows u32 | cols u32 | tag u32`` (tag 0 = f32, 1 = f64) then
  the row-major little-endian payload.
* MOEP packed expert (quant.py:59-61, 493-571): 20-byte header
  ``<4sBBBBIII`` = magic, version, target, bits, granularity, rows, cols,
  groups; ``gpu_int`` continues with (scale, zero_point) float64 pairs and
  LSB-first bit-packed codes, ``cpu_fp`` with a float32 payload. For 8-bit
  codes the code stream IS the row-major u8 matrix, so ``moep_to_device``
  uploads it without any repacking.
* result.json + codes.mat layer results (quant.py:574-610).
"""

from __future__ import annotations

import json
import struct
from pathlib import Path

import numpy as np

from .errors import FormatError

_MOEK_MAGIC = b"MOEK"
_MOEK_HEAD = struct.Struct("<4sIII")
_MOEK_DT = (np.dtype("<f4"), np.dtype("<f8"))

_MOEP_MAGIC = b"MOEP"
_MOEP_HEAD = struct.Struct("<4sBBBBIII")
_MOEP_VERSION = 1
PACK_TARGETS = ("cpu_fp", "gpu_int")
GRANULARITIES = ("per_tensor", "per_token", "per_output_row")


# ── MOEK ──────────────────────────────────────────────────────────────────
def moek_encode(a, dtype: str = "float64") -> bytes:
    from .numkit import ensure_matrix
    if hasattr(a, "detach"):
        a = a.detach().cpu().numpy()
    a = ensure_matrix(a, "matrix")
    kind = np.dtype(dtype).name
    if kind not in ("float32", "float64"):
        raise ValueError(f"unsupported dtype {dtype!r}, expected float32 or float64")
    tag = 0 if kind == "float32" else 1
    body = np.ascontiguousarray(a, dtype=_MOEK_DT[tag])
    if not np.isfinite(body).all():
        raise ValueError("matrix is not representable at the requested precision")
    return _MOEK_HEAD.pack(_MOEK_MAGIC, a.shape[0], a.shape[1], tag) + body.tobytes()


def moek_decode(blob: bytes, where: str = "<bytes>") -> np.ndarray:
    if len(blob) < _MOEK_HEAD.size:
        raise FormatError(f"{where}: truncated header ({len(blob)} bytes)")
    magic, rows, cols, tag = _MOEK_HEAD.unpack_from(blob)
    if magic != _MOEK_MAGIC:
        raise FormatError(f"{where}: bad magic {magic!r}")
    if tag > 1:
        raise FormatError(f"{where}: unknown dtype tag {tag}")
    if rows == 0 or cols == 0:
        raise FormatError(f"{where}: empty matrix {rows}x{cols}")
    dt = _MOEK_DT[tag]
    need = rows * cols * dt.itemsize
    if len(blob) - _MOEK_HEAD.size != need:
        raise FormatError(f"{where}: payload is {len(blob) - _MOEK_HEAD.size} bytes, expected {need}")
    arr = np.frombuffer(blob, dtype=dt, offset=_MOEK_HEAD.size).reshape(rows, cols)
    if not np.isfinite(arr).all():
        raise FormatError(f"{where}: payload contains non-finite entries")
    return np.array(arr)  # owned, writable


# ── MOEP ──────────────────────────────────────────────────────────────────
def _bitpack(codes: np.ndarray, bits: int) -> bytes:
    if bits == 8:
        return np.ascontiguousarray(codes, dtype=np.uint8).tobytes()
    flat = np.ascontiguousarray(codes, dtype=np.uint32).ravel()
    planes = ((flat[:, None] >> np.arange(bits, dtype=np.uint32)) & 1).astype(np.uint8)
    return np.packbits(planes.ravel(), bitorder="little").tobytes()


def _bitunpack(buf: bytes, count: int, bits: int) -> np.ndarray:
    if bits == 8:
        return np.frombuffer(buf, dtype=np.uint8, count=count).astype(np.int32)
    raw = np.unpackbits(np.frombuffer(buf, dtype=np.uint8), bitorder="little", count=count * bits)
    return (raw.reshape(count, bits).astype(np.int32) << np.arange(bits, dtype=np.int32)).sum(axis=1)


def moep_encode(codes, scales, zero_points, bits: int, granularity: str, target: str,
                dequantized: np.ndarray | None = None) -> bytes:
    if target not in PACK_TARGETS:
        raise ValueError(f"unknown pack target {target!r}")
    codes = np.asarray(codes)
    scales = np.asarray(scales, dtype=np.float64).ravel()
    head = _MOEP_HEAD.pack(_MOEP_MAGIC, _MOEP_VERSION, PACK_TARGETS.index(target), bits,
                           GRANULARITIES.index(granularity), codes.shape[0], codes.shape[1], scales.shape[0])
    if target == "cpu_fp":
        return head + np.ascontiguousarray(dequantized, dtype="<f4").tobytes()
    params = np.stack([scales, np.asarray(zero_points, dtype=np.float64).ravel()], axis=1).astype("<f8")
    return head + params.tobytes() + _bitpack(codes, bits)


def moep_header(blob: bytes) -> dict:
    if len(blob) < _MOEP_HEAD.size:
        raise ValueError("not a packed expert blob")
    magic, ver, tgt, bits, gran, rows, cols, groups = _MOEP_HEAD.unpack_from(blob)
    if magic != _MOEP_MAGIC or ver != _MOEP_VERSION:
        raise ValueError("not a packed expert blob")
    return {"target": PACK_TARGETS[tgt], "bits": bits, "granularity": GRANULARITIES[gran],
            "rows": rows, "cols": cols, "groups": groups}


def moep_decode(blob: bytes):
    """-> float32 matrix (cpu_fp) or (codes int32, scales, zps, bits, granularity)."""
    h = moep_header(blob)
    body = blob[_MOEP_HEAD.size:]
    rows, cols = h["rows"], h["cols"]
    if h["target"] == "cpu_fp":
        return np.frombuffer(body, dtype="<f4", count=rows * cols).reshape(rows, cols).copy()
    params = np.frombuffer(body, dtype="<f8", count=2 * h["groups"]).reshape(-1, 2)
    codes = _bitunpack(body[16 * h["groups"]:], rows * cols, h["bits"]).reshape(rows, cols)
    return codes, params[:, 0].copy(), params[:, 1].astype(np.int32), h["bits"], h["granularity"]


def moep_to_device(blob: bytes, device="cuda"):
    """Upload a gpu_int MOEP blob into device tensors for the W8A8 GEMM.
    8-bit payloads are copied straight from the blob bytes (no repacking)."""
    import torch
    h = moep_header(blob)
    if h["target"] != "gpu_int":
        raise ValueError("only gpu_int blobs carry integer codes")
    body = memoryview(blob)[_MOEP_HEAD.size:]
    g = h["groups"]
    params = np.frombuffer(body[:16 * g], dtype="<f8").reshape(g, 2)
    if h["bits"] == 8:
        codes = torch.frombuffer(bytearray(body[16 * g:16 * g + h["rows"] * h["cols"]]), dtype=torch.uint8)
        codes = codes.view(h["rows"], h["cols"]).to(device)
    else:
        codes = torch.from_numpy(_bitunpack(bytes(body[16 * g:]), h["rows"] * h["cols"], h["bits"])
                                 .astype(np.uint8).reshape(h["rows"], h["cols"])).to(device)
    scale = torch.from_numpy(params[:, 0].copy()).to(device)
    zp = torch.from_numpy(params[:, 1].astype(np.int32)).to(device)
    return {"codes": codes, "scale": scale, "zp": zp, "bits": h["bits"], "granularity": h["granularity"]}


# ── layer results ─────────────────────────────────────────────────────────
RESULT_KEYS = ("exponent", "factors", "bits", "mse", "rtn_mse", "ordering", "scales", "zero_points",
               "granularity", "smoothing_loss")


def write_layer_result(out_dir, doc: dict, codes: np.ndarray) -> None:
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    (out / "codes.mat").write_bytes(moek_encode(np.asarray(codes, dtype=np.float64)))
    with open(out / "result.json", "w", encoding="utf-8") as fh:
        json.dump({k: doc[k] for k in RESULT_KEYS}, fh, indent=2)
        fh.write("\n")


def read_layer_result(out_dir):
    out = Path(out_dir)
    doc = json.loads((out / "result.json").read_text(encoding="utf-8"))
    codes = moek_decode((out / "codes.mat").read_bytes(), str(out / "codes.mat")).astype(np.int32)
    return codes, doc
