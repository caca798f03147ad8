"""Oracle restatement of moekit/numkit.py (TEST INFRASTRUCTURE ONLY).

Validation to float64, the pivot-reporting Cholesky, the SPD inverse built
from two triangular solves, and the MOEK matrix container.
"""

from __future__ import annotations

import math
import struct

import numpy as np
from scipy.linalg import solve_triangular


class OracleNotPD(ArithmeticError):
    """Mirror of errors.NotPositiveDefiniteError (errors.py:15-27)."""

    def __init__(self, pivot: int, value: float):
        super().__init__(f"not positive definite: pivot {pivot} = {value:g}")
        self.pivot = pivot
        self.value = value


def as_f64_matrix(a, name: str = "matrix") -> np.ndarray:
    """numkit.ensure_matrix (numkit.py:36-54): 2-D, non-empty, real, finite,
    C-contiguous float64."""
    arr = np.asarray(a)
    if arr.ndim != 2 or min(arr.shape) < 1:
        raise ValueError(f"{name} must be a non-empty 2-D matrix, got {arr.shape}")
    if arr.dtype.kind not in "fiu":
        raise ValueError(f"{name} must be real-valued")
    arr = np.ascontiguousarray(arr, dtype=np.float64)
    if not np.isfinite(arr).all():
        raise ValueError(f"{name} contains non-finite entries")
    return arr


def check_symmetric(h: np.ndarray, tol_rel: float = 1e-9) -> None:
    """numkit._check_square_symmetric (numkit.py:68-74)."""
    if h.shape[0] != h.shape[1]:
        raise ValueError("matrix must be square")
    tol = tol_rel * max(1.0, float(np.abs(h).max()))
    if float(np.abs(h - h.T).max()) > tol:
        raise ValueError("matrix is not symmetric")


def cholesky_lower(h) -> np.ndarray:
    """Left-looking column Cholesky reporting the failing pivot
    (numkit.py:77-94). Column j: d = h_jj - |L_j,:j|^2, then the sub-column
    is (h_{j+1:,j} - L_{j+1:,:j} L_{j,:j}) / sqrt(d)."""
    h = as_f64_matrix(h, "h")
    check_symmetric(h)
    n = h.shape[0]
    lo = np.zeros((n, n))
    for j in range(n):
        row = lo[j, :j]
        pivot = h[j, j] - row @ row
        if not (math.isfinite(pivot) and pivot > 0.0):
            raise OracleNotPD(j, float(pivot))
        root = math.sqrt(pivot)
        lo[j, j] = root
        if j + 1 < n:
            lo[j + 1:, j] = (h[j + 1:, j] - lo[j + 1:, :j] @ row) / root
    return lo


def spd_inverse(h) -> np.ndarray:
    """numkit.spd_inverse (numkit.py:97-107): two triangular solves against
    the identity, then exact symmetrisation."""
    lo = cholesky_lower(h)
    ident = np.eye(lo.shape[0])
    tmp = solve_triangular(lo, ident, lower=True)
    inv = solve_triangular(lo.T, tmp, lower=False)
    return (inv + inv.T) / 2.0


_MOEK = b"MOEK"
_MOEK_TAGS = {0: np.dtype("<f4"), 1: np.dtype("<f8")}


def moek_bytes(a, dtype: str = "float64") -> bytes:
    """numkit.write_matrix byte layout (numkit.py:110-127): 'MOEK', rows,
    cols, dtype tag (u32 LE each), row-major LE payload."""
    a = as_f64_matrix(a)
    tag = {"float32": 0, "float64": 1}[np.dtype(dtype).name]
    body = np.ascontiguousarray(a, dtype=_MOEK_TAGS[tag]).tobytes()
    return _MOEK + struct.pack("<III", a.shape[0], a.shape[1], tag) + body


def moek_parse(blob: bytes) -> np.ndarray:
    """numkit.read_matrix payload rules (numkit.py:130-157)."""
    if len(blob) < 16 or blob[:4] != _MOEK:
        raise ValueError("bad MOEK header")
    rows, cols, tag = struct.unpack("<III", blob[4:16])
    dt = _MOEK_TAGS[tag]
    if len(blob) - 16 != rows * cols * dt.itemsize:
        raise ValueError("bad MOEK payload size")
    return np.frombuffer(blob, dtype=dt, offset=16).reshape(rows, cols).copy()
