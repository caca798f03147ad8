"""Drop-in for moekit.numkit (numkit.py:36-157) on the B200.

``ensure_matrix`` keeps the reference's validation contract (2-D, non-empty,
real, finite -> C-contiguous float64) for host inputs. The factorizations
run on the GPU through cuSOLVER (torch.linalg, a library call off the hot
loop) with the reference's failure reporting: the failing pivot index is
carried by NotPositiveDefiniteError. MOEK matrix files are a host I/O
format and are read/written on the host.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .errors import NotPositiveDefiniteError

SYMMETRY_TOL = 1e-9


def ensure_matrix(a, name: str = "matrix") -> np.ndarray:
    """Validate a host matrix (numkit.py:36-54)."""
    out = np.asarray(a)
    if out.ndim != 2:
        raise ValueError(f"{name} must be 2-D, got shape {out.shape}")
    if out.shape[0] < 1 or out.shape[1] < 1:
        raise ValueError(f"{name} must be non-empty, got shape {out.shape}")
    if out.dtype.kind not in "fiu":
        raise ValueError(f"{name} must be real-valued, got dtype {out.dtype}")
    out = np.ascontiguousarray(out, dtype=np.float64)
    if not np.isfinite(out).all():
        raise ValueError(f"{name} contains non-finite entries")
    return out


def to_device(a, name: str = "matrix", dtype=torch.float64) -> torch.Tensor:
    """Host matrix (validated) or CUDA tensor -> CUDA tensor of ``dtype``."""
    _lib.load()
    if isinstance(a, torch.Tensor):
        if a.dim() != 2 or min(a.shape) < 1:
            raise ValueError(f"{name} must be a non-empty 2-D matrix, got shape {tuple(a.shape)}")
        t = a if a.is_cuda else a.cuda()
        if not torch.isfinite(t).all():
            raise ValueError(f"{name} contains non-finite entries")
        return t.to(dtype).contiguous()
    return torch.from_numpy(ensure_matrix(a, name)).cuda().to(dtype)


def _check_symmetric(h: torch.Tensor, name: str) -> None:
    if h.shape[0] != h.shape[1]:
        raise ValueError(f"{name} must be square, got shape {tuple(h.shape)}")
    tol = SYMMETRY_TOL * max(1.0, float(h.abs().max()))
    asym = float((h - h.T).abs().max())
    if asym > tol:
        raise ValueError(f"{name} is not symmetric (max asymmetry {asym:g})")


def cholesky_device(h: torch.Tensor) -> torch.Tensor:
    """Lower Cholesky factor on the GPU; NotPositiveDefiniteError(pivot)."""
    low, info = torch.linalg.cholesky_ex(h)
    code = int(info.item())
    if code != 0:
        pivot = code - 1
        d = h[pivot, pivot] - (low[pivot, :pivot] @ low[pivot, :pivot] if pivot else 0.0)
        raise NotPositiveDefiniteError(pivot, float(d))
    return low


def cholesky(h):
    """numkit.cholesky (numkit.py:77-94) computed on the GPU."""
    hd = to_device(h, "h")
    _check_symmetric(hd, "h")
    low = cholesky_device(hd)
    return low.cpu().numpy() if not isinstance(h, torch.Tensor) else low


def spd_inverse_device(h: torch.Tensor) -> torch.Tensor:
    low = cholesky_device(h)
    inv = torch.cholesky_inverse(low)
    return (inv + inv.T) / 2.0


def spd_inverse(h):
    """numkit.spd_inverse (numkit.py:97-107) on the GPU, exactly symmetrised."""
    hd = to_device(h, "h")
    _check_symmetric(hd, "h")
    inv = spd_inverse_device(hd)
    return inv.cpu().numpy() if not isinstance(h, torch.Tensor) else inv


def write_matrix(path, a, dtype: str = "float64") -> None:
    """MOEK writer (numkit.py:110-127); see formats.moek_encode."""
    from .formats import moek_encode
    with open(path, "wb") as fh:
        fh.write(moek_encode(a, dtype))


def read_matrix(path) -> np.ndarray:
    """MOEK reader (numkit.py:130-157); see formats.moek_decode."""
    from .formats import moek_decode
    with open(path, "rb") as fh:
        return moek_decode(fh.read(), str(path))
