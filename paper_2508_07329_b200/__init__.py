"""B200-native W8A8 Mixture-of-Experts hot path of arXiv 2508.07329 (HAQ
smoothed-Hessian quantization + statistics-driven expert placement).

Drop-in surface for the reference package ``moekit``:

* ``quant``      — moekit.quant names/signatures, executed by sm_100a kernels
* ``numkit``     — moekit.numkit (validation, factorizations, MOEK files)
* ``trace``      — moekit.trace data model + routing statistics (GPU counts)
* ``placement``  — moekit.placement planners (host logic)
* ``errors``     — the reference exception taxonomy

plus the forward path the reference lacks: ``W8A8Linear``, ``MoELayer`` and
the expert-parallel runtime ``ep``. All compute goes through the C ABI in
``include/moe_b200.h`` (lib/libmoe_b200.so); there is no CPU fallback.
"""

__version__ = "0.1.0"

from . import errors, formats, numkit, placement, quant, trace  # noqa: F401


def __getattr__(name):
    if name == "W8A8Linear":
        from .linear import W8A8Linear
        return W8A8Linear
    if name == "MoELayer":
        from .moe import MoELayer
        return MoELayer
    raise AttributeError(name)


__all__ = ["errors", "formats", "numkit", "placement", "quant", "trace", "W8A8Linear", "MoELayer", "__version__"]
