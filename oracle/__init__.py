"""CPU oracle for the W8A8 MoE hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy (float64 / int64), the reference
algorithm of arXiv 2508.07329's ``moekit`` toolkit for the path named by
BASELINE.json's north star. It exists to CHECK the CUDA path, never to be it:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import it;
* the product package ``paper_2508_07329_b200`` never imports it and has no
  CPU fallback (it raises when its CUDA library is missing).

Parity status:

* quantizer, smoothing, Hessian, GPTQ column loop, channel ordering,
  packing, routing statistics and placement are PINNED: the restatement is
  checked against golden vectors produced by running the unmodified
  reference (``tests/golden/make_golden.py`` imports
  ``/root/reference/pkg/src/moekit``) plus the reference tests' own
  known-answer cases;
* router top-k gating, token permutation, grouped expert FFN (SwiGLU) and
  combine do not exist in the reference; ``moe_ref`` restates them from the
  reference's primitives (quantizer semantics quant.py:191-264, routing
  event format trace.py:40-44). Their parity is UNPINNED at the reference
  level (there is nothing to pin to) and is documented as such.

Module map:
  quant_ref     <- moekit/quant.py
  numkit_ref    <- moekit/numkit.py
  routing_ref   <- moekit/trace.py (statistics) + moekit/placement.py
  moe_ref       <- new MoE forward pieces built from quant_ref primitives
"""
