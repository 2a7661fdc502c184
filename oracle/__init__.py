"""CPU oracle for the KAN / UKAN spline hot path — TEST INFRASTRUCTURE ONLY.

A float64 NumPy restatement of the reference's algorithm (/root/reference/pkg/src/ukan,
itself float64 NumPy); every function cites the reference file:line it follows.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference arm may
import this package, and only as the checker / the timed CPU baseline — never as the
product path (the product is ``paper_2408_11200_b200`` -> ``libukan_b200.so``).

Parity pinning: ``tests/test_oracle_golden.py`` checks this oracle against golden vectors
produced by the reference implementation itself (``tests/golden/make_golden.py`` imports
``ukan`` from the read-only reference tree and runs its own layers / tape / optimizer).
"""
from .spline import (basis_matrix, basis_values, kan_locate, kan_forward_backward,
                     ukan_locate, ukan_keys, positional_encoding, cg_forward,
                     ukan_forward_backward, kan_tangent_forward_backward,
                     ukan_tangent_forward_backward, softmax_xent, mse, adam_step, model_step,
                     kan_rows, kan_feature_grads)

__all__ = [n for n in dir() if not n.startswith("_")]
