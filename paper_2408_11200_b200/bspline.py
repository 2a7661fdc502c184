"""Host-side B-spline constants: the exact basis matrix (bspline.py:24-80 of the reference).

``basis_matrix(k)`` returns the same ``BasisMatrix`` record as the reference: the exact
rational K x K matrix (row i = coefficient of u^i, column j = window slot j) and its float64
rounding.  The float64 values come from the C ABI (``ukan_basis_matrix``, the same numbers the
kernels use) and are checked against the rational matrix computed here.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from . import _lib
from .errors import DomainError

MAX_DEGREE = 10


def _segment_polynomials(k: int) -> list[list[Fraction]]:
    """Monomial coefficients of B_{j,k} on [0,1) for j = -k..0 via Cox-de Boor on unit knots
    (bspline.py:24-51); entry j of the result is the polynomial of window slot j."""
    polys: dict[int, list[Fraction]] = {0: [Fraction(1)]}
    for kk in range(1, k + 1):
        nxt: dict[int, list[Fraction]] = {}
        for j in range(-kk, 1):
            c = [Fraction(0)] * (kk + 1)
            if j in polys:  # (u - j)/kk * B_{j,kk-1}
                for i, a in enumerate(polys[j]):
                    c[i + 1] += a / kk
                    c[i] -= a * Fraction(j, kk)
            if j + 1 in polys:  # (j + kk + 1 - u)/kk * B_{j+1,kk-1}
                for i, a in enumerate(polys[j + 1]):
                    c[i] += a * Fraction(j + kk + 1, kk)
                    c[i + 1] -= a / kk
            nxt[j] = c
        polys = nxt
    return [polys[j - k] for j in range(k + 1)]


@dataclass(frozen=True)
class BasisMatrix:
    degree: int
    rational: tuple
    floats: np.ndarray

    @property
    def K(self) -> int:
        return self.degree + 1


_cache: dict[int, BasisMatrix] = {}


def basis_matrix(k: int) -> BasisMatrix:
    if not (0 <= k <= MAX_DEGREE):
        raise DomainError(f"degree must be in [0, {MAX_DEGREE}], got {k}")
    if k not in _cache:
        cols = _segment_polynomials(k)
        rows = tuple(tuple(cols[j][i] for j in range(k + 1)) for i in range(k + 1))
        K = k + 1
        buf = (ctypes.c_double * (K * K))()
        _lib.check(_lib.load().ukan_basis_matrix(k, ctypes.cast(buf, ctypes.c_void_p)), "basis_matrix")
        floats = np.frombuffer(buf, dtype=np.float64).reshape(K, K).copy()
        exact = np.array([[float(c) for c in r] for r in rows])
        if not np.array_equal(floats, exact):
            raise RuntimeError("C ABI basis matrix disagrees with the exact rational matrix")
        floats.setflags(write=False)
        _cache[k] = BasisMatrix(degree=k, rational=rows, floats=floats)
    return _cache[k]
