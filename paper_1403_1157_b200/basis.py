"""Orthonormal modal P_k bases on the reference triangle / tetrahedron.

Host-side setup for the device tables.  Follows the construction of the
reference (``pkg/src/taxisdg/basis.py:40-124``): graded-lexicographic
monomials, orthonormalised against the exact rational Gram matrix of the
reference simplex, so the only roundoff in a coefficient is the final
float conversion and square root.  The coefficient matrix must agree
with the reference bit-for-bit (it decides every table the kernels
read); ``tests/test_setup_tables.py`` checks that against the golden
fixtures made from the reference.
"""

from __future__ import annotations

import math
from fractions import Fraction
from functools import lru_cache

import numpy as np

__all__ = ["MAX_ORDER", "basis_size", "monomial_exponents", "BasisSet"]

MAX_ORDER = 4


def _check(dim: int, order: int) -> None:
    if dim not in (2, 3):
        raise ValueError(f"dim must be 2 or 3, got {dim}")
    if not 0 <= order <= MAX_ORDER:
        raise ValueError(f"order must be in 0..{MAX_ORDER}, got {order}")


def basis_size(dim: int, order: int) -> int:
    """dim P_k = C(k + d, d)  (reference ``basis.py:27-30``)."""
    _check(dim, order)
    return math.comb(order + dim, dim)


def monomial_exponents(dim: int, order: int) -> list[tuple[int, ...]]:
    """Exponent tuples, grouped by total degree, leading exponent
    descending inside a group (reference ``basis.py:40-50``)."""
    _check(dim, order)
    exps: list[tuple[int, ...]] = []
    for deg in range(order + 1):
        for a in range(deg, -1, -1):
            if dim == 2:
                exps.append((a, deg - a))
            else:
                for b in range(deg - a, -1, -1):
                    exps.append((a, b, deg - a - b))
    return exps


def _simplex_moment(exps) -> Fraction:
    """Exact integral of x^a y^b (z^c) over the unit simplex:
    a! b! (c!) / (a + b (+ c) + d)!."""
    num = 1
    for a in exps:
        num *= math.factorial(a)
    return Fraction(num, math.factorial(sum(exps) + len(exps)))


@lru_cache(maxsize=None)
def _orthonormal_coefficients(dim: int, order: int) -> np.ndarray:
    """Rows: basis functions in the monomial basis.

    Exact LDL^T of the Gram matrix G = L D L^T; the orthonormal basis
    is D^{-1/2} L^{-1} m.  Every step up to the float conversion is in
    rational arithmetic.
    """
    exps = monomial_exponents(dim, order)
    n = len(exps)
    gram = [[_simplex_moment([p + q for p, q in zip(exps[i], exps[j])])
             for j in range(n)] for i in range(n)]
    low = [[Fraction(int(i == j)) for j in range(n)] for i in range(n)]
    diag = [Fraction(0)] * n
    for j in range(n):
        acc = gram[j][j]
        for k in range(j):
            acc -= low[j][k] ** 2 * diag[k]
        diag[j] = acc
        for i in range(j + 1, n):
            acc = gram[i][j]
            for k in range(j):
                acc -= low[i][k] * low[j][k] * diag[k]
            low[i][j] = acc / diag[j]
    # forward substitution for L^{-1} (unit lower triangular)
    inv = [[Fraction(0)] * n for _ in range(n)]
    for i in range(n):
        inv[i][i] = Fraction(1)
        for j in range(i - 1, -1, -1):
            acc = Fraction(0)
            for k in range(j, i):
                acc += low[i][k] * inv[k][j]
            inv[i][j] = -acc
    out = np.empty((n, n))
    for i in range(n):
        scale = math.sqrt(float(diag[i]))
        for j in range(n):
            out[i, j] = float(inv[i][j]) / scale
    return out


class BasisSet:
    """Orthonormal basis of total degree ``order``; mode 0 is the
    constant, so element mass matrices are |det J| * I."""

    def __init__(self, dim: int, order: int):
        _check(dim, order)
        self.dim = dim
        self.order = order
        self.exponents = monomial_exponents(dim, order)
        self.coefficients = _orthonormal_coefficients(dim, order)
        self.size = len(self.exponents)

    @staticmethod
    def _pow(points: np.ndarray, exps) -> np.ndarray:
        val = np.ones(points.shape[0])
        for axis, a in enumerate(exps):
            if a:
                val = val * points[:, axis] ** a
        return val

    def eval(self, points) -> np.ndarray:
        """(npts, nb) basis values."""
        pts = np.asarray(points, dtype=float)
        mono = np.stack([self._pow(pts, e) for e in self.exponents], axis=1)
        return mono @ self.coefficients.T

    def grad(self, points) -> np.ndarray:
        """(npts, nb, dim) reference-coordinate gradients."""
        pts = np.asarray(points, dtype=float)
        out = np.empty((pts.shape[0], self.size, self.dim))
        for axis in range(self.dim):
            cols = []
            for e in self.exponents:
                a = e[axis]
                if a == 0:
                    cols.append(np.zeros(pts.shape[0]))
                    continue
                lowered = list(e)
                lowered[axis] = a - 1
                cols.append(a * self._pow(pts, lowered))
            out[:, :, axis] = np.stack(cols, axis=1) @ self.coefficients.T
        return out
