"""Quadrature rules on the reference simplices (host-side table setup).

Restates the rule family the reference integrates with
(``pkg/src/taxisdg/quadrature.py:84-140``):

* volume: Grundmann-Moeller of odd degree 2s+1 on the unit simplex,
  built in exact rationals (weights of alternating sign);
* faces: Gauss-Legendre on [0, 1] for triangle edges, Grundmann-Moeller
  on the unit triangle for tetrahedron faces.

The operator integrates volumes at degree 3k+1 and faces at 3k+2
(reference ``operator.py:106-109``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from fractions import Fraction
from functools import lru_cache

import numpy as np

__all__ = ["QuadRule", "grundmann_moeller", "gauss_segment",
           "volume_rule", "face_rule"]


@dataclass(frozen=True)
class QuadRule:
    points: np.ndarray   # (n, dim)
    weights: np.ndarray  # (n,)
    degree: int

    def __len__(self) -> int:
        return self.points.shape[0]


def _compositions(total: int, parts: int):
    """All ``parts``-tuples of non-negative ints summing to ``total``,
    first entry increasing slowest-to-fastest as in a stars-and-bars
    enumeration."""
    if parts == 1:
        yield (total,)
        return
    for first in range(total + 1):
        for rest in _compositions(total - first, parts - 1):
            yield (first,) + rest


@lru_cache(maxsize=None)
def grundmann_moeller(dim: int, s: int) -> QuadRule:
    """Degree 2s+1 rule on the unit ``dim``-simplex:

    w_i = (-1)^i 2^{-2s} (deg + dim - 2i)^deg / (i! (deg + dim - i)!),
    nodes (2 beta + 1) / (deg + dim - 2i) in barycentric coordinates,
    |beta| = s - i  (Grundmann & Moeller 1978).
    """
    if dim < 1 or s < 0:
        raise ValueError("need dim >= 1 and s >= 0")
    deg = 2 * s + 1
    pts, wts = [], []
    for i in range(s + 1):
        den = deg + dim - 2 * i
        w = (Fraction(-1) ** i * Fraction(den) ** deg
             / (Fraction(4) ** s * math.factorial(i)
                * math.factorial(deg + dim - i)))
        for beta in _compositions(s - i, dim + 1):
            pts.append([float(Fraction(2 * b + 1, den)) for b in beta[1:]])
            wts.append(float(w))
    return QuadRule(np.array(pts), np.array(wts), deg)


@lru_cache(maxsize=None)
def gauss_segment(degree: int) -> QuadRule:
    """Gauss-Legendre on [0, 1] with degree//2 + 1 nodes."""
    if degree < 0:
        raise ValueError("degree must be >= 0")
    n = degree // 2 + 1
    x, w = np.polynomial.legendre.leggauss(n)
    return QuadRule((0.5 * (x + 1.0)).reshape(-1, 1), 0.5 * w, 2 * n - 1)


def volume_rule(dim: int, degree: int) -> QuadRule:
    if dim not in (2, 3):
        raise ValueError(f"dim must be 2 or 3, got {dim}")
    return grundmann_moeller(dim, max(0, degree // 2))


def face_rule(dim: int, degree: int) -> QuadRule:
    if dim == 2:
        return gauss_segment(degree)
    if dim == 3:
        return volume_rule(2, degree)
    raise ValueError(f"dim must be 2 or 3, got {dim}")
