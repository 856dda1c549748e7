"""Seeded synthetic initial fields.

u_s(x) = 0.1 + 0.05 * sum_b gaussian_bump(c_b, w_b, a_b)(x) with, per
species and per bump (4 bumps in 2D, 8 in 3D), centre ~ U(domain box),
width ~ U(0.05, 0.15), amplitude ~ U(0.5, 1.0), drawn in that order
from ``numpy.random.default_rng(seed)``; the bump is the reference's
``gaussian_bump`` (``pkg/src/taxisdg/model.py:65-73``).  Projected with
``DGSpace.project`` (degree 2k+4, reference ``fespace.py:90-111``).
"""

from __future__ import annotations

import numpy as np

from .model import gaussian_bump

__all__ = ["bump_field", "initial_state"]


def bump_field(dim, n_species, seed, box_lo, box_hi, nbumps=None):
    rng = np.random.default_rng(seed)
    nbumps = nbumps or (4 if dim == 2 else 8)
    bumps = []
    for _ in range(n_species):
        row = []
        for _ in range(nbumps):
            c = rng.uniform(box_lo, box_hi)
            w = rng.uniform(0.05, 0.15)
            a = rng.uniform(0.5, 1.0)
            row.append(gaussian_bump(c, w, a))
        bumps.append(row)

    def fn(x):
        out = np.full(x.shape[:-1] + (n_species,), 0.1)
        for s in range(n_species):
            for f in bumps[s]:
                out[..., s] += 0.05 * f(x)
        return out

    return fn


def initial_state(space, seed: int, box=None) -> np.ndarray:
    """Projected bump field on ``space``; ``box`` defaults to the mesh's
    bounding box."""
    mesh = space.mesh
    lo, hi = ((mesh.vertices.min(axis=0), mesh.vertices.max(axis=0))
              if box is None else box)
    return np.ascontiguousarray(space.project(bump_field(
        mesh.dim, space.n_species, seed, np.asarray(lo), np.asarray(hi))).coeffs)
