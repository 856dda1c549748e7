"""Numerical-flux family selector (host side).

Scheme ids and per-scheme constants of reference
``pkg/src/taxisdg/flux.py:57-95``:

* cdg2: 2 chi_e A r_e(J) on K- ;   cdg: 4 chi_e A r_e(J) on K-
* br2:  2 chi_e A {r_e(J)}         ip:  -(eta0 max(k,1)^2 / h) A [u]
* bo:   no penalty, adjoint consistency term flips sign
* chi_e = 1.5 on triangles, 2 on tetrahedra
* K- = smaller volume, exact ties to the lower element id.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["SCHEME_NAMES", "SCHEME_IDS", "FluxScheme", "chi_factor",
           "minus_is_outside"]

SCHEME_NAMES = ("cdg2", "cdg", "br2", "ip", "bo")
SCHEME_IDS = {name: i for i, name in enumerate(SCHEME_NAMES)}


@dataclass(frozen=True)
class FluxScheme:
    name: str
    ip_eta0: float = 4.0

    def __post_init__(self):
        if self.name not in SCHEME_NAMES:
            raise ValueError(f"unknown flux scheme {self.name!r}; pick one "
                             f"of {SCHEME_NAMES}")
        if self.ip_eta0 <= 0:
            raise ValueError("ip_eta0 must be positive")

    @property
    def id(self) -> int:
        return SCHEME_IDS[self.name]

    @property
    def adjoint_sign(self) -> float:
        return -1.0 if self.name == "bo" else 1.0

    @property
    def uses_lifting(self) -> bool:
        return self.name in ("cdg2", "cdg", "br2")


def chi_factor(dim: int) -> float:
    return {2: 1.5, 3: 2.0}[dim]


def minus_is_outside(vol_in, vol_out, elem_in, elem_out):
    """True where the outside element is K- (reference ``flux.py:92-95``)."""
    vol_in, vol_out = np.asarray(vol_in), np.asarray(vol_out)
    return (vol_out < vol_in) | ((vol_out == vol_in)
                                 & (np.asarray(elem_out) < np.asarray(elem_in)))
