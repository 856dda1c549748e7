"""Model descriptors for the device operator.

The physics itself runs in CUDA (``csrc/models.cuh``); these classes
hold the coefficients and pack them for the kernels.  Formulas, species
order and defaults are those of the reference models
(``pkg/src/taxisdg/model.py``):

* ``PlaqueModel`` (``model.py:130-209``): 6 species (n1, n2, n3, c1, c2,
  c3), taxis flux rows for n1 and n2 with chi(x,y,a,b) = a x/(max(y,0)+b),
  reactions, Heaviside-gated prescribed boundary fluxes on GAMMA1/GAMMA2
  and the lipid influx on GAMMA1_IN.
* ``ReducedModel`` (``model.py:212-264``): 3 species (n1, n3, c1).
* ``DiffusionModel``: pure diagonal diffusion with zero source, closed
  either by zero prescribed flux (reference test model
  ``tests/oracles.py:192-205``) or by a constant Dirichlet value through
  the mirrored exterior trace (``tests/oracles.py:208-220``,
  ``operator.py:436-444``).
"""

from __future__ import annotations

from dataclasses import dataclass, fields

import numpy as np

__all__ = ["PlaqueParams", "PlaqueModel", "ReducedModel", "DiffusionModel",
           "gaussian_bump", "MODEL_PLAQUE", "MODEL_REDUCED",
           "MODEL_DIFFUSION", "N_PARAMS"]

MODEL_PLAQUE, MODEL_REDUCED, MODEL_DIFFUSION = 0, 1, 2
N_PARAMS = 32  # doubles in the device parameter block (csrc/models.cuh)


def gaussian_bump(center, width: float, amplitude: float = 1.0):
    """amplitude * exp(-|x - c|^2 / (2 width^2)) (reference model.py:65-73)."""
    c = np.asarray(center, dtype=float)

    def f(x):
        r2 = ((x - c) ** 2).sum(axis=-1)
        return amplitude * np.exp(-r2 / (2.0 * width * width))

    return f


@dataclass
class PlaqueParams:
    """Coefficients and defaults of reference ``model.py:86-112``."""
    mu1: float = 1e-3
    mu2: float = 1e-3
    mu3: float = 1e-3
    nu1: float = 1e-2
    nu2: float = 1e-2
    nu3: float = 1e-2
    d1: float = 0.05
    d2: float = 0.05
    alpha1: float = 0.1
    alpha2: float = 0.1
    k_ox: float = 0.5
    gamma: float = -0.1
    f1_const: float = 0.1
    chi11_a: float = 5e-3
    chi11_b: float = 0.1
    chi13_a: float = 5e-3
    chi13_b: float = 0.1
    chi21_a: float = 5e-3
    chi21_b: float = 0.1
    chi2n_a: float = 5e-3
    chi2n_b: float = 0.1
    beta1: float = 1.0
    beta2: float = 1.0
    sigma: float = 1.0
    c1_star: float = 0.05
    c1_starstar: float = 0.05
    eps_h: float = 0.0

    def __post_init__(self):
        for name in ("mu1", "mu2", "mu3", "nu1", "nu2", "nu3"):
            if getattr(self, name) <= 0:
                raise ValueError(f"diffusivity {name} must be positive")
        for f in fields(self):
            if f.name.endswith("_b") and getattr(self, f.name) <= 0:
                raise ValueError(f"threshold {f.name} must be positive")
        if self.eps_h < 0:
            raise ValueError("eps_h must be >= 0")

    def replace(self, **kw) -> "PlaqueParams":
        vals = {f.name: getattr(self, f.name) for f in fields(self)}
        vals.update(kw)
        return PlaqueParams(**vals)

    def pack(self) -> np.ndarray:
        """Device order (csrc/models.cuh ``enum PlaqueParam``)."""
        out = np.zeros(N_PARAMS)
        out[:len(fields(self))] = [getattr(self, f.name) for f in fields(self)]
        return out


class PlaqueModel:
    species = ("n1", "n2", "n3", "c1", "c2", "c3")
    n_species = 6
    has_convection = True
    model_id = MODEL_PLAQUE
    boundary_kind = "flux"
    seed_species = "n1"

    def __init__(self, params: PlaqueParams | None = None):
        self.params = params if params is not None else PlaqueParams()

    def diffusivity(self) -> np.ndarray:
        p = self.params
        return np.array([p.mu1, p.mu2, p.mu3, p.nu1, p.nu2, p.nu3])

    def linear_source(self) -> np.ndarray:
        """L with S_lin(u) = L u (the bilinear -c1(a1 n1 + a2 n2) part of
        S_c1 is integrated at the quadrature points)."""
        p = self.params
        L = np.zeros((6, 6))
        L[0, 0] = -p.d1
        L[1, 1] = -p.d2
        L[2, 0] = p.d1 - p.gamma
        L[2, 1] = p.d2
        L[3, 2] = p.f1_const
        L[4, 4] = -p.k_ox
        L[5, 4] = p.k_ox
        return L

    def pack(self) -> np.ndarray:
        return self.params.pack()


class ReducedModel:
    species = ("n1", "n3", "c1")
    n_species = 3
    has_convection = True
    model_id = MODEL_REDUCED
    boundary_kind = "flux"
    seed_species = "n3"

    def __init__(self, params: PlaqueParams | None = None):
        self.params = params if params is not None else PlaqueParams()

    def diffusivity(self) -> np.ndarray:
        p = self.params
        return np.array([p.mu1, p.mu3, p.nu1])

    def linear_source(self) -> np.ndarray:
        p = self.params
        L = np.zeros((3, 3))
        L[1, 0] = p.d1 - p.gamma
        L[2, 1] = p.f1_const
        return L

    def pack(self) -> np.ndarray:
        return self.params.pack()


class DiffusionModel:
    """dU/dt = div(kappa grad U), no source.  ``dirichlet`` None closes
    the walls with zero prescribed flux; a float (or per-species array)
    imposes that constant through the mirrored trace u_out = 2 g - u_in.

    Point data (the reference's x-dependent test models,
    tests/test_operator.py:31-70): ``dirichlet_fn(x, t)`` -> (..., S)
    Dirichlet values at physical points (reference ``dirichlet_value``,
    model.py:273), or ``wall_flux_fn(tag, u, normal, t)`` -> (n, S)
    prescribed fluxes in the inward-normal convention (reference
    ``boundary_flux``, operator.py:446-458) that must not depend on u (the
    operator evaluates them with u = 0 at the wall points).  Both are
    evaluated on the host at the face quadrature points, at t = 0 and again
    whenever an application passes another t (``time_dependent``)."""

    has_convection = False
    model_id = MODEL_DIFFUSION

    def __init__(self, kappa=1.0, n_species: int = 1, dirichlet=None, dirichlet_fn=None,
                 wall_flux_fn=None, time_dependent: bool = False):
        self.n_species = int(n_species)
        self.species = tuple(f"u{i}" for i in range(self.n_species))
        self.kappa = np.broadcast_to(np.asarray(kappa, dtype=float),
                                     (self.n_species,)).copy()
        if dirichlet is not None and dirichlet_fn is not None:
            raise ValueError("give either constant Dirichlet data or dirichlet_fn")
        if wall_flux_fn is not None and (dirichlet is not None or dirichlet_fn is not None):
            raise ValueError("wall fluxes and Dirichlet data are exclusive closures")
        self.dirichlet = (None if dirichlet is None else np.broadcast_to(
            np.asarray(dirichlet, dtype=float), (self.n_species,)).copy())
        self.dirichlet_fn = dirichlet_fn
        self.wall_flux_fn = wall_flux_fn
        self.time_dependent = bool(time_dependent)
        self.boundary_kind = ("dirichlet" if dirichlet is not None or dirichlet_fn is not None
                              else "flux")

    @property
    def has_point_data(self) -> bool:
        return self.dirichlet_fn is not None or self.wall_flux_fn is not None

    def diffusivity(self) -> np.ndarray:
        return self.kappa.copy()

    def linear_source(self) -> np.ndarray:
        return np.zeros((self.n_species, self.n_species))

    def pack(self) -> np.ndarray:
        out = np.zeros(N_PARAMS)
        if self.dirichlet is not None:
            out[:self.n_species] = self.dirichlet
        return out
