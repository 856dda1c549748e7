"""B200-native matrix-free DG operator for the six-species plaque model.

Host-side setup (mesh, basis, quadrature, space, model descriptors) is
numpy; the operator, the fused M^-1 + Runge-Kutta stage update and the
Krylov reductions run in hand-written sm_100a fp64 CUDA kernels behind
the C-ABI in ``include/taxisdg_b200.h``.
"""

from .basis import BasisSet, basis_size, monomial_exponents  # noqa: F401
from .fespace import DGSpace, DiscreteFunction, face_reference_points  # noqa: F401
from .fields import bump_field, initial_state  # noqa: F401
from .flux import SCHEME_NAMES, FluxScheme, chi_factor, minus_is_outside  # noqa: F401
from .mesh import BoundaryTag, Mesh, is_gamma1, unit_cube, unit_square  # noqa: F401
from .model import (DiffusionModel, PlaqueModel, PlaqueParams,  # noqa: F401
                    ReducedModel, gaussian_bump)
from .quadrature import face_rule, volume_rule  # noqa: F401

__version__ = "0.1.0"
