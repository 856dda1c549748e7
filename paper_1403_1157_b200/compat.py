"""Accept the reference's own objects at the drop-in boundary.

A reference user builds ``taxisdg`` objects -- ``DGSpace(mesh, order,
n_species)`` (reference ``fespace.py:46-61``), ``PlaqueModel(PlaqueParams)``
(``model.py:77-209``), ``FluxScheme(name, ip_eta0)`` (``flux.py:63-84``) --
and hands them to ``DiscreteOperator(space, model, scheme, ...)``
(``operator.py:85-92``).  ``adapt`` maps them, duck-typed (the reference
package is not importable on the GPU box), onto this package's host-side
descriptions, which the operator packs for the device:

* space: the reference mesh's (already oriented) vertices and elements
  rebuild this package's ``Mesh`` -- same first-touch face numbering,
  sides, local faces, permutations and geometry (pinned by
  tests/test_setup_golden.py) -- with the reference's per-face boundary
  tags carried over face by face;
* model: ``PlaqueModel`` / ``ReducedModel`` by class, their
  ``PlaqueParams`` copied field by field; the reference's heat test
  models (``tests/oracles.py:192-220``: insulated walls, or constant
  Dirichlet data) become ``DiffusionModel``, subclasses with x- or
  normal-dependent ``dirichlet_value`` / ``boundary_flux`` with point data;
* scheme: name and ``ip_eta0``.

Models whose physics is not compiled for the device (the manufactured
models with x/t-dependent forcing, reference ``model.py:277-414``) raise
``ValueError``, the reference's error type for unusable configurations.
"""

from __future__ import annotations

from dataclasses import fields

import numpy as np

from .fespace import DGSpace
from .flux import FluxScheme
from .mesh import Mesh
from .model import DiffusionModel, PlaqueModel, PlaqueParams, ReducedModel

__all__ = ["adapt", "adapt_space", "adapt_model", "adapt_scheme"]


def _is_ours(obj, cls) -> bool:
    return isinstance(obj, cls)


def adapt_mesh(mesh) -> Mesh:
    if isinstance(mesh, Mesh):
        return mesh
    verts = np.asarray(mesh.vertices, dtype=float)
    elems = np.asarray(mesh.elements, dtype=np.int64)
    fv = np.asarray(mesh.face_vertices, dtype=np.int64)
    ftag = np.asarray(mesh.face_tags)
    bnd = np.flatnonzero(np.asarray(mesh.face_elems)[:, 1] < 0)
    keys_ref = np.sort(fv[bnd], axis=1)
    tags_ref = ftag[bnd]
    order_ref = np.lexsort(keys_ref.T[::-1])

    def tag_fn(keys):
        """The reference's tag of every boundary face, matched by its
        sorted vertex ids."""
        k = np.sort(np.asarray(keys, dtype=np.int64), axis=1)
        o = np.lexsort(k.T[::-1])
        if len(k) != len(keys_ref) or not np.array_equal(k[o], keys_ref[order_ref]):
            raise ValueError("reference mesh boundary does not match its faces")
        out = np.empty(len(k), dtype=np.int8)
        out[o] = tags_ref[order_ref]
        return out

    m = Mesh(verts, elems, tag_fn=tag_fn)
    if not np.array_equal(m.elements, elems) or not np.array_equal(m.face_vertices, fv):
        raise ValueError("reference mesh is not reproduced (element orientation / faces)")
    return m


def adapt_space(space) -> DGSpace:
    if _is_ours(space, DGSpace):
        return space
    return DGSpace(adapt_mesh(space.mesh), int(space.order), int(space.n_species))


def _params(p) -> PlaqueParams:
    return PlaqueParams(**{f.name: float(getattr(p, f.name)) for f in fields(PlaqueParams)})


def _overrides(model, base_name: str, method: str) -> bool:
    """True when a subclass of the reference class ``base_name`` redefines
    ``method``."""
    for cls in type(model).__mro__:
        if cls.__name__ == base_name:
            return getattr(type(model), method) is not getattr(cls, method)
    return False


def adapt_model(model):
    if _is_ours(model, (PlaqueModel, ReducedModel, DiffusionModel)):
        return model
    name = type(model).__name__
    mro = {c.__name__ for c in type(model).__mro__}
    if "PlaqueModel" in mro:
        return PlaqueModel(_params(model.params))
    if "ReducedModel" in mro:
        return ReducedModel(_params(model.params))
    if "ZeroFluxHeat" in mro:
        # a subclass overriding boundary_flux (x / normal-dependent walls,
        # reference tests/test_operator.py:31-51) keeps its data as point data
        if _overrides(model, "ZeroFluxHeat", "boundary_flux"):
            return DiffusionModel(float(model.kappa), wall_flux_fn=model.boundary_flux)
        return DiffusionModel(float(model.kappa))
    if "ConstantDirichletHeat" in mro:
        # likewise an overridden dirichlet_value (tests/test_operator.py:54-70)
        if _overrides(model, "ConstantDirichletHeat", "dirichlet_value"):
            return DiffusionModel(float(model.kappa), dirichlet_fn=model.dirichlet_value)
        return DiffusionModel(float(model.kappa), dirichlet=float(model.value))
    raise ValueError(f"model {name!r} has no device implementation (plaque, reduced, "
                     "zero-flux or constant-Dirichlet diffusion)")


def adapt_scheme(scheme) -> FluxScheme:
    if _is_ours(scheme, FluxScheme):
        return scheme
    return FluxScheme(str(scheme.name), float(getattr(scheme, "ip_eta0", 4.0)))


def adapt(space, model, scheme):
    """(space, model, scheme) of this package for reference or package
    objects (package objects pass through unchanged)."""
    return adapt_space(space), adapt_model(model), adapt_scheme(scheme)
