"""The drop-in boundary accepts the reference's own objects
(``DiscreteOperator(space, model, scheme)`` with ``taxisdg`` DGSpace /
PlaqueModel / FluxScheme, reference operator.py:85-92): the adapted
descriptions pack exactly the tables the package path packs.  Runs in the
build container only (the reference tree is not on the GPU box)."""
import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
if not os.path.isdir(REF):
    pytest.skip("reference package not present", allow_module_level=True)
sys.path.insert(0, REF)
taxisdg = pytest.importorskip("taxisdg")
sys.path.insert(0, "/root/reference/pkg/tests")
oracles = pytest.importorskip("oracles")

from paper_1403_1157_b200 import (DGSpace, DiffusionModel, FluxScheme,  # noqa: E402
                                  PlaqueModel, PlaqueParams, ReducedModel,
                                  unit_cube, unit_square)
from paper_1403_1157_b200.compat import adapt  # noqa: E402
from paper_1403_1157_b200.tables import build_tables  # noqa: E402

from _cases import AMPLIFIED  # noqa: E402

T = taxisdg


def _ref_mesh(kind):
    if kind == "sq4":
        return T.mesh.unit_square(4)
    if kind == "rect":
        m = T.mesh.unit_square(8, 2)
        tags = {tuple(int(x) for x in m.face_vertices[f]): int(m.face_tags[f])
                for f in np.flatnonzero(m.boundary_mask)}
        return T.mesh.Mesh(m.vertices * np.array([4.0, 1.0]), m.elements, tags)
    return T.mesh.unit_cube(2)


def _pkg_mesh(kind):
    if kind == "sq4":
        return unit_square(4)
    if kind == "rect":
        return unit_square(8, 2, lengths=(4.0, 1.0))
    return unit_cube(2)


CASES = [
    ("sq4", 2, "plaque", "cdg2"), ("rect", 3, "plaque_amp", "br2"),
    ("cube", 2, "plaque", "ip"), ("sq4", 1, "reduced", "cdg"),
    ("sq4", 2, "heat", "bo"), ("cube", 1, "dirichlet", "cdg2"),
]


def _models(kind):
    if kind == "plaque":
        return T.model.PlaqueModel(), PlaqueModel()
    if kind == "plaque_amp":
        return (T.model.PlaqueModel(T.model.PlaqueParams(**AMPLIFIED)),
                PlaqueModel(PlaqueParams(**AMPLIFIED)))
    if kind == "reduced":
        return T.model.ReducedModel(), ReducedModel()
    if kind == "heat":
        return oracles.ZeroFluxHeat(kappa=0.7), DiffusionModel(0.7)
    return oracles.ConstantDirichletHeat(0.4, kappa=0.7, dim=3), DiffusionModel(0.7, dirichlet=0.4)


@pytest.mark.parametrize("mesh,k,model,scheme", CASES)
def test_reference_objects_pack_the_package_tables(mesh, k, model, scheme):
    rmodel, pmodel = _models(model)
    rspace = T.fespace.DGSpace(_ref_mesh(mesh), k, rmodel.n_species)
    rscheme = T.flux.FluxScheme(scheme, ip_eta0=3.0)
    space, m, s = adapt(rspace, rmodel, rscheme)
    assert type(m) is type(pmodel) and s == FluxScheme(scheme, 3.0)
    assert np.array_equal(m.pack(), pmodel.pack())
    assert np.array_equal(m.linear_source(), pmodel.linear_source())
    rm = rspace.mesh
    for name in ("vertices", "elements", "face_elems", "face_local", "face_perm",
                 "face_normals", "face_measures", "face_tags", "volumes"):
        assert np.array_equal(getattr(space.mesh, name), getattr(rm, name)), name
    a = build_tables(space, m, s)
    b = build_tables(DGSpace(_pkg_mesh(mesh), k, pmodel.n_species), pmodel, FluxScheme(scheme, 3.0))
    for f in ("vol_phi", "vol_grad", "vol_w", "face_B", "face_G", "face_Pw", "elem_geo",
              "if_elems", "if_code", "if_geo", "bf_elem", "bf_code", "bf_geo", "seg_if"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f


def test_unsupported_reference_model_raises_value_error():
    rspace = T.fespace.DGSpace(T.mesh.unit_square(2), 1, 1)
    with pytest.raises(ValueError):
        adapt(rspace, T.model.HeatModel(1.0), T.flux.FluxScheme("cdg2"))


def test_package_objects_pass_through():
    space = DGSpace(unit_square(2), 1, 6)
    m, s = PlaqueModel(), FluxScheme("cdg2")
    a = adapt(space, m, s)
    assert a[0] is space and a[1] is m and a[2] is s


def test_x_dependent_heat_models_adapt_with_point_data():
    """The reference's linear-field test models (tests/test_operator.py:31-70:
    a ZeroFluxHeat with a normal-dependent boundary_flux, a
    ConstantDirichletHeat with an x-dependent dirichlet_value) adapt to
    DiffusionModel with point data, evaluated through the reference's own
    methods."""
    class LinearWall(oracles.ZeroFluxHeat):
        def __init__(self):
            super().__init__(kappa=0.8)

        def boundary_flux(self, tag, U, normal, t):
            qn = -self.kappa * (normal @ np.array([2.0, -1.0]))
            return np.broadcast_to(qn[:, None], U.shape).copy()

    class LinearDirichlet(oracles.ConstantDirichletHeat):
        def __init__(self):
            super().__init__(0.0, kappa=0.8)

        def dirichlet_value(self, x, t):
            return (0.3 + 2.0 * x[..., 0] - 1.0 * x[..., 1])[..., None]

    space = T.fespace.DGSpace(T.mesh.unit_square(3), 2)
    _, wall, _ = adapt(space, LinearWall(), T.flux.FluxScheme("cdg2"))
    assert isinstance(wall, DiffusionModel) and wall.wall_flux_fn is not None
    n = np.array([[0.0, -1.0], [1.0, 0.0]])
    assert np.allclose(wall.wall_flux_fn(1, np.zeros((2, 1)), n, 0.0)[:, 0],
                       -0.8 * (n @ np.array([2.0, -1.0])))
    _, dmod, _ = adapt(space, LinearDirichlet(), T.flux.FluxScheme("cdg2"))
    assert dmod.boundary_kind == "dirichlet" and dmod.dirichlet_fn is not None
    assert np.allclose(dmod.dirichlet_fn(np.array([[0.5, 0.25]]), 0.0), [[1.05]])
    _, plain, _ = adapt(space, oracles.ConstantDirichletHeat(0.4, kappa=0.8),
                        T.flux.FluxScheme("cdg2"))
    assert plain.dirichlet_fn is None and plain.dirichlet[0] == 0.4
