"""The CPU oracle (oracle/) against outputs of the real reference."""
import numpy as np
import pytest

from oracle import OracleOperator, sdirk_integrate, ssprk3
from paper_1403_1157_b200 import (DGSpace, DiffusionModel, FluxScheme, Mesh,
                                  PlaqueModel, PlaqueParams, unit_cube,
                                  unit_square)
from paper_1403_1157_b200.fields import initial_state

from _cases import AMPLIFIED, operator_case, operator_names, \
    rel_l2_per_species


def _golden_names():
    import os
    here = os.path.join(os.path.dirname(__file__), "golden", "operator.npz")
    return sorted({k.split("__")[0] for k in np.load(here).files})


@pytest.mark.parametrize("name", _golden_names())
def test_oracle_apply_matches_reference(golden, name):
    space, model, scheme, U, R, F = operator_case(golden, name)
    op = OracleOperator(space, model, scheme)
    got = op.apply(U)
    scale = np.abs(R).max()
    assert np.abs(got - R).max() <= 1e-12 * scale
    np.testing.assert_allclose(op.apply_f(U), F, rtol=0,
                               atol=1e-12 * np.abs(F).max())


def test_oracle_threads_change_grouping_only(golden):
    space, model, scheme, U, R, _ = operator_case(golden, "sq4_p2_amp_cdg2")
    a = OracleOperator(space, model, scheme, nthreads=1).apply(U)
    b = OracleOperator(space, model, scheme, nthreads=3).apply(U)
    assert np.abs(a - b).max() <= 1e-13 * np.abs(a).max()


def test_initial_state_matches_reference_projection(golden):
    t = golden["trajectories"]
    space = DGSpace(unit_square(32), 1, 6)
    U0 = initial_state(space, seed=1)
    np.testing.assert_allclose(U0, t["c1__U0"], rtol=0, atol=1e-15)


def test_oracle_ssprk3_c1(golden):
    t = golden["trajectories"]
    space = DGSpace(unit_square(32), 1, 6)
    op = OracleOperator(space, PlaqueModel(), FluxScheme("cdg2"))
    U = ssprk3(op, t["c1__U0"], float(t["c1__dt"]), 10)
    assert rel_l2_per_species(space, U, t["c1__U10"]).max() <= 1e-13


def test_oracle_ssprk3_3d(golden):
    t = golden["trajectories"]
    from paper_1403_1157_b200 import BoundaryTag
    space = DGSpace(unit_cube(3, gamma1_in=None, top_tag=BoundaryTag.NO_FLOW),
                    2, 6)
    op = OracleOperator(space, PlaqueModel(), FluxScheme("cdg2"))
    U = ssprk3(op, t["cubez3__U0"], 2e-4, 3)
    assert rel_l2_per_species(space, U, t["cubez3__U3"]).max() <= 1e-13


def test_oracle_sdirk3(golden):
    t = golden["trajectories"]
    space = DGSpace(unit_square(4), 2, 6)
    op = OracleOperator(space, PlaqueModel(), FluxScheme("cdg2"))
    U = sdirk_integrate(op, t["sdirk__U0"], 0.01, 2,
                        {"rtol": 1e-11, "atol": 1e-13, "gmres_rtol": 1e-6})
    assert rel_l2_per_species(space, U, t["sdirk__U2"]).max() <= 1e-10


def _two_triangles():
    return Mesh(np.array([[0.0, 0.0], [1.0, 0.0], [1.0, 1.0], [0.0, 1.0]]),
                np.array([[0, 1, 2], [0, 2, 3]]))


@pytest.mark.parametrize("scheme", ["cdg2", "br2", "ip"])
@pytest.mark.parametrize("dirichlet", [False, True])
def test_oracle_matches_dense_diffusion_matrix(golden, scheme, dirichlet):
    """Reference's independent loop oracle (tests/oracles.py:223-327)."""
    h = golden["heat"]
    for mname, mesh in (("two", _two_triangles()), ("sq2", unit_square(2))):
        for k in (1, 2):
            space = DGSpace(mesh, k)
            model = DiffusionModel(0.35, dirichlet=0.0 if dirichlet else None)
            op = OracleOperator(space, model, FluxScheme(scheme))
            n = space.n_dofs
            base = op.apply(np.zeros(space.shape)).ravel()
            A = np.empty((n, n))
            for j in range(n):
                e = np.zeros(n)
                e[j] = 1.0
                A[:, j] = op.apply(e.reshape(space.shape)).ravel() - base
            R = h[f"dense_{mname}_{k}_{scheme}_{int(dirichlet)}"]
            assert np.abs(A - R).max() <= 1e-10 * np.abs(R).max()


@pytest.mark.parametrize("scheme", ["cdg2", "cdg", "br2", "ip", "bo"])
@pytest.mark.parametrize("dirichlet", [0, 1])
def test_oracle_heat_models(golden, scheme, dirichlet):
    h = golden["heat"]
    space = DGSpace(unit_square(3), 2)
    model = DiffusionModel(0.7, dirichlet=0.4 if dirichlet else None)
    op = OracleOperator(space, model, FluxScheme(scheme))
    key = f"heat_sq3_{scheme}_{dirichlet}"
    R = h[f"{key}__R"]
    assert np.abs(op.apply(h[f"{key}__U"]) - R).max() <= 1e-12 * np.abs(R).max()
