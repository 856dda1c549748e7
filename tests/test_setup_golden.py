"""Host-side setup (basis, quadrature, face points, meshes) against the
reference's own arrays (tests/golden/tables.npz, meshes.npz)."""
import numpy as np
import pytest

from paper_1403_1157_b200 import (BasisSet, BoundaryTag,
                                  face_reference_points, face_rule,
                                  unit_cube, unit_square)
from paper_1403_1157_b200.quadrature import gauss_segment, grundmann_moeller


@pytest.mark.parametrize("dim", [2, 3])
def test_basis_bitwise(golden, dim):
    t = golden["tables"]
    for k in range(5):
        b = BasisSet(dim, k)
        assert np.array_equal(b.coefficients, t[f"basis_coeff_{dim}_{k}"])
        pts = grundmann_moeller(dim, max(1, k)).points
        np.testing.assert_allclose(b.eval(pts), t[f"basis_eval_{dim}_{k}"],
                                   rtol=0, atol=1e-13)
        np.testing.assert_allclose(b.grad(pts), t[f"basis_grad_{dim}_{k}"],
                                   rtol=0, atol=1e-12)


def test_quadrature_bitwise(golden):
    t = golden["tables"]
    for dim in (1, 2, 3):
        for s in range(7):
            r = grundmann_moeller(dim, s)
            assert np.array_equal(r.points, t[f"gm_points_{dim}_{s}"])
            assert np.array_equal(r.weights, t[f"gm_weights_{dim}_{s}"])
    for deg in range(12):
        r = gauss_segment(deg)
        assert np.array_equal(r.points, t[f"gauss_points_{deg}"])
        assert np.array_equal(r.weights, t[f"gauss_weights_{deg}"])


def test_face_reference_points_bitwise(golden):
    t = golden["tables"]
    for dim in (2, 3):
        fr = face_rule(dim, 8)
        for lf in range(dim + 1):
            for pm in range(2 if dim == 2 else 6):
                assert np.array_equal(face_reference_points(dim, lf, pm,
                                                            fr.points),
                                      t[f"frp_{dim}_{lf}_{pm}"])


MESHES = {
    "sq3_": lambda: unit_square(3),
    "sq52_": lambda: unit_square(5, 2),
    "rect82_": lambda: unit_square(8, 2, lengths=(4.0, 1.0)),
    "jit82_": lambda: unit_square(8, 2, lengths=(4.0, 1.0), jitter=0.1,
                                  seed=3),
    "cube2_": lambda: unit_cube(2),
    "cube322_": lambda: unit_cube(3, 2, 2),
    "cubez2_": lambda: unit_cube(2, gamma1_in=None,
                                 top_tag=BoundaryTag.NO_FLOW),
}


@pytest.mark.parametrize("prefix", sorted(MESHES))
def test_mesh_matches_reference(golden, prefix):
    m = golden["meshes"]
    mesh = MESHES[prefix]()
    J, detJ, Jinv = mesh.jacobians()
    exact = {"vertices": mesh.vertices, "elements": mesh.elements,
             "volumes": mesh.volumes, "diameters": mesh.diameters,
             "face_vertices": mesh.face_vertices,
             "face_elems": mesh.face_elems, "face_local": mesh.face_local,
             "face_perm": mesh.face_perm, "face_tags": mesh.face_tags,
             "detJ": detJ, "Jinv": Jinv}
    for name, arr in exact.items():
        # volumes decide the K- tie rule: they must be bit-identical
        assert np.array_equal(arr, m[prefix + name]), name
    np.testing.assert_allclose(mesh.face_normals, m[prefix + "face_normals"],
                               rtol=0, atol=1e-15)
    np.testing.assert_allclose(mesh.face_measures,
                               m[prefix + "face_measures"], rtol=1e-15)


def test_kminus_ties_on_uniform_meshes():
    # every interior face of a uniform dyadic mesh is a
    # volume tie (non-dyadic spacings such as unit_cube(3) give ulp-level
    # volume differences that the K- rule does see -- one more reason the
    # volumes must be bit-identical to the reference's)
    for mesh in (unit_square(8, 4, lengths=(4.0, 1.0)), unit_cube(4)):
        fe = mesh.face_elems[mesh.face_elems[:, 1] >= 0]
        assert np.array_equal(mesh.volumes[fe[:, 0]], mesh.volumes[fe[:, 1]])
        assert np.all(fe[:, 0] < fe[:, 1])
