"""Generate golden fixtures by running the REAL reference (``taxisdg``).

Run in the build container only (the reference tree does not exist on
the GPU box):

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Writes ``tests/golden/*.npz``.  Every array in them is produced by the
reference's own public API (``DiscreteOperator.apply/apply_f``,
``BasisSet``, ``volume_rule``/``face_rule``, ``Mesh``, ``integrate``);
the only thing defined here is the seeded initial-field recipe
(SURVEY.md section 8(d)), whose coefficients are projected with the
reference's ``DGSpace.project``.
"""

from __future__ import annotations

import math
import os
import sys
import time

import numpy as np

import taxisdg
from taxisdg.basis import BasisSet
from taxisdg.fespace import DGSpace, face_reference_points
from taxisdg.flux import FluxScheme
from taxisdg.mesh import BoundaryTag, Mesh, unit_cube, unit_square
from taxisdg.model import PlaqueModel, PlaqueParams, ReducedModel, gaussian_bump
from taxisdg.operator import DiscreteOperator
from taxisdg.quadrature import face_rule, gauss_segment, grundmann_moeller
from taxisdg.timeint import integrate

sys.path.insert(0, "/root/reference/pkg/tests")
import oracles  # noqa: E402  (reference test models)

HERE = os.path.dirname(os.path.abspath(__file__))
assert "/root/reference" in taxisdg.__file__, taxisdg.__file__


def bump_field(dim, n_species, seed, box_lo, box_hi, nbumps=None):
    """u_s = 0.1 + 0.05 * sum_b gaussian_bump(c_b, w_b, a_b); per species,
    per bump: centre ~ U(box), width ~ U(0.05, 0.15), amplitude ~
    U(0.5, 1.0), drawn in that order from default_rng(seed)."""
    rng = np.random.default_rng(seed)
    nbumps = nbumps or (4 if dim == 2 else 8)
    bumps = []
    for s in range(n_species):
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


def mesh_arrays(mesh, prefix):
    J, detJ, Jinv = mesh.jacobians()
    return {f"{prefix}vertices": mesh.vertices,
            f"{prefix}elements": mesh.elements,
            f"{prefix}volumes": mesh.volumes,
            f"{prefix}diameters": mesh.diameters,
            f"{prefix}face_vertices": mesh.face_vertices,
            f"{prefix}face_elems": mesh.face_elems,
            f"{prefix}face_local": mesh.face_local,
            f"{prefix}face_perm": mesh.face_perm,
            f"{prefix}face_normals": mesh.face_normals,
            f"{prefix}face_measures": mesh.face_measures,
            f"{prefix}face_tags": mesh.face_tags,
            f"{prefix}detJ": detJ, f"{prefix}Jinv": Jinv}


def scaled(mesh, lengths):
    v = mesh.vertices * np.asarray(lengths)[None, :]
    tags = {tuple(int(x) for x in mesh.face_vertices[f]): int(mesh.face_tags[f])
            for f in np.flatnonzero(mesh.boundary_mask)}
    return Mesh(v, mesh.elements, tags)


def jittered_square(nx, ny, lengths, amp, seed):
    base = unit_square(nx, ny)
    v = base.vertices * np.asarray(lengths)[None, :]
    rng = np.random.default_rng(seed)
    h = np.asarray(lengths) / np.array([nx, ny])
    shift = rng.uniform(-amp, amp, size=v.shape) * h[None, :]
    vi = np.arange(len(v)) % (nx + 1)
    vj = np.arange(len(v)) // (nx + 1)
    interior = (vi > 0) & (vi < nx) & (vj > 0) & (vj < ny)
    v = v.copy()
    v[interior] += shift[interior]
    tags = {tuple(int(x) for x in base.face_vertices[f]): int(base.face_tags[f])
            for f in np.flatnonzero(base.boundary_mask)}
    return Mesh(v, base.elements, tags)


def kuhn_cube_z0_gamma1(n):
    """C4-style tags: z=0 GAMMA1, everything else NO_FLOW."""
    m = unit_cube(n)
    tags = {}
    for f in np.flatnonzero(m.boundary_mask):
        key = tuple(int(x) for x in m.face_vertices[f])
        z = m.vertices[list(key), 2]
        if np.all(z == 0.0):
            tags[key] = int(BoundaryTag.GAMMA1)
    return Mesh(m.vertices, m.elements, tags)


def tables():
    out = {}
    for dim, kmax in ((2, 4), (3, 4)):
        for k in range(kmax + 1):
            b = BasisSet(dim, k)
            out[f"basis_coeff_{dim}_{k}"] = b._coeff
            pts = grundmann_moeller(dim, max(1, k))
            out[f"basis_eval_{dim}_{k}"] = b.eval(pts.points)
            out[f"basis_grad_{dim}_{k}"] = b.grad(pts.points)
    for dim in (1, 2, 3):
        for s in range(7):
            r = grundmann_moeller(dim, s)
            out[f"gm_points_{dim}_{s}"] = r.points
            out[f"gm_weights_{dim}_{s}"] = r.weights
    for deg in range(12):
        r = gauss_segment(deg)
        out[f"gauss_points_{deg}"] = r.points
        out[f"gauss_weights_{deg}"] = r.weights
    for dim in (2, 3):
        fr = face_rule(dim, 8)
        for lf in range(dim + 1):
            for pm in range(2 if dim == 2 else 6):
                out[f"frp_{dim}_{lf}_{pm}"] = face_reference_points(
                    dim, lf, pm, fr.points)
    np.savez_compressed(os.path.join(HERE, "tables.npz"), **out)


def meshes():
    out = {}
    out.update(mesh_arrays(unit_square(3), "sq3_"))
    out.update(mesh_arrays(unit_square(5, 2), "sq52_"))
    out.update(mesh_arrays(scaled(unit_square(8, 2), (4.0, 1.0)), "rect82_"))
    out.update(mesh_arrays(jittered_square(8, 2, (4.0, 1.0), 0.1, 3), "jit82_"))
    out.update(mesh_arrays(unit_cube(2), "cube2_"))
    out.update(mesh_arrays(unit_cube(3, 2, 2), "cube322_"))
    out.update(mesh_arrays(kuhn_cube_z0_gamma1(2), "cubez2_"))
    np.savez_compressed(os.path.join(HERE, "meshes.npz"), **out)


# --------------------------------------------------------------- operator

AMPLIFIED = dict(chi11_a=1.0, chi13_a=0.6, chi21_a=0.8, chi2n_a=0.7,
                 c1_star=0.12, c1_starstar=0.13)


def operator_cases():
    """(name, mesh key, order, model kind, param overrides, scheme, seed).

    The metadata is stored next to the arrays so the tests rebuild the
    exact same case with the product's setup code."""
    amp = AMPLIFIED
    cases = []
    for scheme in ("cdg2", "cdg", "br2", "ip", "bo"):
        cases.append((f"sq4_p2_{scheme}", "sq4", 2, "plaque", {}, scheme, 11))
        cases.append((f"sq4_p2_amp_{scheme}", "sq4", 2, "plaque", amp,
                      scheme, 12))
    for k in (0, 1, 3):
        cases.append((f"sq4_p{k}_amp_cdg2", "sq4", k, "plaque", amp, "cdg2",
                      13 + k))
    cases.append(("sq4_p2_smooth_cdg2", "sq4", 2, "plaque",
                  dict(eps_h=0.02, **amp), "cdg2", 17))
    cases.append(("rect82_p2_cdg2", "rect82", 2, "plaque", amp, "cdg2", 18))
    cases.append(("jit82_p3_cdg2", "jit82", 3, "plaque", amp, "cdg2", 19))
    cases.append(("jit82_p3_br2", "jit82", 3, "plaque", amp, "br2", 20))
    for scheme in ("cdg2", "br2", "ip", "cdg", "bo"):
        cases.append((f"cube2_p2_{scheme}", "cube2", 2, "plaque", amp,
                      scheme, 21))
    cases.append(("cube2_p1_cdg2", "cube2", 1, "plaque", amp, "cdg2", 22))
    cases.append(("cube2_p3_cdg2", "cube2", 3, "plaque", amp, "cdg2", 23))
    cases.append(("cubez2_p2_cdg2", "cubez2", 2, "plaque", {}, "cdg2", 24))
    cases.append(("sq4_p2_reduced_cdg2", "sq4", 2, "reduced", amp, "cdg2",
                  27))
    cases.append(("cube2_p2_reduced_br2", "cube2", 2, "reduced", amp, "br2",
                  28))
    return cases


MESHES = {
    "sq4": lambda: unit_square(4),
    "rect82": lambda: scaled(unit_square(8, 2), (4.0, 1.0)),
    "jit82": lambda: jittered_square(8, 2, (4.0, 1.0), 0.1, 3),
    "cube2": lambda: unit_cube(2),
    "cubez2": lambda: kuhn_cube_z0_gamma1(2),
}


def operators():
    import json
    out = {}
    for name, mkey, k, kind, over, scheme, seed in operator_cases():
        mesh = MESHES[mkey]()
        params = PlaqueParams(**over)
        model = PlaqueModel(params) if kind == "plaque" else ReducedModel(params)
        space = DGSpace(mesh, k, n_species=model.n_species)
        lo = mesh.vertices.min(axis=0)
        hi = mesh.vertices.max(axis=0)
        U = space.project(bump_field(mesh.dim, model.n_species, seed, lo,
                                     hi)).coeffs
        op = DiscreteOperator(space, model, FluxScheme(scheme))
        out[f"{name}__meta"] = np.array(json.dumps(
            {"mesh": mkey, "order": k, "model": kind, "params": over,
             "scheme": scheme, "seed": seed}))
        out[f"{name}__U"] = U
        out[f"{name}__R"] = op.apply(U, 0.0)
        out[f"{name}__F"] = op.apply_f(U, 0.0)
    np.savez_compressed(os.path.join(HERE, "operator.npz"), **out)


def heat_cases():
    """Linear diffusion: ZeroFluxHeat and ConstantDirichletHeat (mirror
    ghost) from the reference test oracles, plus the dense diffusion
    matrix of the reference's independent loop oracle."""
    out = {}
    rng = np.random.default_rng(5)
    two = Mesh(np.array([[0.0, 0.0], [1.0, 0.0], [1.0, 1.0], [0.0, 1.0]]),
               np.array([[0, 1, 2], [0, 2, 3]]))
    for mname, mesh in (("two", two), ("sq2", unit_square(2))):
        for k in (1, 2):
            for scheme in ("cdg2", "br2", "ip"):
                for dirichlet in (False, True):
                    space = DGSpace(mesh, k)
                    R = oracles.dense_diffusion_matrix(space, 0.35, scheme,
                                                       dirichlet=dirichlet)
                    out[f"dense_{mname}_{k}_{scheme}_{int(dirichlet)}"] = R
    for scheme in ("cdg2", "cdg", "br2", "ip", "bo"):
        for dirichlet in (False, True):
            mesh = unit_square(3)
            space = DGSpace(mesh, 2)
            model = (oracles.ConstantDirichletHeat(0.4, 0.7, 2) if dirichlet
                     else oracles.ZeroFluxHeat(0.7))
            op = DiscreteOperator(space, model, FluxScheme(scheme))
            U = rng.standard_normal(space.shape)
            key = f"heat_sq3_{scheme}_{int(dirichlet)}"
            out[f"{key}__U"] = U
            out[f"{key}__R"] = op.apply(U, 0.0)
    np.savez_compressed(os.path.join(HERE, "heat.npz"), **out)


def ssprk3(op, U, dt, steps):
    """Shu-Osher SSP-RK3 as a composition of the reference apply_f."""
    for _ in range(steps):
        U1 = U + dt * op.apply_f(U, 0.0)
        U2 = 0.75 * U + 0.25 * (U1 + dt * op.apply_f(U1, 0.0))
        U = U / 3.0 + (2.0 / 3.0) * (U2 + dt * op.apply_f(U2, 0.0))
    return U


def trajectories():
    out = {}
    # C1: unit_square(32), p=1, 6 species, cdg2, default coefficients,
    # 10 SSP-RK3 steps at dt = 8.0e-4 (0.8 * 2.51 / rho(J))
    mesh = unit_square(32)
    space = DGSpace(mesh, 1, n_species=6)
    U0 = space.project(bump_field(2, 6, 1, np.zeros(2), np.ones(2))).coeffs
    op = DiscreteOperator(space, PlaqueModel(), FluxScheme("cdg2"))
    out["c1__U0"] = U0
    out["c1__dt"] = np.array(8.0e-4)
    out["c1__U10"] = ssprk3(op, U0, 8.0e-4, 10)
    # C2/C4-style small replicas: p=2 rectangle, amplified taxis, 5 steps
    mesh = scaled(unit_square(16, 4), (4.0, 1.0))
    space = DGSpace(mesh, 2, n_species=6)
    op = DiscreteOperator(space, PlaqueModel(PlaqueParams(**AMPLIFIED)),
                          FluxScheme("cdg2"))
    U0 = space.project(bump_field(2, 6, 2, np.zeros(2),
                                  np.array([4.0, 1.0]))).coeffs
    out["rect164__U0"] = U0
    out["rect164__U5"] = ssprk3(op, U0, 2e-5, 5)
    mesh = kuhn_cube_z0_gamma1(3)
    space = DGSpace(mesh, 2, n_species=6)
    op = DiscreteOperator(space, PlaqueModel(), FluxScheme("cdg2"))
    U0 = space.project(bump_field(3, 6, 4, np.zeros(3), np.ones(3))).coeffs
    out["cubez3__U0"] = U0
    out["cubez3__U3"] = ssprk3(op, U0, 2e-4, 3)
    # implicit: SDIRK3 + JFNK with tightened tolerances
    mesh = unit_square(4)
    space = DGSpace(mesh, 2, n_species=6)
    op = DiscreteOperator(space, PlaqueModel(), FluxScheme("cdg2"))
    U0 = space.project(bump_field(2, 6, 9, np.zeros(2), np.ones(2))).coeffs
    res = integrate(op, U0, 0.0, math.inf, 0.01, order=3,
                    newton_kwargs={"rtol": 1e-11, "atol": 1e-13,
                                   "gmres_rtol": 1e-6},
                    n_steps=2)
    out["sdirk__U0"] = U0
    out["sdirk__U2"] = res.U
    out["sdirk__dt"] = np.array(0.01)
    np.savez_compressed(os.path.join(HERE, "trajectories.npz"), **out)


# rho(J) ~ C nu_max / h^2 per (d, k) (measured on the reference)
RHO_C = {(2, 1): 490.0, (2, 2): 1717.0, (2, 3): 4371.0, (3, 2): 7150.0, (3, 3): 16361.0}


def cfl_dt(mesh, d, k):
    """The configs' explicit step 0.8 * 2.51 / rho, rho = C nu_max / h^2."""
    h = float(mesh.diameters.min())
    return 0.8 * 2.51 / (RHO_C[(d, k)] * 1e-2 / h ** 2)


def trajectories_stated():
    """Every BASELINE config at its STATED step count on a scaled replica
    (same physics, order, flux, tags and stepping), run by
    the reference: C2 100 SSP-RK3 steps, C4 20 steps (cdg2, br2, ip),
    C5 10 steps at p=3 in 3D, C3 50 SDIRK3 steps on a jittered p=3 mesh
    at the stiffness ratio dt a_ii rho = 500 (tightened Newton / GMRES
    tolerances)."""
    out = {}

    def run(key, mesh, k, box, seed, steps, schemes=("cdg2",)):
        space = DGSpace(mesh, k, n_species=6)
        d = mesh.dim
        U0 = space.project(bump_field(d, 6, seed, np.zeros(d), np.asarray(box, float))).coeffs
        dt = cfl_dt(mesh, d, k)
        out[f"{key}__U0"] = U0
        out[f"{key}__dt"] = np.array(dt)
        out[f"{key}__steps"] = np.array(steps)
        for name in schemes:
            tic = time.perf_counter()
            op = DiscreteOperator(space, PlaqueModel(), FluxScheme(name))
            out[f"{key}__{name}__U"] = ssprk3(op, U0, dt, steps)
            print(f"  {key} {name}: {time.perf_counter() - tic:.1f}s", flush=True)

    # C2: [0,4]x[0,1], p=2, 100 SSP-RK3 steps
    run("c2r", scaled(unit_square(16, 4), (4.0, 1.0)), 2, (4.0, 1.0), 2, 100)
    # C4: unit cube, z=0 GAMMA1 / no-flow elsewhere, p=2, 20 steps, + br2 / ip
    run("c4r", kuhn_cube_z0_gamma1(3), 2, (1.0, 1.0, 1.0), 4, 20, ("cdg2", "br2", "ip"))
    # C5: [0,2]x[0,1]^2 with the generator's default tags, p=3, 10 steps
    run("c5r", scaled(unit_cube(4, 2, 2), (2.0, 1.0, 1.0)), 3, (2.0, 1.0, 1.0), 5, 10)
    # C3: jittered [0,4]x[0,1], p=3, 50 SDIRK3 + JFNK steps
    mesh = jittered_square(8, 2, (4.0, 1.0), 0.1, 7)
    space = DGSpace(mesh, 3, n_species=6)
    U0 = space.project(bump_field(2, 6, 3, np.zeros(2), np.array([4.0, 1.0]))).coeffs
    h = float(mesh.diameters.min())
    gamma = 0.4358665215
    dt = 500.0 / (gamma * RHO_C[(2, 3)] * 1e-2 / h ** 2)
    nk = {"rtol": 1e-10, "atol": 1e-13, "gmres_rtol": 1e-4, "gmres_maxiter": 400}
    op = DiscreteOperator(space, PlaqueModel(), FluxScheme("cdg2"))
    tic = time.perf_counter()
    res = integrate(op, U0, 0.0, math.inf, dt, order=3, newton_kwargs=nk, n_steps=50)
    print(f"  c3r sdirk3: {time.perf_counter() - tic:.1f}s, {res.gmres_iterations} GMRES",
          flush=True)
    out["c3r__U0"] = U0
    out["c3r__dt"] = np.array(dt)
    out["c3r__U50"] = res.U
    out["c3r__nk"] = np.array([nk["rtol"], nk["atol"], nk["gmres_rtol"], nk["gmres_maxiter"]])
    np.savez_compressed(os.path.join(HERE, "trajectories_stated.npz"), **out)


def diagnostics():
    """Reference output formats for the device diagnostics: a VTK snapshot
    (vtkio.write_vtk) and species totals (DiscreteFunction.species_totals)
    of seeded states on a 2D and a 3D mesh."""
    import tempfile
    from taxisdg.vtkio import write_vtk
    out = {}
    for key, mesh, k in (("sq3", unit_square(3), 2), ("cube1", unit_cube(1), 1)):
        d = mesh.dim
        space = DGSpace(mesh, k, n_species=6)
        U = space.project(bump_field(d, 6, 13, np.zeros(d), np.ones(d))).coeffs
        fn = space.function(U)
        with tempfile.TemporaryDirectory() as tmp:
            path = write_vtk(os.path.join(tmp, "s.vtk"), fn,
                             names=["n1", "n2", "n3", "c1", "c2", "c3"])
            text = open(path).read()
        out[f"{key}__U"] = U
        out[f"{key}__vtk"] = np.array(text)
        out[f"{key}__totals"] = fn.species_totals()
    np.savez_compressed(os.path.join(HERE, "diagnostics.npz"), **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["tables", "meshes", "operators", "heat_cases", "trajectories",
                             "trajectories_stated", "diagnostics"]
    for fn in (globals()[w] for w in which):
        tic = time.perf_counter()
        fn()
        print(f"{fn.__name__}: {time.perf_counter() - tic:.1f}s", flush=True)
