"""Parity at every BASELINE config's STATED step count (north_star: per-
species relative broken-L2 <= 1e-10 "after the stated number of steps"),
on scaled replicas the live reference ran (tests/golden/make_golden.py
``trajectories_stated``: same physics, order, flux, tags and stepping),
plus the reference acceptance checks that run on the device.

C1 (10 SSP-RK3 steps) is in test_gpu_operator.py.  Reference call sites:
``timeint.py:347-380`` (integrate), ``tests/test_acceptance.py:298-339``
(lipid balance), ``tests/test_operator.py:141-151`` (quadrature
override)."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_1403_1157_b200 import (BoundaryTag, DGSpace, DiffusionModel,  # noqa: E402
                                  FluxScheme, PlaqueModel, PlaqueParams,
                                  unit_cube, unit_square)
from paper_1403_1157_b200.mesh import Mesh  # noqa: E402

from _cases import rel_l2_per_species  # noqa: E402

pytestmark = pytest.mark.gpu
TOL_L2 = 1e-10


def _op(space, model, scheme, **kw):
    from paper_1403_1157_b200.operator import DiscreteOperator
    return DiscreteOperator(space, model, scheme, **kw)


def _jittered(nx, ny, lengths, amp, seed):
    """make_golden.jittered_square: the reference unit_square's vertices,
    scaled, interior vertices moved by U(-amp h, amp h) (this generator's
    RNG stream differs from unit_square(jitter=...))."""
    base = unit_square(nx, ny)
    v = base.vertices * np.asarray(lengths)[None, :]
    rng = np.random.default_rng(seed)
    h = np.asarray(lengths) / np.array([nx, ny])
    shift = rng.uniform(-amp, amp, size=v.shape) * h[None, :]
    vi, vj = np.arange(len(v)) % (nx + 1), np.arange(len(v)) // (nx + 1)
    interior = (vi > 0) & (vi < nx) & (vj > 0) & (vj < ny)
    v = v.copy()
    v[interior] += shift[interior]
    tags = {tuple(int(x) for x in base.face_vertices[f]): int(base.face_tags[f])
            for f in np.flatnonzero(base.boundary_mask)}
    return Mesh(v, base.elements, tags)


STATED = {
    "c2r": (lambda: unit_square(16, 4, lengths=(4.0, 1.0)), 2, ("cdg2",)),
    "c4r": (lambda: unit_cube(3, gamma1_in=None, top_tag=BoundaryTag.NO_FLOW), 2,
            ("cdg2", "br2", "ip")),
    "c5r": (lambda: unit_cube(4, 2, 2, lengths=(2.0, 1.0, 1.0)), 3, ("cdg2",)),
}


@pytest.mark.parametrize("key,scheme", [(k, s) for k, v in STATED.items() for s in v[2]])
def test_explicit_configs_at_their_stated_step_counts(golden, key, scheme):
    """C2 100, C4 20 (cdg2 / br2 / ip) and C5 (3D p=3) 10 SSP-RK3 steps
    through tdg_ssprk3_step against the reference's trajectory."""
    g = golden["trajectories_stated"]
    mesh_fn, k, _ = STATED[key]
    space = DGSpace(mesh_fn(), k, 6)
    op = _op(space, PlaqueModel(), FluxScheme(scheme))
    U = torch.from_numpy(g[f"{key}__U0"]).cuda()
    work = op.new_work()
    steps, dt = int(g[f"{key}__steps"]), float(g[f"{key}__dt"])
    for _ in range(steps):
        op.ssprk3_step(U, work, dt)
    ref = g[f"{key}__{scheme}__U"]
    err = rel_l2_per_species(space, U.cpu().numpy(), ref)
    assert err.max() <= TOL_L2, err
    # the trajectory moved far more than the tolerance
    assert rel_l2_per_species(space, g[f"{key}__U0"], ref).max() > 1e4 * TOL_L2


def test_c3_sdirk3_at_its_stated_step_count(golden):
    """C3 replica (jittered [0,4]x[0,1], p=3): 50 SDIRK3 + JFNK steps at the
    stiffness ratio dt a_ii rho = 500 with the reference's own stepper
    settings as make_golden ran them, through the device JFNK/GMRES."""
    from paper_1403_1157_b200.timeint import integrate
    g = golden["trajectories_stated"]
    space = DGSpace(_jittered(8, 2, (4.0, 1.0), 0.1, 7), 3, 6)
    op = _op(space, PlaqueModel(), FluxScheme("cdg2"))
    rtol, atol, grtol, gmax = (float(x) for x in g["c3r__nk"])
    res = integrate(op, g["c3r__U0"], 0.0, math.inf, float(g["c3r__dt"]), order=3,
                    n_steps=50, newton_kwargs={"rtol": rtol, "atol": atol,
                                               "gmres_rtol": grtol, "gmres_maxiter": int(gmax)})
    err = rel_l2_per_species(space, res.U, g["c3r__U50"])
    assert err.max() <= TOL_L2, err


def _seeded_plaque_state(space, seed=11):
    from paper_1403_1157_b200.fields import initial_state
    return initial_state(space, seed)


def test_lipid_balance_over_100_sdirk3_steps():
    """Reference tests/test_acceptance.py:298-339 on the device: sealed
    walls keep c2 + c3 invariant over 100 SDIRK3 steps (drift <= 1e-8);
    from zero with inflow only, the lipid budget grows at sigma |Gamma1,in|
    per unit time (<= 1 %)."""
    from paper_1403_1157_b200.timeint import integrate
    closed = PlaqueModel(PlaqueParams(sigma=0.0, beta1=0.0, beta2=0.0))
    mesh = unit_square(8)
    space = DGSpace(mesh, 2, 6)
    op = _op(space, closed, FluxScheme("cdg2"))
    U0 = _seeded_plaque_state(space)
    res = integrate(op, U0, 0.0, math.inf, 0.01, order=3, n_steps=100,
                    newton_kwargs={"rtol": 1e-11, "atol": 1e-13, "gmres_rtol": 1e-6})
    assert res.steps == 100
    tot0 = space.function(U0).species_totals()
    tot1 = space.function(res.U).species_totals()
    drift = abs((tot1[4] + tot1[5]) - (tot0[4] + tot0[5])) / abs(tot0[4] + tot0[5])
    assert drift <= 1e-8, drift
    inflow = PlaqueModel(PlaqueParams(sigma=1.0, nu2=1.0, beta1=0.0, beta2=0.0))
    op2 = _op(space, inflow, FluxScheme("cdg2"))
    res2 = integrate(op2, space.zeros(), 0.0, math.inf, 0.01, order=3, n_steps=50,
                     newton_kwargs={"rtol": 1e-8, "atol": 1e-11})
    tot2 = space.function(res2.U).species_totals()
    expected = 1.0 * mesh.boundary_measure(BoundaryTag.GAMMA1_IN) * 50 * 0.01
    assert abs(tot2[4] + tot2[5] - expected) / expected <= 0.01


def test_quadrature_degree_override():
    """Reference tests/test_operator.py:141-151: a lower quadrature degree
    (vol_degree = face_degree = 2, through the generic kernels) integrates
    linear data exactly, like the default rule."""
    space = DGSpace(unit_square(2), 1)
    model = DiffusionModel(1.0)
    lo = _op(space, model, FluxScheme("br2"), vol_degree=2, face_degree=2)
    hi = _op(space, model, FluxScheme("br2"))
    assert lo.tables.nq_vol < hi.tables.nq_vol and lo.tables.nq_face < hi.tables.nq_face
    fn = space.project(lambda x: x[..., 0][..., None])
    assert np.allclose(lo.apply(fn.coeffs), hi.apply(fn.coeffs), atol=1e-13)


def test_reference_style_stepper_over_numpy_apply_f(golden):
    """The drop-in at the reference's own call shape: the reference's SDIRK3
    + JFNK stepper (restated in numpy, oracle.sdirk_integrate, reference
    timeint.py:137-380) calling the device operator's apply_f(numpy) ->
    numpy exactly as it calls the reference operator, against the
    reference's own trajectory."""
    from oracle import sdirk_integrate
    t = golden["trajectories"]
    space = DGSpace(unit_square(4), 2, 6)
    op = _op(space, PlaqueModel(), FluxScheme("cdg2"))
    U = sdirk_integrate(op, t["sdirk__U0"], 0.01, 2,
                        newton_kwargs={"rtol": 1e-11, "atol": 1e-13, "gmres_rtol": 1e-6})
    err = rel_l2_per_species(space, U, t["sdirk__U2"])
    assert err.max() <= TOL_L2, err


def test_integrate_hands_numpy_to_callbacks():
    """integrate() with a numpy U0 calls back with numpy states, like the
    reference (timeint.py:376-378), so reference callbacks such as
    space.function(U).species_totals() (analysis.conservation_audit,
    scenarios' balance.csv) work unchanged."""
    from paper_1403_1157_b200.timeint import integrate
    space = DGSpace(unit_square(4), 1, 6)
    op = _op(space, PlaqueModel(), FluxScheme("cdg2"))
    U0 = _seeded_plaque_state(space)
    seen = []

    def record(step, t, U):
        assert isinstance(U, np.ndarray) and U.shape == space.shape
        seen.append(space.function(U).species_totals())

    res = integrate(op, U0, 0.0, math.inf, 0.01, order=3, n_steps=3, callback=record)
    assert len(seen) == 3 and isinstance(res.U, np.ndarray)
    assert np.allclose(seen[-1], space.function(res.U).species_totals(), rtol=0, atol=0)


def test_c2_full_size_against_oracle_port():
    """Full-size C2 (512x128 cells, p=2, 4.7M DoFs): SSP-RK3 steps on the
    device against the same steps of the pinned CPU oracle port
    (oracle/taxis_oracle.py, checked against the reference's golden outputs
    in tests/test_oracle_golden.py; reference operator.py:253-288).  20 steps
    by default (about half a minute of CPU work on 16 cores); TDG_LONG=1
    runs the config's stated 100 steps (three minutes: 1 passed in 185.7 s
    on the B200 box, profiles/r02_c2_full_100_steps.log)."""
    import os
    from threadpoolctl import threadpool_limits
    from oracle import OracleOperator
    from paper_1403_1157_b200.fields import initial_state
    space = DGSpace(unit_square(512, 128, lengths=(4.0, 1.0)), 2, 6)
    model, scheme = PlaqueModel(), FluxScheme("cdg2")
    U0 = initial_state(space, 2)
    dt = 1.43e-5                      # 0.8 * 2.51 / rho at C2
    steps = 100 if os.environ.get("TDG_LONG") == "1" else 20
    op = _op(space, model, scheme)
    U = torch.from_numpy(U0).cuda()
    work = op.new_work()
    for _ in range(steps):
        op.ssprk3_step(U, work, dt)
    got = U.cpu().numpy()
    try:
        import psutil
        cores = psutil.cpu_count(logical=False) or os.cpu_count() or 1
    except ImportError:
        cores = os.cpu_count() or 1
    ref_op = OracleOperator(space, model, scheme, nthreads=max(1, min(cores, 32)))
    V = U0.copy()
    with threadpool_limits(1):
        for _ in range(steps):
            V1 = V + dt * ref_op.apply_f(V)
            V2 = 0.75 * V + 0.25 * (V1 + dt * ref_op.apply_f(V1))
            V = V / 3.0 + (2.0 / 3.0) * (V2 + dt * ref_op.apply_f(V2))
    err = rel_l2_per_species(space, got, V)
    assert err.max() <= TOL_L2, err
    assert rel_l2_per_species(space, U0, V).max() > 1e3 * TOL_L2
