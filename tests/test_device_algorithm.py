"""The kernels' reformulated arithmetic (emulated in numpy from the same
packed tables the device receives) against the reference's golden
outputs.  Pins the reformulation (exact-stiffness diffusion, jn-only
face terms, modal linear source) on CPU; the GPU tests then pin the
kernels themselves."""
import numpy as np
import pytest

from paper_1403_1157_b200 import DGSpace, DiffusionModel, FluxScheme, unit_square
from paper_1403_1157_b200.tables import build_tables, scheme_constants

from _cases import operator_case
from _device_emulator import DeviceEmulator
from test_oracle_golden import _golden_names


def _emulate(space, model, scheme, U, **kw):
    t = build_tables(space, model, scheme)
    em = DeviceEmulator(t, model, scheme.id, *scheme_constants(space, scheme), **kw)
    return em.apply(U)


@pytest.mark.parametrize("name", [n for n in _golden_names() if "_p0_" not in n])
def test_emulated_kernels_match_reference(golden, name):
    space, model, scheme, U, R, _ = operator_case(golden, name)
    got = _emulate(space, model, scheme, U)
    assert np.abs(got - R).max() <= 1e-12 * np.abs(R).max()


@pytest.mark.parametrize("name", [n for n in _golden_names()
                                  if "_p0_" not in n and n.startswith(("sq", "jit", "rect"))])
def test_emulated_signature_run_order_matches_reference(golden, name):
    """The 2D signature-run kernel's operation order (csrc/kernels_sig_body.cuh:
    normal derivative after the contraction, adjoint term projected with
    (X jn) . grad phi) against the same golden outputs."""
    space, model, scheme, U, R, _ = operator_case(golden, name)
    if space.mesh.dim != 2:
        pytest.skip("2D kernel")
    got = _emulate(space, model, scheme, U, normal_after=True)
    assert np.abs(got - R).max() <= 1e-12 * np.abs(R).max()


@pytest.mark.parametrize("scheme", ["cdg2", "cdg", "br2", "ip", "bo"])
@pytest.mark.parametrize("dirichlet", [0, 1])
def test_emulated_heat(golden, scheme, dirichlet):
    h = golden["heat"]
    space = DGSpace(unit_square(3), 2)
    model = DiffusionModel(0.7, dirichlet=0.4 if dirichlet else None)
    key = f"heat_sq3_{scheme}_{dirichlet}"
    R = h[f"{key}__R"]
    got = _emulate(space, model, FluxScheme(scheme), h[f"{key}__U"])
    assert np.abs(got - R).max() <= 1e-12 * np.abs(R).max()
