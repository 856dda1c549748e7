"""Modal formulation of the 3D face operator (tables.modal_face_factors,
the face-group kernel's algebra), checked on the CPU against the direct
per-point face terms of the device emulator (reference operator.py:326-424
restated): every interior face of small Kuhn meshes, all five schemes,
p = 1..3, amplified taxis so both LLF branches and every lifting side run.
"""
import numpy as np
import pytest

from paper_1403_1157_b200 import DGSpace, FluxScheme, PlaqueModel, PlaqueParams
from paper_1403_1157_b200.mesh import unit_cube, unit_square
from paper_1403_1157_b200.tables import (build_tables, face_classes, modal_face_factors,
                                         scheme_constants)
from paper_1403_1157_b200.fields import initial_state

from _cases import AMPLIFIED
from _device_emulator import DeviceEmulator

CIN = 1 << 10


def _modal_face(em, mf, cls_in, cls_out, U, code, ein, eout, g):
    """One interior face through the modal factors (no per-point traces of
    the full basis; pointwise work only for the LLF flux)."""
    t = em.t
    d, S = t.dim, t.n_species
    A = em.A
    tin, tout = code & 31, (code >> 5) & 31
    sfac, h, idi, ido = g[2 * d:2 * d + 4]
    Bf, Bd, T, Td, L, Mff, Mfd = (mf[k] for k in ("Bf", "Bd", "T", "Td", "L", "Mff", "Mfd"))
    ci, co = U[ein], U[eout]
    a_in, a_out = ci @ T[tin].T, co @ T[tout].T           # (S, nfm)
    d_in, d_out = ci @ Td[cls_in].T, co @ Td[cls_out].T   # (S, ndm)
    a_j = a_in - a_out + (ci @ mf["Tlo"][tin].T - co @ mf["Tlo"][tout].T)
    gm = 0.5 * (d_in + d_out)
    ui, uo = a_in @ Bf.T, a_out @ Bf.T                    # (S, F) physics inputs
    gn = gm @ Bd.T
    dU = ui - uo
    cnv = np.zeros((t.nq_face, S))
    em._conv(ui.T, uo.T, gn.T, dU.T, cnv)
    w = t.face_w
    Ybr = A[:, None] * (gm @ Mfd.T) - (cnv.T * w[None, :]) @ Bf
    name = em.scheme
    if name == 3:       # ip
        Ybr -= (em.eta / h) * A[:, None] * (a_j @ Mff.T)
    elif name != 4:     # cdg2 / cdg / br2
        br2 = name == 2
        wside = 0.5 if br2 else 1.0
        fac0 = (4.0 if name == 1 else 2.0) * em.chi_e * wside * 0.5 * sfac * A[:, None]
        if br2 or (code & CIN):
            Ybr -= fac0 * idi * (a_j @ L[tin].T)
        if br2 or not (code & CIN):
            Ybr -= fac0 * ido * (a_j @ L[tout].T)
    Xbr = 0.5 * em.adj * A[:, None] * (a_j @ Mfd)
    ri = sfac * (Ybr @ T[tin] + Xbr @ Td[cls_in])
    ro = sfac * (-Ybr @ T[tout] + Xbr @ Td[cls_out])
    return ri, ro


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("order", [1, 2, 3])
@pytest.mark.parametrize("scheme", ["cdg2", "cdg", "br2", "ip", "bo"])
def test_modal_face_terms_match_direct(dim, order, scheme):
    space = DGSpace(unit_cube(2, 2, 2) if dim == 3 else unit_square(4, 3), order, 6)
    model = PlaqueModel(PlaqueParams(**AMPLIFIED))
    sch = FluxScheme(scheme)
    t = build_tables(space, model, sch)
    fold = face_classes(t)
    mf = modal_face_factors(t, fold)
    chi_e, adj, eta = scheme_constants(space, sch)
    em = DeviceEmulator(t, model, sch.id, chi_e, adj, eta)
    U = initial_state(space, 41)
    worst = 0.0
    for f in range(len(t.if_code)):
        code = int(t.if_code[f])
        ein, eout = t.if_elems[f]
        ri, ro = em.face_contrib(U, code, ein, eout, t.if_geo[f])
        mi, mo = _modal_face(em, mf, fold[0][f, 0], fold[0][f, 1], U, code, ein, eout,
                             t.if_geo[f])
        scale = max(np.abs(ri).max(), np.abs(ro).max())
        worst = max(worst, np.abs(mi - ri).max() / scale, np.abs(mo - ro).max() / scale)
    assert worst <= 1e-12, worst


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("order", [1, 2, 3])
def test_modal_factors_reconstruct_the_tables(dim, order):
    """Bf T = face_B and Bd Td = the folded normal-derivative tables, with
    orthonormal Bf, Bd (tables.modal_face_factors)."""
    space = DGSpace(unit_cube(2, 2, 2) if dim == 3 else unit_square(4, 3), order, 6)
    t = build_tables(space, PlaqueModel(), FluxScheme("cdg2"))
    fold = face_classes(t)
    mf = modal_face_factors(t, fold)
    assert np.allclose(mf["Bf"].T @ mf["Bf"], np.eye(mf["nfm"]), atol=1e-13)
    for k in range(t.face_B.shape[0]):
        assert np.abs(mf["Bf"] @ mf["T"][k] - t.face_B[k]).max() <= 1e-14 * np.abs(t.face_B[k]).max()
    for c, (tab, jv) in enumerate(fold[1]):
        Gn = np.einsum("qia,a->qi", t.face_G[tab], jv)
        assert np.abs(mf["Bd"] @ mf["Td"][c] - Gn).max() <= 1e-12 * max(1, np.abs(Gn).max())
