"""Algorithmic work per operator application.

Flops follow the reference's own operation sequence (FMA = 2, div = 1,
max/abs/compare = 0; weights and metric folded into tables = 0; cdg2
lifting on K- only).  They are the numerator of every roofline fraction
this repo reports, so a kernel that does less work than the reference
(the CUDA kernels do: exact-stiffness diffusion, normal-derivative-only
face traces) is credited with the reference's work, and
``executed_flops`` is reported beside it.
"""

from __future__ import annotations

__all__ = ["vol_flops", "face_flops", "bface_flops", "apply_flops",
           "apply_bytes", "executed_flops", "executed_split", "modal_face_flops"]


def vol_flops(d, nb, Q, S=6):
    return 4 * Q * nb * S * (1 + d) + 4 * Q * S * d * d + Q * (28 + 8 * d + S * d) + S * nb


def face_flops(d, nb, F, S=6):
    return (4 * F * nb * S * (1 + d) + 8 * F * nb * S + 4 * d * F * nb
            + 4 * F * S * d * d + 6 * F * S * d + 2 * F * F * S + 16 * F * S
            + F * (50 + 38 * d) + 4 * d * d)


def bface_flops(d, nb, F, S=6):
    return 4 * F * nb * S + 6 * F + 2 * F * S


def apply_flops(d, nb, Q, F, ne, n_int, n_bnd, S=6):
    """(volume, interior faces, boundary faces) flops of one application."""
    return (ne * vol_flops(d, nb, Q, S), n_int * face_flops(d, nb, F, S),
            n_bnd * bface_flops(d, nb, F, S))


def apply_bytes(d, n_dofs, ne, n_int, n_bnd, rk_stage=True):
    """Compulsory HBM bytes of one application (+ the SSP-RK3 stage's
    U^n read, 2/3 of the stages)."""
    b = 16 * n_dofs + ne * 8 * (d * d + 1) + (n_int + n_bnd) * (8 * (d + 1) + 12)
    if rk_stage:
        b += 8 * n_dofs * 2 / 3
    return b


def modal_face_flops(d, k, nb, F, S=6):
    """Flops per interior face of the modal face kernel (csrc/kernels_tcm.cuh):
    face / d-modes of both sides, point values of the jump, u_in and gav,
    the LLF physics, the projection of the pointwise flux, the modal
    brackets (A Mfd g, lifting, adjoint term) and the back-projection to
    both sides' volume modes (no tensor-core padding)."""
    nfm, ndm = (k + 1) * (k + 2) // 2, k * (k + 1) // 2
    per_species = (4 * (nfm + ndm) * nb + 2 * F * (2 * nfm + ndm) + 2 * F * nfm
                   + 4 * nfm * ndm + 2 * nfm * nfm + 4 * (nfm + ndm) * nb)
    return S * per_species + 120 * F


def executed_split(d, nb, Q, F, ne, n_int, n_bnd, S=6, face_classes=False,
                   vol_classes=False, modal_order=None):
    """(volume, interior faces, boundary faces) flops of the reformulated
    sequence the kernels run (plaque model), without tensor-core padding:
    volume: values of 4 species and reference gradients of 3 at every
    point, 2 pulled-back flux rows + the bilinear source projected, exact
    stiffness diffusion (d(d+1)/2 metric-scaled GEMMs, or one per species
    against the element class's summed stiffness) and the modal linear
    source; faces: u and d_n u per side and species (Jinv n folded into the
    gradient tables per face, or precomputed per face-geometry class),
    lifting on one side, projection to both sides."""
    nsym = d * (d + 1) // 2
    vol = (Q * (2 * nb * (4 + 3 * d) + 2 * 3 * d * d + 40 + 2 * (2 * d * nb + nb))
           + S * nb * 2 * nb * (1 if vol_classes else nsym + 1) + S * nb * 2 * S)
    face = ((0 if face_classes else 2 * 2 * F * nb * d) + 2 * 2 * 2 * F * nb * S
            + 2 * F * F * S + F * 120 + 2 * 2 * 2 * F * nb * S)
    if modal_order is not None:   # the modal face kernel
        face = modal_face_flops(d, modal_order, nb, F, S)
    bface = 2 * F * nb + 2 * F * nb * S
    return ne * vol, n_int * face, n_bnd * bface


def executed_flops(d, nb, Q, F, ne, n_int, n_bnd, S=6, face_classes=False, vol_classes=False,
                   modal_order=None):
    """Sum of ``executed_split``."""
    return sum(executed_split(d, nb, Q, F, ne, n_int, n_bnd, S, face_classes, vol_classes,
                              modal_order))
