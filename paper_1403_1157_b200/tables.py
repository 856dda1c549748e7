"""Pack reference tables, geometry and the face lists for the device.

Host-side (numpy) construction of everything ``tdg_create`` consumes
(include/taxisdg_b200.h ``tdg_desc``).  Sources in the reference:

* volume tables Phi, Gref, w at degree 3k+1 and face tables B, G,
  Pw = (B B^T) w per (local face, permutation) at degree 3k+2
  (``operator.py:106-140``);
* per-face data of ``_build_groups`` (``operator.py:147-206``): inside /
  outside element, normal, sfac = measure / reference face measure,
  h = min neighbour diameter, K- flag (``flux.py:92-95``);
* element geometry detJ, Jinv (``mesh.py:267-277``).

Device layout choices (B200-first, not the reference's):

* the normal enters the face terms only through jn = Jinv n per side,
  so faces carry jn_in, jn_out (2d doubles) instead of n and two Jinv;
* the volume diffusion term uses the metric M = Jinv Jinv^T (symmetric,
  d(d+1)/2 doubles per element) and exact stiffness blocks
  KS_ac[j][i] = sum_q w_q G[q,j,c] G[q,i,a] (+ transpose for c != a),
  integrated with the reference's own rule;
* the faces are coloured (``tdg_color_faces``: elements = vertices, faces
  = edges) and run colour by colour, each colour one launch ("segment")
  in which no element is written twice: the faces add their two
  contribution blocks straight into the elements' face-sum rows, with no
  atomics and no per-face buffers, and the fixed segment order fixes
  every sum.  This replaces the reference's race-freedom device (private
  per-partition buffers merged in part order, ``operator.py:262-284``).
  Within a segment the faces are sorted by their (inside table, outside
  table) signature so a warp's table reads are uniform.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .fespace import DGSpace, face_reference_points
from .flux import FluxScheme, chi_factor, minus_is_outside
from .quadrature import face_rule, volume_rule

__all__ = ["OperatorTables", "build_tables", "color_faces", "sym_pairs"]

REF_FACE_MEASURE = {2: 1.0, 3: 0.5}
CODE_MINUS_IN = 1 << 10
CODE_MIRROR = 1 << 14
CODE_SKIP_OUT = 1 << 15
CODE_FIRST_IN = 1 << 16
CODE_FIRST_OUT = 1 << 17


def sym_pairs(d: int):
    return [(a, b) for a in range(d) for b in range(a, d)]


@dataclass
class OperatorTables:
    dim: int
    order: int
    n_species: int
    nb: int
    nq_vol: int
    nq_face: int
    vol_phi: np.ndarray
    vol_grad: np.ndarray
    vol_w: np.ndarray
    vol_stiff: np.ndarray
    face_B: np.ndarray
    face_G: np.ndarray
    face_Pw: np.ndarray
    face_w: np.ndarray
    elem_geo: np.ndarray
    if_elems: np.ndarray
    if_code: np.ndarray
    if_geo: np.ndarray
    bf_elem: np.ndarray
    bf_code: np.ndarray
    bf_geo: np.ndarray
    n_cut: int = 0
    # colour segments, run in order (the last n_seg_cut hold the faces
    # that read ghost rows): interior faces seg_if[s]..seg_if[s+1], walls
    # seg_bf[s]..seg_bf[s+1]; if_seg = segment of every interior face
    n_seg: int = 0
    n_seg_cut: int = 0
    seg_if: np.ndarray = None
    seg_bf: np.ndarray = None
    if_seg: np.ndarray = None
    # host-only: element-local face index per side (audit, emulator)
    if_lf: np.ndarray = None
    bf_lf: np.ndarray = None
    if_fid: np.ndarray = None   # mesh face id of every interior (+ mirror) face
    bf_fid: np.ndarray = None   # mesh face id of every wall face
    if_chunk: np.ndarray = None  # element chunk of every interior face (vol_chunk_bounds)
    bf_chunk: np.ndarray = None
    face_pts: np.ndarray = None  # face rule points (reference face coordinates)


def _face_tables(space: DGSpace, frule):
    d = space.mesh.dim
    nperm = 2 if d == 2 else 6
    Bs, Gs, Ps = [], [], []
    for lf in range(d + 1):
        for pm in range(nperm):
            xi = face_reference_points(d, lf, pm, frule.points)
            B = space.basis.eval(xi)
            Bs.append(B)
            Gs.append(space.basis.grad(xi))
            Ps.append((B @ B.T) * frule.weights[None, :])
    return np.stack(Bs), np.stack(Gs), np.stack(Ps)


def color_faces(elem_in, elem_out, n_elements, order=None):
    """Greedy colouring of the face graph (``tdg_color_faces``, host C++
    in the library): faces visited in ``order`` take the smallest colour
    none of their written elements (>= 0) holds.  Returns (colours, n)."""
    import ctypes
    from . import _native
    lib = _native.load()
    a = np.ascontiguousarray(elem_in, dtype=np.int32)
    b = np.ascontiguousarray(elem_out, dtype=np.int32)
    n = len(a)
    col = np.empty(n, dtype=np.int32)
    o = None if order is None else np.ascontiguousarray(order, dtype=np.int64)
    p = lambda x: ctypes.c_void_p(x.ctypes.data) if x is not None and len(x) else None
    nc = lib.tdg_color_faces(n, p(a), p(b), int(n_elements), p(o), p(col))
    _native.check(nc if nc < 0 else 0, "tdg_color_faces")
    return col, int(nc)


def _class_order(lf_in, lf_out, d):
    """Visit order of the greedy colouring: faces grouped by their
    (local face in, local face out) class (out = d+1 for one-sided faces);
    on the structured triangle / Kuhn meshes this gives d+1 colours."""
    klass = lf_in.astype(np.int64) * (d + 2) + np.where(lf_out >= 0, lf_out, d + 1)
    return np.lexsort((np.arange(len(klass)), klass))


def build_tables(space: DGSpace, model, scheme: FluxScheme,
                 vol_degree=None, face_degree=None, n_owned=None,
                 global_ids=None) -> OperatorTables:
    """Pack tables, element geometry and face lists.

    Slab-decomposed runs pass a local mesh whose first ``n_owned``
    elements are owned and the rest are ghosts, plus the ``global_ids``
    of all local elements (the K- tie rule breaks ties by global id).
    Faces with no owned side are dropped; a face whose inside is a ghost
    is flipped (the face terms are symmetric under swapping the sides up
    to roundoff); a face whose outside is a ghost writes only its inside
    slot (SKIP_OUT)."""
    mesh = space.mesh
    d, k, S, nb = mesh.dim, space.order, space.n_species, space.nb
    nperm = 2 if d == 2 else 6
    vr = volume_rule(d, 3 * k + 1 if vol_degree is None else vol_degree)
    fr = face_rule(d, 3 * k + 2 if face_degree is None else face_degree)
    phi = space.basis.eval(vr.points)
    grad = space.basis.grad(vr.points)
    K = np.einsum("q,qjc,qia->caji", vr.weights, grad, grad)  # [c][a][j][i]
    ks = []
    for c, a in sym_pairs(d):
        blk = K[c, a].copy()
        if c != a:
            blk += K[a, c]
        ks.append(blk)
    ks = np.stack(ks)
    fB, fG, fPw = _face_tables(space, fr)

    ne = mesh.n_elements
    n_owned = ne if n_owned is None else int(n_owned)
    gid = (np.arange(ne, dtype=np.int64) if global_ids is None
           else np.asarray(global_ids, dtype=np.int64))
    J, detJ, Jinv = mesh.jacobians()
    Mmet = np.einsum("eab,ecb->eac", Jinv, Jinv)
    egeo = np.concatenate([detJ[:, None]] + [Mmet[:, a, b][:, None]
                                             for a, b in sym_pairs(d)], axis=1)

    fe = mesh.face_elems.copy()
    fl = mesh.face_local.astype(np.int64)
    fp = mesh.face_perm.astype(np.int64)
    nrm = mesh.face_normals.copy()
    interior = fe[:, 1] >= 0
    owned = lambda e: (e >= 0) & (e < n_owned)
    flip = interior & ~owned(fe[:, 0]) & owned(fe[:, 1])
    fe[flip] = fe[flip][:, ::-1]
    fl[flip] = fl[flip][:, ::-1]
    fp[flip] = fp[flip][:, ::-1]
    nrm[flip] *= -1.0
    dirichlet = getattr(model, "boundary_kind", "flux") == "dirichlet"
    sfac_all = mesh.face_measures / REF_FACE_MEASURE[d]
    tid = fl * nperm + fp

    # interior faces (+ mirror faces for Dirichlet models)
    fi = np.flatnonzero(interior & owned(fe[:, 0]))
    ein, eout = fe[fi, 0], fe[fi, 1]
    n = nrm[fi]
    jin = np.einsum("fab,fb->fa", Jinv[ein], n)
    jout = np.einsum("fab,fb->fa", Jinv[eout], n)
    h = np.minimum(mesh.diameters[ein], mesh.diameters[eout])
    mi = ~minus_is_outside(mesh.volumes[ein], mesh.volumes[eout],
                           gid[ein], gid[eout])
    code = (tid[fi, 0] | (tid[fi, 1] << 5) | np.where(mi, CODE_MINUS_IN, 0)
            | np.where(owned(eout), 0, CODE_SKIP_OUT))
    geo = np.concatenate([jin, jout, sfac_all[fi, None], h[:, None],
                          1.0 / detJ[ein, None], 1.0 / detJ[eout, None]],
                         axis=1)
    el = np.stack([ein, eout], axis=1)
    lfs = np.stack([fl[fi, 0], fl[fi, 1]], axis=1)
    fids = fi.astype(np.int64)
    bmask = ~interior & owned(fe[:, 0])
    if dirichlet:
        bi = np.flatnonzero(bmask)
        be = fe[bi, 0]
        bj = np.einsum("fab,fb->fa", Jinv[be], nrm[bi])
        bgeo = np.concatenate([bj, np.zeros_like(bj), sfac_all[bi, None],
                               mesh.diameters[be, None], 1.0 / detJ[be, None],
                               np.zeros((len(bi), 1))], axis=1)
        bcode = (tid[bi, 0] | CODE_MINUS_IN | CODE_MIRROR
                 | (mesh.face_tags[bi].astype(np.int64) << 11))
        code = np.concatenate([code, bcode])
        geo = np.concatenate([geo, bgeo])
        el = np.concatenate([el, np.stack([be, np.full(len(bi), -1)], axis=1)])
        lfs = np.concatenate([lfs, np.stack([fl[bi, 0], np.full(len(bi), -1)],
                                            axis=1)])
        fids = np.concatenate([fids, bi.astype(np.int64)])
        nbf = np.zeros(0, dtype=np.int64)
    else:
        nbf = np.flatnonzero(bmask)
    # ---- colour segments ------------------------------------------------
    # part 1: the faces that read owned rows only (non-cut interior faces
    # and walls), coloured together; part 2 (slab runs): the faces whose
    # outside is a ghost row, coloured among themselves (one written side)
    cut = (code & CODE_SKIP_OUT) != 0
    n_cut = int(cut.sum())
    nif, nbw = len(code), len(nbf)
    w_out = np.where(cut | (el[:, 1] < 0), -1, el[:, 1])
    main = np.flatnonzero(~cut)
    m_in = np.concatenate([el[main, 0], fe[nbf, 0]])
    m_out = np.concatenate([w_out[main], np.full(nbw, -1)])
    m_lfi = np.concatenate([lfs[main, 0], fl[nbf, 0]])
    m_lfo = np.concatenate([np.where(w_out[main] >= 0, lfs[main, 1], -1), np.full(nbw, -1)])
    col_m, nc1 = color_faces(m_in, m_out, n_owned, _class_order(m_lfi, m_lfo, d))
    cidx = np.flatnonzero(cut)
    col_c, nc2 = color_faces(el[cidx, 0], np.full(len(cidx), -1), n_owned,
                             _class_order(lfs[cidx, 0], np.full(len(cidx), -1), d))
    seg_f = np.empty(nif, dtype=np.int64)
    seg_f[main] = col_m[:len(main)]
    seg_f[cidx] = nc1 + col_c
    seg_w = col_m[len(main):].astype(np.int64)
    n_seg = nc1 + nc2
    # element chunk of every face (the host-data stepping's copy chunks,
    # vol_chunk_bounds): the later chunk of its owned elements
    cbnd = np.asarray(vol_chunk_bounds(n_owned), dtype=np.int64)
    def echunk(e):
        return np.clip(np.searchsorted(cbnd, e, side="right") - 1, 0, VOL_CHUNKS - 1)
    e_out_own = np.where((el[:, 1] >= 0) & (el[:, 1] < n_owned), el[:, 1], el[:, 0])
    chunk_f = np.maximum(echunk(el[:, 0]), echunk(e_out_own))
    chunk_w = echunk(fe[nbf, 0])
    # interior faces by (segment, chunk, signature); walls by (segment,
    # chunk, table, tag): a segment's faces of one chunk are contiguous
    order = np.lexsort((code & 1023, chunk_f, seg_f))
    code, geo, el, lfs, seg_f = code[order], geo[order], el[order], lfs[order], seg_f[order]
    fids, chunk_f = fids[order], chunk_f[order]
    btag = mesh.face_tags[nbf].astype(np.int64)
    border = np.lexsort((btag, tid[nbf, 0], chunk_w, seg_w))
    nbf, btag, seg_w, chunk_w = nbf[border], btag[border], seg_w[border], chunk_w[border]
    bcode = tid[nbf, 0] | (btag << 11)
    seg_if = np.searchsorted(seg_f, np.arange(n_seg + 1), side="left")
    seg_bf = np.searchsorted(seg_w, np.arange(n_seg + 1), side="left")
    # first written side of every element in segment order: it writes the
    # element's face-sum row, later sides add to it
    wr_out = np.flatnonzero((el[:, 1] >= 0) & ((code & (CODE_SKIP_OUT | CODE_MIRROR)) == 0))
    e_all = np.concatenate([el[:, 0], el[wr_out, 1], fe[nbf, 0]])
    s_all = np.concatenate([seg_f, seg_f[wr_out], seg_w])
    first_seg = np.full(n_owned, np.iinfo(np.int64).max)
    np.minimum.at(first_seg, e_all, s_all)
    if n_owned and (first_seg == np.iinfo(np.int64).max).any():
        raise ValueError("an owned element has no face (non-conforming face lists)")
    fin = first_seg[el[:, 0]] == seg_f
    fout = np.zeros(nif, dtype=bool)
    fout[wr_out] = first_seg[el[wr_out, 1]] == seg_f[wr_out]
    code = code | np.where(fin, CODE_FIRST_IN, 0) | np.where(fout, CODE_FIRST_OUT, 0)
    bcode = bcode | np.where(first_seg[fe[nbf, 0]] == seg_w, CODE_FIRST_IN, 0)

    c64 = lambda a: np.ascontiguousarray(a, dtype=np.float64)
    i32 = lambda a: np.ascontiguousarray(a, dtype=np.int32)
    return OperatorTables(
        dim=d, order=k, n_species=S, nb=nb, nq_vol=len(vr), nq_face=len(fr),
        vol_phi=c64(phi), vol_grad=c64(grad), vol_w=c64(vr.weights),
        vol_stiff=c64(ks), face_B=c64(fB), face_G=c64(fG), face_Pw=c64(fPw),
        face_w=c64(fr.weights), elem_geo=c64(egeo[:n_owned]),
        if_elems=i32(el), if_code=i32(code), if_geo=c64(geo),
        bf_elem=i32(fe[nbf, 0]), bf_code=i32(bcode), bf_geo=c64(sfac_all[nbf]),
        n_cut=n_cut, n_seg=int(n_seg), n_seg_cut=int(nc2),
        seg_if=seg_if.astype(np.int64), seg_bf=seg_bf.astype(np.int64),
        if_seg=seg_f.astype(np.int32), if_lf=i32(lfs), bf_lf=i32(fl[nbf, 0]),
        if_fid=fids, bf_fid=nbf.astype(np.int64), face_pts=np.asarray(fr.points, dtype=float),
        if_chunk=chunk_f.astype(np.int32), bf_chunk=chunk_w.astype(np.int32))


def seg_chunk_offsets(seg: np.ndarray, chunk: np.ndarray, n_seg: int) -> np.ndarray:
    """Offsets of the (segment, chunk) runs of an array sorted by (segment,
    chunk): int64 [n_seg * VOL_CHUNKS + 1]; run (s, c) is [o[s C + c],
    o[s C + c + 1]).  The host-data stepping runs its first stage chunk by
    chunk as the state arrives (csrc/capi.cu tdg_ssprk3_steps_host)."""
    key = np.asarray(seg, dtype=np.int64) * VOL_CHUNKS + np.asarray(chunk, dtype=np.int64)
    return np.searchsorted(key, np.arange(n_seg * VOL_CHUNKS + 1), side="left").astype(np.int64)


def _ceil(x, m):
    return (x + m - 1) // m * m


def mma_face_tables(t: OperatorTables):
    """Zero-padded per-signature operand tables of the tensor-core face
    kernel (csrc/kernels_mma.cuh), concatenated per table id:

    TB   [FP][NBK]        B[q][k]               traces u = B c
    TGa  [d][FP][NBK]     G[q][k][a]            traces d_n u = sum_a jn_a (G_a c)
    TBW  [NBM][FP]        w_q B[q][i]           modal lifting m = (wB)^T dU
    TBT  [NBM][FP]        B[q][i]               projection of Y
    TGTa [d][NBM][FP]     G[q][i][a]            projection of X jn_a
    with FP = ceil8(F), NBK = ceil4(nb), NBM = ceil8(nb).  Returns the
    flat array and the per-table stride."""
    d, nb, F = t.dim, t.nb, t.nq_face
    FP, NBK, NBM = _ceil(F, 8), _ceil(nb, 4), _ceil(nb, 8)
    NT = t.face_B.shape[0]
    parts = []
    for k in range(NT):
        B, G = t.face_B[k], t.face_G[k]                    # (F, nb), (F, nb, d)
        TB = np.zeros((FP, NBK)); TB[:F, :nb] = B
        TG = np.zeros((d, FP, NBK)); TG[:, :F, :nb] = G.transpose(2, 0, 1)
        TBW = np.zeros((NBM, FP)); TBW[:nb, :F] = (t.face_w[:, None] * B).T
        TBT = np.zeros((NBM, FP)); TBT[:nb, :F] = B.T
        TGT = np.zeros((d, NBM, FP)); TGT[:, :nb, :F] = G.transpose(2, 1, 0)
        parts.append(np.concatenate([x.ravel() for x in (TB, TG, TBW, TBT, TGT)]))
    stride = len(parts[0])
    return np.ascontiguousarray(np.concatenate(parts)), stride


def _pi_cols(nb: int):
    """Output-column permutation of the transposed tensor-core kernels:
    pi(8 nt + 2 t + j) = 4 (2 nt + j) + t; returns (pi clipped, valid)."""
    NBN = _ceil(nb, 8)
    n = np.arange(NBN)
    pi = 4 * (2 * (n // 8) + (n % 8) % 2) + (n % 8) // 2
    ok = pi < nb
    return np.where(ok, pi, 0), ok


_LANE = np.arange(32)
_LG, _LT = _LANE >> 2, _LANE & 3       # m8n8k4 fragment coordinates g, t


def _frag_kq(A):
    """[4 KT][8 QT] table (B operand rows k = 4 kt + t, columns q = 8 qt + g)
    -> fragment-major [KT][QT][32 lanes]."""
    KT, QT = A.shape[0] // 4, A.shape[1] // 8
    kt, qt = np.meshgrid(np.arange(KT), np.arange(QT), indexing="ij")
    return A[4 * kt[..., None] + _LT, 8 * qt[..., None] + _LG]


def _frag_qn(A):
    """[8 QT][8 NNT] table (B operand rows q = 8 qt + 2 t + ks, columns
    n = 8 nt + g) -> fragment-major [QT][2][NNT][32 lanes]."""
    QT, NNT = A.shape[0] // 8, A.shape[1] // 8
    qt, ks, nt = np.meshgrid(np.arange(QT), np.arange(2), np.arange(NNT), indexing="ij")
    return A[8 * qt[..., None] + 2 * _LT + ks[..., None], 8 * nt[..., None] + _LG]


def _frag_kn(A):
    """[4 KT][8 NNT] table (B operand rows k = 4 kt + t, columns n = 8 nt + g)
    -> fragment-major [KT][NNT][32 lanes]."""
    KT, NNT = A.shape[0] // 4, A.shape[1] // 8
    kt, nt = np.meshgrid(np.arange(KT), np.arange(NNT), indexing="ij")
    return A[4 * kt[..., None] + _LT, 8 * nt[..., None] + _LG]


def tc_face_tables(t: OperatorTables):
    """Per-signature operand tables of the 3D species-rows tensor-core face
    kernel (csrc/kernels_tcf.cuh), concatenated per table id, stored
    fragment-major (``_frag_kq`` / ``_frag_qn``: one warp-wide B-operand
    load is 32 consecutive fragments):

    TR  [KT][QT][32][4]        (B[q][k], G[q][k][0..2]) B^T / G_a^T fragments:
                               traces u = c B^T and d_n u = c (sum_a jn_a G_a)^T,
                               one 32-byte load per lane
    PR  [QT][2][NNT][32][4]    (B[q][pi(n)], G[q][pi(n)][0..2]): projection of
                               Y (B) and of X (sum_a jn_a G_a)
    WB  [QT][2][NNT][32]       w_q B[q][pi(n)]  modal lifting m = dU (w B)
    BT  [KT][QT][32]           B[q][k]          rho = m B^T
    with QP = ceil8(F), NBK = ceil4(nb), NBN = ceil8(nb).  Returns the flat
    array and the per-signature stride."""
    d, nb, F = t.dim, t.nb, t.nq_face
    if d != 3:
        raise ValueError("the species-rows face kernel is 3D only")
    QP, NBK, NBN = _ceil(F, 8), _ceil(nb, 4), _ceil(nb, 8)
    pic, ok = _pi_cols(nb)
    parts = []
    for k in range(t.face_B.shape[0]):
        B, G = t.face_B[k], t.face_G[k]                    # (F, nb), (F, nb, d)
        BT = np.zeros((NBK, QP)); BT[:nb, :F] = B.T
        GT = np.zeros((d, NBK, QP)); GT[:, :nb, :F] = G.transpose(2, 1, 0)
        BP = np.zeros((QP, NBN)); BP[:F] = B[:, pic] * ok
        GP = np.zeros((d, QP, NBN)); GP[:, :F] = G.transpose(2, 0, 1)[:, :, pic] * ok
        WB = np.zeros((QP, NBN)); WB[:F] = (t.face_w[:, None] * B)[:, pic] * ok
        TR = np.stack([_frag_kq(BT)] + [_frag_kq(GT[a]) for a in range(d)], axis=-1)
        PR = np.stack([_frag_qn(BP)] + [_frag_qn(GP[a]) for a in range(d)], axis=-1)
        parts.append(np.concatenate([TR.ravel(), PR.ravel(), _frag_qn(WB).ravel(),
                                     _frag_kq(BT).ravel()]))
    stride = len(parts[0])
    return np.ascontiguousarray(np.concatenate(parts)), stride


def _row_classes(rows: np.ndarray):
    """Classes of identical rows of an int64 matrix: (unique rows in order
    of first appearance, class of every row).  Hash-factorised (O(n), the
    C5 meshes have 1e8 rows) and verified row by row; falls back to the
    sorting np.unique on a hash collision."""
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    h = np.zeros(len(rows), dtype=np.uint64)
    with np.errstate(over="ignore"):
        for j in range(rows.shape[1]):
            c = rows[:, j].view(np.uint64)
            h = (h ^ c) * np.uint64(0x9E3779B97F4A7C15) + np.uint64(0x632BE59BD9B4E019 + j)
            h ^= h >> np.uint64(29)
    try:
        import pandas as pd
        inv, first = pd.factorize(h.view(np.int64), sort=False)
        inv = inv.astype(np.int64)
        idx = np.empty(len(first), dtype=np.int64)
        idx[inv[::-1]] = np.arange(len(rows) - 1, -1, -1)   # first row of each class
        uniq = rows[idx]
        if np.array_equal(rows, uniq[inv]):
            return uniq, inv
    except ImportError:
        pass
    uniq, inv = np.unique(rows, axis=0, return_inverse=True)
    return uniq, inv.reshape(-1)


def face_classes(t: OperatorTables, max_classes: int = 512):
    """Face-geometry classes: every interior face side is a (trace-table id,
    Jinv n) pair; meshes of congruent cells have few of them (Kuhn cubes: 6
    per side; the structured triangles likewise).  Returns (int32 [nif][2]
    class of the inside / outside side, [(table id, Jinv n)] per class) or
    None (no interior faces, Dirichlet mirror faces, or more than
    ``max_classes`` classes)."""
    d = t.dim
    nif = len(t.if_code)
    if nif == 0 or (t.if_code & CODE_MIRROR).any():
        return None
    code = t.if_code.astype(np.int64)
    tid = np.concatenate([code & 31, (code >> 5) & 31])
    jn = np.ascontiguousarray(np.concatenate([t.if_geo[:, 0:d], t.if_geo[:, d:2 * d]]))
    key = np.concatenate([tid[:, None], jn.view(np.int64)], axis=1)
    uniq, inv = _row_classes(key)
    if len(uniq) > max_classes:
        return None
    cls = np.ascontiguousarray(np.stack([inv[:nif], inv[nif:]], axis=1), dtype=np.int32)
    keys = [(int(row[0]), row[1:].copy().view(np.float64)) for row in uniq]
    return cls, keys


def tc_face_fold_tables(t: OperatorTables, max_classes: int = 512):
    """Face-geometry classes of the species-rows face kernel: every
    interior face side is a (table id, Jinv n) pair; meshes of congruent
    cells (the Kuhn cubes: 6 classes per side) have few of them, and per
    class the normal-derivative fragments sum_a (Jinv n)_a G_a can be
    formed once instead of per face (they are a linear combination of the
    signature's gradient tables, operator.py:375,386).  Per class:

    TRF [KT][QT][32][2]        (B[q][k], G_n[q][k])        traces
    PRF [QT][2][NNT][32][2]    (B[q][pi(n)], G_n[q][pi(n)]) projection
    PBF [QT][2][NNT][32]       B[q][pi(n)]                  projection, by kind
    PGF [QT][2][NNT][32]       G_n[q][pi(n)]                (face-group kernel)

    Returns (flat tables, per-class stride, int32 [nif][2] class of the
    inside / outside side, [(table id, Jinv n)] per class) or None when the
    mesh has more than ``max_classes`` classes (the kernel then folds per
    face)."""
    d, nb, F = t.dim, t.nb, t.nq_face
    if d != 3:
        return None
    fc = face_classes(t, max_classes)
    if fc is None:
        return None
    cls, keys = fc
    QP, NBK, NBN = _ceil(F, 8), _ceil(nb, 4), _ceil(nb, 8)
    pic, ok = _pi_cols(nb)
    parts = []
    for k, jv in keys:
        B, G = t.face_B[k], t.face_G[k]                     # (F, nb), (F, nb, d)
        Gn = np.einsum("qia,a->qi", G, jv)
        BT = np.zeros((NBK, QP)); BT[:nb, :F] = B.T
        GT = np.zeros((NBK, QP)); GT[:nb, :F] = Gn.T
        BP = np.zeros((QP, NBN)); BP[:F] = B[:, pic] * ok
        GP = np.zeros((QP, NBN)); GP[:F] = Gn[:, pic] * ok
        TRF = np.stack([_frag_kq(BT), _frag_kq(GT)], axis=-1)
        PRF = np.stack([_frag_qn(BP), _frag_qn(GP)], axis=-1)
        parts.append(np.concatenate([TRF.ravel(), PRF.ravel(), _frag_qn(BP).ravel(),
                                     _frag_qn(GP).ravel()]))
    return np.ascontiguousarray(np.concatenate(parts)), len(parts[0]), cls, keys


def tc_face_blocks(t: OperatorTables, block: int = 8):
    """Blocks of up to ``block`` consecutive interior faces with one trace-
    table signature each (the 3D species-rows face kernel runs a block per
    warp), never straddling a colour segment.  Returns (int32 [nblk][2] =
    (first face, count), block offsets of the segments [n_seg+1])."""
    nif = len(t.if_code)
    if nif == 0:
        return np.zeros((0, 2), np.int32), np.zeros(t.n_seg + 1, np.int64)
    sig = ((t.if_code.astype(np.int64) & 1023)
           + (t.if_seg.astype(np.int64) * VOL_CHUNKS + t.if_chunk) * 1024)
    brk = np.flatnonzero(np.diff(sig)) + 1
    starts = np.concatenate([[0], brk])
    lens = np.diff(np.concatenate([starts, [nif]]))
    nblk = (lens + block - 1) // block
    rs = np.repeat(starts, nblk)
    j = np.arange(nblk.sum()) - np.repeat(np.cumsum(nblk) - nblk, nblk)
    first = rs + block * j
    cnt = np.minimum(block, np.repeat(starts + lens, nblk) - first)
    blocks = np.ascontiguousarray(np.stack([first, cnt], axis=1), dtype=np.int32)
    seg_blk = np.searchsorted(first, t.seg_if, side="left").astype(np.int64)
    return blocks, seg_blk


def _o_basis(A: np.ndarray, rank: int) -> np.ndarray:
    """Orthonormal basis of the column space of A (F x m), which must have
    numerical rank ``rank`` (the face rules have negative weights, so the
    basis is orthonormal in the plain inner product and W enters through
    small Gram matrices)."""
    U, s, _ = np.linalg.svd(A, full_matrices=False)
    if len(s) > rank and s[rank] > 1e-11 * s[0]:
        raise ValueError(f"trace space rank above {rank}: singular values {s[:rank + 2]}")
    if s[rank - 1] < 1e-8 * s[0]:
        raise ValueError(f"trace space rank below {rank}")
    return U[:, :rank]


def modal_face_factors(t: OperatorTables, fold):
    """Low-rank factors of the 3D face operator (the face-group kernel's
    modal formulation).  On a face the traces of the degree-k volume basis
    span P_k of the face triangle, (k+1)(k+2)/2 functions, and the traces of
    a directional derivative (Jinv n fixed per face-geometry class) span
    P_{k-1}, k(k+1)/2 functions: with orthonormal bases Bf (F x nfm) and
    Bd (F x ndm) of those spaces at the face points,

        face_B[tab]  = Bf T[tab],     T[tab]  = Bf^T face_B[tab]
        G_n[class]   = Bd Td[class],  Td[class] = Bd^T G_n[class]

    exactly (to roundoff).  With W = diag(face weights), Mff = Bf^T W Bf and
    Mfd = Bf^T W Bd, the face terms of reference operator.py:326-424 reduce
    to modal algebra except the pointwise LLF flux (a_j = T_in c_in -
    T_out c_out, g = (Td_in c_in + Td_out c_out) / 2):

        B^T W rho,  rho = B (B^T W dU)   ->  T^T (Mff T_l T_l^T Mff) a_j
        B^T W (A gav)                    ->  A T^T Mfd g
        G_n^T W X,  X ~ dU               ->  Td^T Mfd^T a_j
        B^T W (eta/h A dU)  (ip)         ->  eta/h A T^T Mff a_j

    ``fold``: ``face_classes``' (cls, keys) or ``tc_face_fold_tables``'
    result (the class keys are its last entry).
    Returns dict(Bf, Bd, T [ntab][nfm][nb], Td [ncls][ndm][nb],
    L [ntab][nfm][nfm] = Mff T T^T Mff, Mff, Mfd, nfm, ndm)."""
    d, k, nb = t.dim, t.order, t.nb
    # P_k / P_{k-1} on the face: a triangle (3D) or a segment (2D)
    nfm, ndm = ((k + 1) * (k + 2) // 2, k * (k + 1) // 2) if d == 3 else (k + 1, k)
    w = t.face_w
    B = t.face_B                                     # (ntab, F, nb)
    Bf = _o_basis(np.concatenate(list(B), axis=1), nfm)
    # T = Bf^+ B in extended precision, kept as a double-double pair (T,
    # Tlo): the jump T_in c_in - T_out c_out of a continuous field cancels
    # to roundoff only if both tables carry B to well below one ulp (the
    # fp64-rounded T alone leaves ~1e-14 |c| in the jump, which the 1/h
    # penalties amplify)
    Bl = Bf.astype(np.longdouble)
    G = np.linalg.inv((Bf.T @ Bf).astype(np.float64)).astype(np.longdouble)
    eye = np.eye(nfm, dtype=np.longdouble)
    for _ in range(3):
        G = G + G @ (eye - (Bl.T @ Bl) @ G)
    Tx = np.stack([G @ (Bl.T @ B[k].astype(np.longdouble)) for k in range(len(B))])
    T = Tx.astype(np.float64)
    Tlo = (Tx - T.astype(np.longdouble)).astype(np.float64)
    cls_keys = fold[-1]
    Gn = np.stack([np.einsum("qia,a->qi", t.face_G[int(tab)], jv) for tab, jv in cls_keys])
    if ndm > 0:
        Bd = _o_basis(np.concatenate(list(Gn), axis=1), ndm)
        Td = np.einsum("qm,cqi->cmi", Bd, Gn)
    else:
        Bd = np.zeros((len(w), 0))
        Td = np.zeros((len(Gn), 0, nb))
    Mff = np.einsum("qm,q,qn->mn", Bf, w, Bf)
    Mfd = np.einsum("qm,q,qn->mn", Bf, w, Bd)
    L = np.einsum("mk,tki,tli,ln->tmn", Mff, T, T, Mff)
    return {"Bf": Bf, "Bd": Bd, "T": T, "Tlo": Tlo, "Td": Td, "L": L, "Mff": Mff, "Mfd": Mfd,
            "nfm": nfm, "ndm": ndm}


def _pi_mat(M: np.ndarray, rows: int, ncols: int):
    """[rows][8 ceil(ncols/8)] with column n holding M[:, pi(n)] (zero past
    ncols) -- the output-column permutation of the DMMA kernels."""
    pic, ok = _pi_cols(ncols)
    out = np.zeros((rows, len(pic)))
    out[:M.shape[0]] = M[:, pic] * ok
    return out


def modal_face_tables(t: OperatorTables, fold):
    """Operand tables of the modal face-group kernel (csrc/kernels_tcm.cuh)
    from ``modal_face_factors``.  The kernel keeps one modal vector per row,
    v = (face modes a | d-modes d), nv = nfm + ndm entries (16 at p = 3), in
    the DMMA accumulator layout with pi-permuted columns; a GEMM over the a
    (d) part uses the k-steps that hold them and zero table rows for the
    other part.  Fragment-major, concatenated as

      global     BF  [KA][QT][32]           Bf^T         point values of the a part
                 BD  [KTV-KD0][QT][32]      Bd^T         of the d part
                 WB  [QT][2][NAT][32]       w Bf (pi)    projection of the pointwise flux
                 MFD [KTV-KD0][NAT][32]     Mfd (pi)     A gav term   (d -> a)
                 MDF [KA][NNV-NAT0][32]     Mfd^T (pi)   adjoint term (a -> d)
                 MFF [KA][NAT][32]          Mff (pi)     ip penalty   (a -> a)
      per table  L   [KA][NAT][32]          L (pi)       lifting (Mff T T^T Mff)
      per class  TD1 [KT][NNV][32]          (T | Td)^T   v of the coefficients
                 TD4 [KTV][NNT][32]         (T ; Td)     back to the volume modes (inside)
                 TD4M[KTV][NNT][32]         (-T ; Td)    (outside: the flux changes sign)

    KA = ceil(nfm/4) k-steps hold the a part, k-steps KD0 = floor(nfm/4) ..
    KTV = ceil(nv/4) the d part; NNV = ceil(nv/8) output tiles, the a part in
    tiles [0, NAT = ceil(nfm/8)), the d part in [NAT0 = floor(nfm/8), NNV).
    Returns the flat array."""
    mf = modal_face_factors(t, fold)
    nb, F = t.nb, t.nq_face
    nfm, ndm = mf["nfm"], mf["ndm"]
    nv = nfm + ndm
    KT, KA, KTV, KD0 = -(-nb // 4), -(-nfm // 4), -(-nv // 4), nfm // 4
    NNV, NAT, NAT0 = -(-nv // 8), -(-nfm // 8), nfm // 8
    QP = _ceil(F, 8)
    pv, okv = _pi_cols(nv)                 # combined output columns
    pv = np.where(okv, pv, nv)             # out of range -> the zero column
    w = np.zeros(QP); w[:F] = t.face_w
    Bf = np.zeros((QP, nv + 1)); Bf[:F, :nfm] = mf["Bf"]       # columns: combined modes
    Bd = np.zeros((QP, nv + 1)); Bd[:F, nfm:nv] = mf["Bd"][:, :ndm]
    Mfd = mf["Mfd"][:, :ndm]
    # square operators on the combined index, zero-padded by one
    def comb(rows_a, rows_d, Xaa=None, Xad=None, Xda=None):
        M = np.zeros((nv + 1, nv + 1))
        if Xaa is not None: M[:nfm, :nfm] = Xaa
        if Xad is not None: M[:nfm, nfm:nv] = Xad
        if Xda is not None: M[nfm:nv, :nfm] = Xda
        return M
    def kn(M, k0, k1, n0, n1):
        """B operand [k][n]: rows = combined k in [4 k0, 4 k1), columns
        tiles [n0, n1) of the pi-permuted combined outputs, M[k][out]."""
        rows = np.arange(4 * k0, 4 * k1)
        rows = np.where(rows < nv, rows, nv)
        cols = pv[8 * n0:8 * n1]
        return _frag_kn(M[np.ix_(rows, cols)])
    BFr = Bf[:, np.where(np.arange(4 * KA) < nfm, np.arange(4 * KA), nv)]
    BDr = Bd[:, np.where(np.arange(4 * KD0, 4 * KTV) < nv, np.arange(4 * KD0, 4 * KTV), nv)]
    WB = (w[:, None] * Bf)[:, pv[:8 * NAT]]
    parts = [_frag_kq(BFr.T), _frag_kq(BDr.T), _frag_qn(WB),
             kn(comb(0, 0, Xda=Mfd.T), KD0, KTV, 0, NAT),        # out_a += Mfd d
             kn(comb(0, 0, Xad=Mfd), 0, KA, NAT0, NNV),           # out_d += Mfd^T a
             kn(comb(0, 0, Xaa=mf["Mff"]), 0, KA, 0, NAT)]        # out_a += Mff a
    for k in range(t.face_B.shape[0]):
        parts.append(kn(comb(0, 0, Xaa=mf["L"][k].T), 0, KA, 0, NAT))
    # the class's table id comes from the class key (tc_face_fold_tables)
    for c, (tab, _jv) in enumerate(fold[-1]):
        T, Td = mf["T"][tab], mf["Td"][c][:ndm]
        V = np.zeros((nb, nv + 1)); V[:, :nfm] = T.T; V[:, nfm:nv] = Td.T   # (T | Td)^T
        TD1 = V[np.where(np.arange(4 * KT) < nb, np.arange(4 * KT), nb - 1)][:, pv[:8 * NNV]]
        TD1[np.arange(4 * KT) >= nb] = 0.0
        pic, ok = _pi_cols(nb)
        R = np.zeros((4 * KTV, len(pic)))
        R[:nfm] = T[:, pic] * ok
        R[nfm:nv] = Td[:, pic] * ok
        RM = R.copy(); RM[:nfm] *= -1.0
        parts += [_frag_kn(TD1), _frag_kn(R), _frag_kn(RM)]
    return np.ascontiguousarray(np.concatenate([p.ravel() for p in parts]))


def tc_face_groups(t: OperatorTables, cls: np.ndarray, n_species: int):
    """Face groups of the face-group tensor-core kernel (csrc/kernels_tcg.cuh):
    runs of NFQ = 8 / gcd(S, 8) interior faces of one colour segment that
    share the inside and outside face-geometry class (``cls`` from
    ``tc_face_fold_tables``) and the lifting side (K- flag), so the S NFQ
    (face, species) rows fill whole DMMA M tiles and share every B operand.
    The faces keep their segment, so the face-sum order (and every bit of
    the result) is that of the per-face kernels.  Returns (int32
    [ngroups][NFQ] face ids, -1 past a run's end; int64 group offsets of the
    segments [n_seg+1])."""
    nfq = 8 // int(np.gcd(int(n_species), 8))
    nif = len(t.if_code)
    if nif == 0:
        return np.zeros((0, nfq), np.int32), np.zeros(t.n_seg + 1, np.int64)
    minus = (t.if_code.astype(np.int64) >> 10) & 1
    ncls = int(cls.max()) + 1
    sc = t.if_seg.astype(np.int64) * VOL_CHUNKS + t.if_chunk
    key = ((sc * ncls + cls[:, 0]) * ncls + cls[:, 1]) * 2 + minus
    order = np.argsort(key, kind="stable")
    ks = key[order]
    brk = np.flatnonzero(np.diff(ks)) + 1
    starts = np.concatenate([[0], brk])
    lens = np.diff(np.concatenate([starts, [nif]]))
    ng = (lens + nfq - 1) // nfq
    # slot j of group i of run r holds order[start_r + nfq i + j] inside the run
    run_of = np.repeat(np.arange(len(starts)), ng)
    gi = np.arange(ng.sum()) - np.repeat(np.cumsum(ng) - ng, ng)
    pos = starts[run_of][:, None] + nfq * gi[:, None] + np.arange(nfq)[None, :]
    inside = pos < (starts + lens)[run_of][:, None]
    groups = np.where(inside, order[np.minimum(pos, nif - 1)], -1).astype(np.int32)
    gseg = t.if_seg[order[starts[run_of]]].astype(np.int64)
    seg_g = np.searchsorted(gseg, np.arange(t.n_seg + 1), side="left").astype(np.int64)
    return np.ascontiguousarray(groups), seg_g


VOL_CHUNKS = 8   # element chunks of the host-data entry points (tdg_ctx::kChunks)


def vol_chunk_bounds(ne: int):
    """Element chunk boundaries of the host-data entry points (ctx.cuh
    chunk_start): ne k / 8 rounded down to a multiple of 8 elements."""
    return [ne if k >= VOL_CHUNKS else (ne * k // VOL_CHUNKS) // 8 * 8
            for k in range(VOL_CHUNKS + 1)]


def tc_volume_classes(t: OperatorTables, max_classes: int = 16):
    """Element-geometry classes of the tensor-core volume kernel: meshes of
    congruent cells (the Kuhn cubes: 6 tetrahedron shapes) have few distinct
    geometry records (detJ, sym(Jinv Jinv^T)), and per class the exact
    stiffness sum_p M_p KS_p is one matrix, so a warp of 8 same-class
    elements runs its diffusion as one GEMM per species instead of
    d(d+1)/2 metric-scaled ones (reference operator.py:292-324 diffusion
    term).  Elements keep their rows; the kernel visits them through a
    permutation, sorted by class inside each of the VOL_CHUNKS element
    chunks (``vol_chunk_bounds``) so chunked launches stay exact.

    Returns (class tables [ncls][KT][NNT][32] fragment-major as
    ``_frag_kn``, int32 element ids [ntask][8] (-1 pads a class's last
    task), int32 class of every task [ntask], int64 task offsets of the
    chunks [VOL_CHUNKS + 1]) or None with more than ``max_classes``."""
    ne = t.elem_geo.shape[0]
    if ne == 0:
        return None
    uniq, cls = _row_classes(np.ascontiguousarray(t.elem_geo).view(np.int64))
    if len(uniq) > max_classes:
        return None
    nb = t.nb
    NBK, NBN = _ceil(nb, 4), _ceil(nb, 8)
    pic, ok = _pi_cols(nb)
    geo = uniq.view(np.float64)
    tabs = []
    for g in geo:
        Kc = np.einsum("p,pij->ij", g[1:], t.vol_stiff)
        KP = np.zeros((NBK, NBN)); KP[:nb] = Kc[:, pic] * ok
        tabs.append(_frag_kn(KP).ravel())
    perm, tcls, toff = [], [], [0]
    cb = vol_chunk_bounds(ne)
    for k in range(VOL_CHUNKS):
        e0, e1 = cb[k], cb[k + 1]
        c = cls[e0:e1]
        order = np.argsort(c, kind="stable") + e0
        cs = cls[order]
        brk = np.flatnonzero(np.diff(cs)) + 1
        starts = np.concatenate([[0], brk]) if len(cs) else np.zeros(0, np.int64)
        lens = np.diff(np.concatenate([starts, [len(cs)]]))
        ntask = 0
        for s0, ln in zip(starts, lens):
            nt = (ln + 7) // 8
            ids = np.full(nt * 8, -1, np.int64)
            ids[:ln] = order[s0:s0 + ln]
            perm.append(ids)
            tcls.append(np.full(nt, cs[s0], np.int64))
            ntask += nt
        toff.append(toff[-1] + ntask)
    perm = np.concatenate(perm).astype(np.int32)
    tcls = np.concatenate(tcls).astype(np.int32)
    return (np.ascontiguousarray(np.concatenate(tabs)), perm.reshape(-1, 8), tcls,
            np.asarray(toff, dtype=np.int64))


def tc_volume_tables(t: OperatorTables) -> np.ndarray:
    """Operand tables of the transposed tensor-core volume kernel
    (csrc/kernels_tc.cuh, k_volume_tc), concatenated, each stored
    fragment-major (one warp-wide B-operand load = 32 consecutive doubles):

    PHT [NBK][QP]        Phi[q][k]                    B of the point values
    GT  [d][NBK][QP]     G[q][k][a]                   B of the reference gradients
    PP  [QP][NBN]        w_q Phi[q][pi(n)]            projection of the bilinear source
    PG  [d][QP][NBN]     w_q G[q][pi(n)][a]           projection of the flux rows
    KS  [nsym][NBK][NBN] KS_p[k][pi(n)]               diffusion stiffness blocks
    with QP = ceil8(Q), NBK = ceil4(nb), NBN = ceil8(nb) and the output
    column permutation pi(8 nt + 2 t + j) = 4 (2 nt + j) + t (entries with
    pi(n) >= nb are zero)."""
    d, nb = t.dim, t.nb
    Q = t.vol_phi.shape[0]
    QP, NBK, NBN = _ceil(Q, 8), _ceil(nb, 4), _ceil(nb, 8)
    nsym = d * (d + 1) // 2
    pic, ok = _pi_cols(nb)
    w = t.vol_w
    PHT = np.zeros((NBK, QP)); PHT[:nb, :Q] = t.vol_phi.T
    GT = np.zeros((d, NBK, QP)); GT[:, :nb, :Q] = t.vol_grad.transpose(2, 1, 0)
    PP = np.zeros((QP, NBN)); PP[:Q] = (w[:, None] * t.vol_phi)[:, pic] * ok
    PG = np.zeros((d, QP, NBN))
    PG[:, :Q] = (w[:, None, None] * t.vol_grad).transpose(2, 0, 1)[:, :, pic] * ok
    KS = np.zeros((nsym, NBK, NBN)); KS[:, :nb] = t.vol_stiff[:, :, pic] * ok
    parts = ([_frag_kq(PHT)] + [_frag_kq(GT[a]) for a in range(d)] + [_frag_qn(PP)]
             + [_frag_qn(PG[a]) for a in range(d)] + [_frag_kn(KS[q]) for q in range(nsym)])
    return np.ascontiguousarray(np.concatenate([x.ravel() for x in parts]))


def scheme_constants(space: DGSpace, scheme: FluxScheme):
    d, k = space.mesh.dim, space.order
    return (chi_factor(d), scheme.adjoint_sign,
            scheme.ip_eta0 * max(k, 1) ** 2)
