"""Face colouring / segment order of the accumulating face kernels (host
side, no GPU): every colour segment writes each element at most once, each
element's first written face side carries the write flag, structured
meshes get d+1 colours, and slab meshes keep their cut faces in the last
segments.  (The reference keeps its sums race-free with private
per-partition buffers merged in part order, operator.py:262-284.)"""
import numpy as np
import pytest

from paper_1403_1157_b200 import DGSpace, FluxScheme, PlaqueModel, DiffusionModel
from paper_1403_1157_b200.mesh import unit_cube, unit_square
from paper_1403_1157_b200.tables import (CODE_FIRST_IN, CODE_FIRST_OUT, CODE_MIRROR,
                                         CODE_SKIP_OUT, build_tables, color_faces,
                                         tc_face_blocks, tc_face_fold_tables,
                                         tc_face_groups)


def _check(t, n_owned):
    el, code = t.if_elems, t.if_code
    wr = (el[:, 1] >= 0) & ((code & (CODE_SKIP_OUT | CODE_MIRROR)) == 0)
    seg_w = np.repeat(np.arange(t.n_seg), np.diff(t.seg_bf))
    e = np.concatenate([el[:, 0], el[wr, 1], t.bf_elem]).astype(np.int64)
    s = np.concatenate([t.if_seg, t.if_seg[wr], seg_w]).astype(np.int64)
    first = np.concatenate([(code & CODE_FIRST_IN) != 0, (code[wr] & CODE_FIRST_OUT) != 0,
                            (t.bf_code & CODE_FIRST_IN) != 0])
    # race freedom: (element, segment) pairs are unique
    pair = e * t.n_seg + s
    assert len(np.unique(pair)) == len(pair)
    # exactly one first side per owned element, in its lowest segment
    assert np.array_equal(np.bincount(e[first], minlength=n_owned), np.ones(n_owned))
    lo = np.full(n_owned, 1 << 40)
    np.minimum.at(lo, e, s)
    assert np.array_equal(lo[e[first]], s[first])
    # segment offsets are consistent with the per-face segment ids
    assert np.array_equal(np.searchsorted(t.if_seg, np.arange(t.n_seg + 1)), t.seg_if)
    # every element has d+1 face sides
    assert np.array_equal(np.bincount(e, minlength=n_owned), np.full(n_owned, t.dim + 1))


@pytest.mark.parametrize("mesh,ncol", [
    (lambda: unit_square(7, 5), 3),
    (lambda: unit_square(6, 4, lengths=(4.0, 1.0), jitter=0.1, seed=3), 3),
    (lambda: unit_cube(3), 4),
    (lambda: unit_cube(4, 2, 3), 4),
])
def test_structured_meshes_get_d_plus_1_colours(mesh, ncol):
    m = mesh()
    space = DGSpace(m, 1, 6)
    t = build_tables(space, PlaqueModel(), FluxScheme("cdg2"))
    assert t.n_seg == ncol and t.n_seg_cut == 0
    _check(t, m.n_elements)


def test_dirichlet_mirror_faces_are_coloured():
    m = unit_square(4)
    t = build_tables(DGSpace(m, 2, 1), DiffusionModel(0.5, dirichlet=0.3), FluxScheme("ip"))
    assert len(t.bf_code) == 0 and (t.if_code & CODE_MIRROR).any()
    _check(t, m.n_elements)


def test_greedy_colouring_is_proper_on_an_irregular_graph():
    rng = np.random.default_rng(0)
    n_el, n_f = 200, 500
    a = rng.integers(0, n_el, n_f)
    b = rng.integers(-1, n_el, n_f)
    b[b == a] = -1
    col, nc = color_faces(a, b, n_el)
    assert col.min() >= 0 and col.max() == nc - 1
    for c in range(nc):
        m = col == c
        ids = np.concatenate([a[m], b[m][b[m] >= 0]])
        assert len(np.unique(ids)) == len(ids)


def test_slab_cut_faces_run_last():
    from paper_1403_1157_b200.configs import CONFIGS
    from paper_1403_1157_b200.decomp import build_slab
    import dataclasses
    cfg = dataclasses.replace(CONFIGS["c4"], cells=(6, 3, 3))
    slab = build_slab(cfg, 1, 3)
    space = DGSpace(slab.mesh, 2, 6)
    t = build_tables(space, PlaqueModel(), FluxScheme("cdg2"), n_owned=slab.n_owned,
                     global_ids=slab.global_ids)
    assert t.n_cut > 0 and t.n_seg_cut >= 1
    ncut_start = t.seg_if[t.n_seg - t.n_seg_cut]
    assert ncut_start == len(t.if_code) - t.n_cut
    assert ((t.if_code[ncut_start:] & CODE_SKIP_OUT) != 0).all()
    assert t.seg_bf[t.n_seg - t.n_seg_cut] == len(t.bf_code)  # no walls in cut segments
    _check(t, slab.n_owned)
    blocks, seg_blk = tc_face_blocks(t)
    # blocks never straddle a segment
    for s in range(t.n_seg):
        for f0, n in blocks[seg_blk[s]:seg_blk[s + 1]]:
            assert t.seg_if[s] <= f0 and f0 + n <= t.seg_if[s + 1]


@pytest.mark.parametrize("cells,order,scheme,S", [
    ((3, 3, 3), 3, "cdg2", 6), ((4, 2, 3), 2, "br2", 6), ((4, 3, 2), 1, "ip", 6),
    ((3, 2, 2), 2, "cdg2", 3)])
def test_face_groups_cover_each_face_once_within_one_class(cells, order, scheme, S):
    """tables.tc_face_groups (face-group tensor-core kernel): every interior
    face sits in exactly one group slot; a group's faces share the colour
    segment, both sides' face-geometry class and the K- flag; groups hold
    8 / gcd(S, 8) slots, only a run's last group has empty (-1) slots, and
    the segment offsets bracket each segment's groups."""
    from paper_1403_1157_b200 import ReducedModel
    model = PlaqueModel() if S == 6 else ReducedModel()
    t = build_tables(DGSpace(unit_cube(*cells), order, S), model, FluxScheme(scheme))
    fold = tc_face_fold_tables(t)
    assert fold is not None
    cls = fold[2]
    groups, seg_g = tc_face_groups(t, cls, S)
    nfq = 8 // int(np.gcd(S, 8))
    assert groups.shape[1] == nfq
    ids = groups[groups >= 0]
    assert np.array_equal(np.sort(ids), np.arange(len(t.if_code)))
    assert (groups[:, 0] >= 0).all()
    # -1 slots only at the end of a group
    valid = groups >= 0
    assert (np.diff(valid.astype(int), axis=1) <= 0).all()
    f0 = groups[:, :1]
    g = np.where(valid, groups, f0)
    minus = (t.if_code >> 10) & 1
    for arr in (t.if_seg, cls[:, 0], cls[:, 1], minus):
        assert (arr[g] == arr[f0]).all()
    assert seg_g[0] == 0 and seg_g[-1] == len(groups)
    for s in range(t.n_seg):
        assert (t.if_seg[groups[seg_g[s]:seg_g[s + 1], 0]] == s).all()
    # a run (same segment, element chunk, classes, K- side) has at most one
    # partial group, and a group never straddles a chunk
    assert (t.if_chunk[g] == t.if_chunk[f0]).all()
    partial = ~valid.all(axis=1)
    f = f0[:, 0]
    key = (((t.if_seg[f] * 8 + t.if_chunk[f]) * 10**3 + cls[f, 0]) * 10**3 + cls[f, 1]) * 2 + minus[f]
    assert len(np.unique(key[partial])) == partial.sum()


@pytest.mark.parametrize("cells,order", [((4, 2, 2), 3), ((4, 4, 4), 2), ((3, 3, 3), 1)])
def test_volume_classes_cover_each_element_once_per_chunk(cells, order):
    """tables.tc_volume_classes (tensor-core volume kernel): every element
    sits in exactly one task slot, a task's elements share the geometry
    record (so one summed stiffness serves the warp), tasks stay inside
    their element chunk [ne k / 8, ne (k+1) / 8) (chunked host-data
    launches), and the class tables are sum_p M_p KS_p."""
    from paper_1403_1157_b200.tables import VOL_CHUNKS, tc_volume_classes, vol_chunk_bounds
    t = build_tables(DGSpace(unit_cube(*cells), order, 6), PlaqueModel(), FluxScheme("cdg2"))
    r = tc_volume_classes(t)
    assert r is not None
    tabs, perm, tcls, toff = r
    ne = t.elem_geo.shape[0]
    ids = perm[perm >= 0]
    assert np.array_equal(np.sort(ids), np.arange(ne))
    assert (perm[:, 0] >= 0).all()
    assert toff[0] == 0 and toff[-1] == len(perm) and (np.diff(toff) >= 0).all()
    geo = t.elem_geo
    cb = vol_chunk_bounds(ne)
    assert all(b % 8 == 0 for b in cb[:-1]) and cb[-1] == ne
    for k in range(VOL_CHUNKS):
        e0, e1 = cb[k], cb[k + 1]
        blk = perm[toff[k]:toff[k + 1]]
        v = blk[blk >= 0]
        assert ((v >= e0) & (v < e1)).all() and len(v) == e1 - e0
    for task in range(len(perm)):
        v = perm[task][perm[task] >= 0]
        assert (geo[v] == geo[v[0]]).all()
    # class table of the first task's class == sum_p M_p KS_p (fragment layout)
    from paper_1403_1157_b200.tables import _ceil, _frag_kn, _pi_cols
    nb = t.nb
    pic, ok = _pi_cols(nb)
    Kc = np.einsum("p,pij->ij", geo[perm[0, 0], 1:], t.vol_stiff)
    KP = np.zeros((_ceil(nb, 4), _ceil(nb, 8))); KP[:nb] = Kc[:, pic] * ok
    stride = len(tabs) // (tcls.max() + 1)
    assert np.allclose(tabs[tcls[0] * stride:(tcls[0] + 1) * stride], _frag_kn(KP).ravel(),
                       rtol=0, atol=1e-13 * np.abs(Kc).max())


@pytest.mark.parametrize("cells,order", [((6, 4, 4), 2), ((5, 3, 3), 3)])
def test_segment_chunk_runs_read_only_arrived_chunks(cells, order):
    """tables.seg_chunk_offsets (host-data stepping: the first stage runs
    chunk by chunk as the state arrives): within every colour segment the
    faces and walls are ordered by element chunk, run (s, c) holds exactly
    the segment's faces of chunk c, and a face of chunk c touches elements
    of chunks <= c only (all copied in when it runs)."""
    from paper_1403_1157_b200.tables import VOL_CHUNKS, seg_chunk_offsets, vol_chunk_bounds
    t = build_tables(DGSpace(unit_cube(*cells), order, 6), PlaqueModel(), FluxScheme("cdg2"))
    ne = t.elem_geo.shape[0]
    cb = np.asarray(vol_chunk_bounds(ne))
    ch = lambda e: np.searchsorted(cb, e, side="right") - 1
    off = seg_chunk_offsets(t.if_seg, t.if_chunk, t.n_seg)
    assert off[0] == 0 and off[-1] == len(t.if_code)
    for s in range(t.n_seg):
        for c in range(VOL_CHUNKS):
            a, b = off[s * VOL_CHUNKS + c], off[s * VOL_CHUNKS + c + 1]
            assert (t.if_seg[a:b] == s).all() and (t.if_chunk[a:b] == c).all()
            el = t.if_elems[a:b]
            assert (ch(el[:, 0]) <= c).all() and (ch(el[el[:, 1] >= 0, 1]) <= c).all()
            assert (np.maximum(ch(el[:, 0]), ch(np.where(el[:, 1] >= 0, el[:, 1], el[:, 0]))) == c).all()
    bseg = np.repeat(np.arange(t.n_seg), np.diff(t.seg_bf))
    boff = seg_chunk_offsets(bseg, t.bf_chunk, t.n_seg)
    assert boff[-1] == len(t.bf_code)
    assert (ch(t.bf_elem) == t.bf_chunk).all()
