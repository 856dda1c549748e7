"""Conforming simplicial meshes with a vectorised face table.

Host-side setup.  Reproduces the conventions of the reference mesh
(``pkg/src/taxisdg/mesh.py``) that the operator's results depend on:

* element orientation: negative signed volume swaps the last two
  vertices (``mesh.py:138-149``);
* signed volumes, centroids, diameters (``mesh.py:127-159``) -- the
  volumes feed the K- tie rule, so they are computed with the same
  numpy calls;
* face table: faces are keyed by their sorted vertex ids; side 0 is the
  first element touching the face in element-scan order, side 1 the
  second; faces are numbered by first touch (``mesh.py:161-214``); the
  per-side local-face index and vertex permutation index
  (``LOCAL_FACES``/``PERMUTATIONS``, ``mesh.py:61-71``); unit normal
  outward from side 0 and measure (``mesh.py:216-234``);
* affine maps x = v0 + J xi with J's columns the edges from v0
  (``mesh.py:267-277``).

Unlike the reference (a Python loop, ~45 us per triangle) the face table
is built with sorts over all element-local faces, so the C2/C3/C4
meshes build in seconds.
"""

from __future__ import annotations

import itertools
from enum import IntEnum

import numpy as np

__all__ = ["BoundaryTag", "is_gamma1", "LOCAL_FACES", "PERMUTATIONS",
           "REF_VERTICES", "MeshError", "Mesh", "unit_square", "unit_cube"]


class MeshError(ValueError):
    pass


class BoundaryTag(IntEnum):
    """Boundary classes (reference ``mesh.py:46-52``); 0 = interior."""
    GAMMA1 = 1
    GAMMA1_IN = 2
    GAMMA2 = 3
    NO_FLOW = 4


def is_gamma1(tag: int) -> bool:
    return int(tag) in (BoundaryTag.GAMMA1, BoundaryTag.GAMMA1_IN)


LOCAL_FACES = {
    2: ((1, 2), (2, 0), (0, 1)),
    3: ((1, 2, 3), (0, 2, 3), (0, 1, 3), (0, 1, 2)),
}
PERMUTATIONS = {
    2: ((0, 1), (1, 0)),
    3: tuple(itertools.permutations((0, 1, 2))),
}
REF_VERTICES = {
    2: np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]]),
    3: np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0],
                 [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]]),
}


def _perm_codes(dim: int) -> np.ndarray:
    """Lookup: base-dim code of a permutation tuple -> its index."""
    lut = np.full(dim ** dim, -1, dtype=np.int8)
    for idx, p in enumerate(PERMUTATIONS[dim]):
        code = 0
        for v in p:
            code = code * dim + v
        lut[code] = idx
    return lut


def signed_volumes(vertices: np.ndarray, elements: np.ndarray) -> np.ndarray:
    """Same arithmetic as reference ``mesh.py:127-136``; the K- rule
    compares these values for exact ties."""
    v0 = vertices[elements[:, 0]]
    edges = vertices[elements[:, 1:]] - v0[:, None, :]
    if vertices.shape[1] == 2:
        det = edges[:, 0, 0] * edges[:, 1, 1] - edges[:, 0, 1] * edges[:, 1, 0]
        return det / 2.0
    return np.linalg.det(edges) / 6.0


class Mesh:
    """Unstructured conforming simplicial mesh in 2 or 3 dimensions.

    ``boundary_tags`` is a dict {sorted vertex tuple: tag} (the
    reference's API) or None; ``tag_fn(keys) -> tags`` is a vectorised
    alternative used by the structured generators.
    """

    def __init__(self, vertices, elements, boundary_tags=None,
                 default_tag: int = BoundaryTag.NO_FLOW, tag_fn=None):
        vertices = np.ascontiguousarray(vertices, dtype=float)
        elements = np.ascontiguousarray(elements, dtype=np.int64)
        if vertices.ndim != 2 or vertices.shape[1] not in (2, 3):
            raise MeshError(f"vertices must be (n, 2|3), got {vertices.shape}")
        dim = vertices.shape[1]
        if elements.ndim != 2 or elements.shape[1] != dim + 1:
            raise MeshError(f"elements must be (n, {dim + 1})")
        if elements.size and (elements.min() < 0
                              or elements.max() >= len(vertices)):
            raise MeshError("element vertex index out of range")
        self.dim = dim
        self.vertices = vertices
        self.elements = self._orient(vertices, elements)
        self._geometry()
        self._faces(boundary_tags or {}, int(default_tag), tag_fn)
        self._jac = None

    # -- construction ----------------------------------------------------

    @staticmethod
    def _orient(vertices, elements):
        vols = signed_volumes(vertices, elements)
        scale = np.abs(vols).max(initial=1.0)
        if np.any(np.abs(vols) <= 1e-14 * scale):
            bad = int(np.argmin(np.abs(vols)))
            raise MeshError(f"element {bad} is degenerate")
        out = elements.copy()
        neg = vols < 0
        out[neg, -2] = elements[neg, -1]
        out[neg, -1] = elements[neg, -2]
        return out

    def _geometry(self):
        self.volumes = signed_volumes(self.vertices, self.elements)
        corners = self.vertices[self.elements]
        self.centroids = corners.mean(axis=1)
        diam = np.zeros(len(self.elements))
        for a, b in itertools.combinations(range(self.dim + 1), 2):
            np.maximum(diam, np.linalg.norm(corners[:, a] - corners[:, b],
                                            axis=1), out=diam)
        self.diameters = diam

    def _faces(self, tag_dict, default_tag, tag_fn):
        dim, ne = self.dim, len(self.elements)
        nl = dim + 1
        loc = np.array(LOCAL_FACES[dim])                      # (nl, dim)
        ev = self.elements[:, loc]                            # (ne, nl, dim)
        keys = np.sort(ev, axis=2).reshape(-1, dim)
        order = np.lexsort(tuple(keys[:, c] for c in range(dim - 1, -1, -1)))
        sk = keys[order]
        start = np.ones(len(sk), dtype=bool)
        start[1:] = np.any(sk[1:] != sk[:-1], axis=1)
        starts = np.flatnonzero(start)
        counts = np.diff(np.append(starts, len(sk)))
        if np.any(counts > 2):
            raise MeshError("mesh is not conforming (face shared by > 2)")
        first = order[starts]                 # flat e*nl+lf, smallest touch
        second = np.where(counts == 2, order[np.minimum(starts + 1,
                                                         len(sk) - 1)], -1)
        fo = np.argsort(first, kind="stable")  # number faces by first touch
        first, second = first[fo], second[fo]
        nf = len(first)
        self.face_vertices = keys[first]
        fe = np.full((nf, 2), -1, dtype=np.int64)
        fl = np.full((nf, 2), -1, dtype=np.int8)
        fp = np.full((nf, 2), -1, dtype=np.int8)
        lut = _perm_codes(dim)
        for col, flat in enumerate((first, second)):
            ok = flat >= 0
            e = flat[ok] // nl
            lf = flat[ok] % nl
            fe[ok, col] = e
            fl[ok, col] = lf
            p = np.argsort(ev[e, lf], axis=1)   # ef[p[i]] == key[i]
            code = np.zeros(len(e), dtype=np.int64)
            for c in range(dim):
                code = code * dim + p[:, c]
            fp[ok, col] = lut[code]
        self.face_elems, self.face_local, self.face_perm = fe, fl, fp
        self._face_geometry()
        tags = np.zeros(nf, dtype=np.int8)
        bnd = np.flatnonzero(fe[:, 1] < 0)
        if tag_fn is not None:
            tags[bnd] = np.asarray(tag_fn(self.face_vertices[bnd]),
                                   dtype=np.int8)
        else:
            tags[bnd] = default_tag
            if tag_dict:
                lookup = {tuple(int(v) for v in self.face_vertices[f]): f
                          for f in bnd}
                for key, tag in tag_dict.items():
                    f = lookup.get(tuple(sorted(int(v) for v in key)))
                    if f is None:
                        raise MeshError(f"tagged face {key} is not a "
                                        "boundary face")
                    tags[f] = int(tag)
        if np.any((tags[bnd] < 1) | (tags[bnd] > 4)):
            raise MeshError("invalid boundary tag")
        self.face_tags = tags

    def _face_geometry(self):
        pts = self.vertices[self.face_vertices]               # (nf, dim, dim)
        if self.dim == 2:
            t = pts[:, 1] - pts[:, 0]
            meas = np.sqrt(t[:, 0] ** 2 + t[:, 1] ** 2)
            nrm = np.stack([t[:, 1], -t[:, 0]], axis=1) / meas[:, None]
        else:
            cr = np.cross(pts[:, 1] - pts[:, 0], pts[:, 2] - pts[:, 0])
            ln = np.sqrt((cr ** 2).sum(axis=1))
            meas = ln / 2.0
            nrm = cr / ln[:, None]
        e = self.face_elems[:, 0]
        lf = self.face_local[:, 0].astype(np.int64)
        opp = self.vertices[self.elements[e, lf]]
        flip = np.einsum("fd,fd->f", nrm, pts.mean(axis=1) - opp) < 0
        nrm[flip] *= -1.0
        self.face_normals = nrm
        self.face_measures = meas

    # -- queries -----------------------------------------------------------

    @property
    def n_vertices(self) -> int:
        return len(self.vertices)

    @property
    def n_elements(self) -> int:
        return len(self.elements)

    @property
    def n_faces(self) -> int:
        return len(self.face_vertices)

    @property
    def boundary_mask(self) -> np.ndarray:
        return self.face_elems[:, 1] < 0

    def jacobians(self):
        """(J, detJ, Jinv) with the reference's numpy calls."""
        if self._jac is None:
            v0 = self.vertices[self.elements[:, 0]]
            J = np.ascontiguousarray(np.swapaxes(
                self.vertices[self.elements[:, 1:]] - v0[:, None, :], 1, 2))
            self._jac = (J, np.linalg.det(J), np.ascontiguousarray(
                np.linalg.inv(J)))
        return self._jac

    def boundary_measure(self, tag: int) -> float:
        return float(self.face_measures[self.face_tags == int(tag)].sum())

    def partition(self, nparts: int) -> np.ndarray:
        """Recursive coordinate bisection on centroids (reference
        ``mesh.py:432-456``): split on the widest axis, order by
        (coordinate, element id), left part gets len*floor(P/2)/P."""
        if nparts < 1:
            raise ValueError("nparts must be >= 1")
        parts = np.zeros(self.n_elements, dtype=np.int64)
        stack = [(np.arange(self.n_elements), 0, nparts)]
        while stack:
            idx, first, count = stack.pop()
            if count == 1:
                parts[idx] = first
                continue
            cen = self.centroids[idx]
            axis = int(np.argmax(cen.max(axis=0) - cen.min(axis=0)))
            order = np.lexsort((idx, cen[:, axis]))
            lp = count // 2
            nleft = len(idx) * lp // count
            stack.append((idx[order[:nleft]], first, lp))
            stack.append((idx[order[nleft:]], first + lp, count - lp))
        return parts


# ---------------------------------------------------------------------------
# structured generators (element order, vertex order and tags as in the
# reference generators ``mesh.py:463-554``)


def _square_parts(nx, ny, gamma1_in, lengths, jitter, seed, cells_x):
    """Vertices, elements (two triangles (a,b,c), (a,c,d) per cell, cell
    order x fastest), global element ids and the tag function of the
    cell columns [cells_x[0], cells_x[1]) of the nx x ny grid.  Vertex
    coordinates are the global grid's, bit for bit."""
    i0, i1 = cells_x
    xs = np.linspace(0.0, 1.0, nx + 1)
    ys = np.linspace(0.0, 1.0, ny + 1)
    nvx = i1 - i0 + 1                               # local vertex columns
    X, Y = np.meshgrid(xs[i0:i1 + 1], ys)
    verts = np.stack([X.ravel(), Y.ravel()], axis=1)
    I, J = np.meshgrid(np.arange(i1 - i0), np.arange(ny))
    I, J = I.ravel(), J.ravel()
    a = J * nvx + I
    b, c, d = a + 1, a + nvx + 1, a + nvx
    elems = np.empty((2 * len(a), 3), dtype=np.int64)
    elems[0::2] = np.stack([a, b, c], axis=1)
    elems[1::2] = np.stack([a, c, d], axis=1)
    gcell = J * nx + (I + i0)
    gids = np.empty(2 * len(a), dtype=np.int64)
    gids[0::2] = 2 * gcell
    gids[1::2] = 2 * gcell + 1

    def tag_fn(keys):
        vi, vj = keys % nvx + i0, keys // nvx          # global grid indices
        tags = np.full(len(keys), int(BoundaryTag.NO_FLOW), dtype=np.int8)
        bottom = (vj[:, 0] == 0) & (vj[:, 1] == 0)
        top = (vj[:, 0] == ny) & (vj[:, 1] == ny)
        g0 = vi.min(axis=1)
        mid = 0.5 * (xs[g0] + xs[np.minimum(g0 + 1, nx)])
        inflow = (gamma1_in[0] <= mid) & (mid <= gamma1_in[1])
        tags[bottom] = np.where(inflow[bottom], int(BoundaryTag.GAMMA1_IN),
                                int(BoundaryTag.GAMMA1))
        tags[top] = int(BoundaryTag.GAMMA2)
        return tags

    if tuple(lengths) != (1.0, 1.0):
        verts = verts * np.asarray(lengths, dtype=float)[None, :]
    if jitter > 0.0:
        # the global jitter field, sliced: slabs see the same vertices
        rng = np.random.default_rng(seed)
        h = np.asarray(lengths, dtype=float) / np.array([nx, ny])
        shift = rng.uniform(-jitter, jitter, size=((ny + 1) * (nx + 1), 2)) * h[None, :]
        gvi = np.arange(len(verts)) % nvx + i0
        gvj = np.arange(len(verts)) // nvx
        interior = (gvi > 0) & (gvi < nx) & (gvj > 0) & (gvj < ny)
        verts = verts.copy()
        verts[interior] += shift[(gvj * (nx + 1) + gvi)[interior]]
    return verts, elems, gids, tag_fn


def unit_square(nx: int, ny: int | None = None,
                gamma1_in=(0.25, 0.75), lengths=(1.0, 1.0),
                jitter: float = 0.0, seed: int = 0) -> Mesh:
    """Two triangles (a,b,c), (a,c,d) per cell of an nx x ny grid.

    Tags follow the reference generator on the unit square (bottom
    GAMMA1 with GAMMA1_IN where the edge midpoint x is inside
    ``gamma1_in``, top GAMMA2, sides NO_FLOW); ``lengths`` then scales
    the coordinates (config C2/C3 use [0,4]x[0,1]).  ``jitter`` > 0
    moves every interior vertex by a seeded U(-jitter*h, jitter*h) per
    coordinate, h the cell size along that axis (config C3).
    """
    ny = nx if ny is None else ny
    if nx < 1 or ny < 1:
        raise ValueError("nx and ny must be >= 1")
    verts, elems, _, tag_fn = _square_parts(nx, ny, gamma1_in, lengths,
                                            jitter, seed, (0, nx))
    return Mesh(verts, elems, tag_fn=tag_fn)


# Kuhn triangulation: monotone vertex paths 0 -> 7 through the cube
# corners (bit 0 = +x, bit 1 = +y, bit 2 = +z), one per axis permutation
KUHN_PATHS = [(0, 1 << p0, (1 << p0) | (1 << p1), 7)
              for p0, p1, _ in itertools.permutations((0, 1, 2))]


def _cube_parts(nx, ny, nz, gamma1_in, top_tag, lengths, cells_x):
    i0, i1 = cells_x
    xs = np.linspace(0.0, 1.0, nx + 1)
    ys = np.linspace(0.0, 1.0, ny + 1)
    zs = np.linspace(0.0, 1.0, nz + 1)
    nvx = i1 - i0 + 1
    Z, Y, X = np.meshgrid(zs, ys, xs[i0:i1 + 1], indexing="ij")
    verts = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)
    K, J, I = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(i1 - i0),
                          indexing="ij")
    I, J, K = I.ravel(), J.ravel(), K.ravel()

    def vid(i, j, k):
        return (k * (ny + 1) + j) * nvx + i

    elems = np.empty((6 * len(I), 4), dtype=np.int64)
    for t, path in enumerate(KUHN_PATHS):
        elems[t::6] = np.stack([vid(I + (b & 1), J + ((b >> 1) & 1),
                                    K + ((b >> 2) & 1)) for b in path], axis=1)
    gcell = (K * ny + J) * nx + (I + i0)
    gids = (6 * gcell[:, None] + np.arange(6)[None, :]).ravel()

    def tag_fn(keys):
        vi = keys % nvx + i0
        vj = (keys // nvx) % (ny + 1)
        vk = keys // (nvx * (ny + 1))
        tags = np.full(len(keys), int(BoundaryTag.NO_FLOW), dtype=np.int8)
        bottom = np.all(vk == 0, axis=1)
        top = np.all(vk == nz, axis=1)
        g0, h0 = vi.min(axis=1), vj.min(axis=1)
        cx = 0.5 * (xs[g0] + xs[np.minimum(g0 + 1, nx)])
        cy = 0.5 * (ys[h0] + ys[np.minimum(h0 + 1, ny)])
        if gamma1_in is None:
            inflow = np.zeros(len(keys), dtype=bool)
        else:
            x0, x1, y0, y1 = gamma1_in
            inflow = (x0 <= cx) & (cx <= x1) & (y0 <= cy) & (cy <= y1)
        tags[bottom] = np.where(inflow[bottom], int(BoundaryTag.GAMMA1_IN),
                                int(BoundaryTag.GAMMA1))
        if top_tag is not None:
            tags[top] = int(top_tag)
        return tags

    if tuple(lengths) != (1.0, 1.0, 1.0):
        verts = verts * np.asarray(lengths, dtype=float)[None, :]
    return verts, elems, gids, tag_fn


def unit_cube(nx: int, ny: int | None = None, nz: int | None = None,
              gamma1_in=(0.25, 0.75, 0.25, 0.75), top_tag=BoundaryTag.GAMMA2,
              lengths=(1.0, 1.0, 1.0)) -> Mesh:
    """Six Kuhn tetrahedra per cell.  Bottom (z=0) GAMMA1 with the
    rectangle ``gamma1_in`` = (x0, x1, y0, y1) tagged GAMMA1_IN by cell
    centre (None: no inflow patch), top ``top_tag`` (reference: GAMMA2),
    everything else NO_FLOW."""
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    if min(nx, ny, nz) < 1:
        raise ValueError("nx, ny, nz must be >= 1")
    verts, elems, _, tag_fn = _cube_parts(nx, ny, nz, gamma1_in, top_tag,
                                          lengths, (0, nx))
    return Mesh(verts, elems, tag_fn=tag_fn)
