"""Element tiles for the fused single-pass operator kernel.

One CTA of the fused kernel owns a tile of up to ``TE`` elements.  It
gathers their coefficient rows and the rows of their face neighbours
outside the tile (the halo) into shared memory once, evaluates the
volume terms, then every face touching the tile, accumulating into
shared-memory residual rows, and writes each output row exactly once.
A face whose two elements lie in different tiles is evaluated by both
tiles, each writing only its own side; faces inside a tile write both.

This module builds the tiles on the host:

* tiles are consecutive chunks of the owned elements in Morton
  (Z-order) of their centroids, so they are compact blobs on any mesh;
* within a tile the owned rows are sorted by element id (reference-order
  coefficient rows of a tile then form a few long contiguous runs);
* the face entries of a tile are coloured so that no written row appears
  twice in one colour: colours run one after another with a CTA barrier
  in between, so shared-memory accumulation is race-free and the sums
  have a fixed order (bitwise reproducible, no atomics);
* inside a colour, entries are ordered (interior before wall, then by
  trace-table signature) so warps see uniform control flow and tables.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .tables import CODE_MIRROR, OperatorTables

__all__ = ["TileSet", "build_tiles", "CODE_WALL", "CODE_WIN", "CODE_WOUT",
           "SLOT_NONE"]

CODE_WALL = 1 << 16   # prescribed-flux wall face (inside row only)
CODE_WIN = 1 << 17    # accumulate into the inside row (owned by the tile)
CODE_WOUT = 1 << 18   # accumulate into the outside row (owned by the tile)
SLOT_NONE = 0xFFFF


@dataclass
class TileSet:
    te: int
    n_tiles: int
    n_colors: int
    max_rows: int            # owned + halo rows of the largest tile
    rows: np.ndarray         # int32, element row per tile slot (CSR by tile_ptr)
    tile_ptr: np.ndarray     # int32 [T+1]
    tile_nown: np.ndarray    # int32 [T]
    color_ptr: np.ndarray    # int32 [T*(NC+1)] offsets into the entry arrays
    ent_slots: np.ndarray    # int32 slot_in | slot_out << 16
    ent_code: np.ndarray     # int32
    ent_geo: np.ndarray      # float64 [nent, 2d+4]

    def stats(self) -> dict:
        nown = self.tile_nown.astype(np.int64)
        rows = np.diff(self.tile_ptr).astype(np.int64)
        return {"tiles": self.n_tiles, "colors": self.n_colors,
                "halo_fraction": float((rows - nown).sum() / nown.sum()),
                "entries": int(len(self.ent_code)),
                "max_rows": int(self.max_rows)}


def _morton(cen: np.ndarray) -> np.ndarray:
    d = cen.shape[1]
    bits = 20 if d == 2 else 16
    lo, hi = cen.min(axis=0), cen.max(axis=0)
    q = ((cen - lo) / np.maximum(hi - lo, 1e-300) * ((1 << bits) - 1)).astype(np.int64)
    code = np.zeros(len(cen), dtype=np.int64)
    for b in range(bits):
        for a in range(d):
            code |= ((q[:, a] >> b) & 1) << (b * d + a)
    return code


def _color(ent_tile, w_in, w_out, n_el) -> np.ndarray:
    """Conflict-free colours: no (tile, written row) twice per colour.
    Iterative vectorised greedy: every conflicting entry but the first
    moves to the next colour until no conflicts remain."""
    n = len(ent_tile)
    color = np.zeros(n, dtype=np.int64)
    idx = np.arange(n)
    while True:
        keys = []
        ids = []
        for w in (w_in, w_out):
            ok = w >= 0
            keys.append((color[ok] * (n_el + 1) + w[ok]))
            ids.append(idx[ok])
        key = np.concatenate(keys)
        eid = np.concatenate(ids)
        order = np.lexsort((eid, key))
        ks, es = key[order], eid[order]
        dup = np.zeros(len(ks), dtype=bool)
        dup[1:] = ks[1:] == ks[:-1]
        bump = np.unique(es[dup])
        if len(bump) == 0:
            return color
        color[bump] += 1


def build_tiles(t: OperatorTables, centroids: np.ndarray, te: int = 256) -> TileSet:
    """Tile the owned elements (rows [0, n_owned)) of ``t``."""
    n_own = t.elem_geo.shape[0]
    d = t.dim
    nfg = 2 * d + 4
    order = np.argsort(_morton(centroids[:n_own]), kind="stable")
    n_tiles = max(1, (n_own + te - 1) // te)
    tile_of = np.full(max(n_own, 1) + 0, -1, dtype=np.int64)
    tile_of[order] = np.arange(n_own) // te
    # owned rows per tile sorted by element id
    own_tile = tile_of[:n_own]
    own_sorted = np.lexsort((np.arange(n_own), own_tile))
    own_cnt = np.bincount(own_tile, minlength=n_tiles)
    own_start = np.concatenate([[0], np.cumsum(own_cnt)])
    own_slot = np.empty(n_own, dtype=np.int64)
    own_slot[own_sorted] = np.arange(n_own) - own_start[own_tile[own_sorted]]

    def tile_of_row(e):
        out = np.full(len(e), -1, dtype=np.int64)
        ok = (e >= 0) & (e < n_own)
        out[ok] = tile_of[e[ok]]
        return out

    # face entries: (tile, e_in, e_out, code, geo, write flags)
    ein, eout = t.if_elems[:, 0].astype(np.int64), t.if_elems[:, 1].astype(np.int64)
    code = t.if_code.astype(np.int64)
    mirror = (code & CODE_MIRROR) != 0
    tin, tout = tile_of_row(ein), tile_of_row(np.where(mirror, -1, eout))
    ent = []
    # inside-owned entries (also carry the outside when it is in the same tile)
    a = np.flatnonzero(tin >= 0)
    same = (tout[a] == tin[a])
    ent.append((tin[a], a, np.where(same, CODE_WIN | CODE_WOUT, CODE_WIN), 0))
    # outside-owned entries when the outside lives in another tile
    b = np.flatnonzero((tout >= 0) & (tout != tin))
    ent.append((tout[b], b, np.full(len(b), CODE_WOUT), 0))
    ent_tile = np.concatenate([e[0] for e in ent])
    ent_face = np.concatenate([e[1] for e in ent])
    ent_flag = np.concatenate([e[2] for e in ent])
    e_in, e_out = ein[ent_face], eout[ent_face]
    e_code = code[ent_face] | ent_flag
    e_geo = t.if_geo[ent_face]
    # prescribed-flux wall faces
    nb = len(t.bf_code)
    if nb:
        bin_ = t.bf_elem.astype(np.int64)
        ent_tile = np.concatenate([ent_tile, tile_of_row(bin_)])
        e_in = np.concatenate([e_in, bin_])
        e_out = np.concatenate([e_out, np.full(nb, -1)])
        e_code = np.concatenate([e_code, t.bf_code.astype(np.int64) | CODE_WALL | CODE_WIN])
        g = np.zeros((nb, nfg))
        g[:, 2 * d] = t.bf_geo
        e_geo = np.concatenate([e_geo, g])
    assert np.all(ent_tile >= 0)

    # halo rows: non-owned-by-tile elements referenced by the entries
    refs_t = np.concatenate([ent_tile, ent_tile])
    refs_e = np.concatenate([e_in, e_out])
    ok = refs_e >= 0
    refs_t, refs_e = refs_t[ok], refs_e[ok]
    is_own = (refs_e < n_own) & (tile_of_row(refs_e) == refs_t)
    ht, he = refs_t[~is_own], refs_e[~is_own]
    hkey = np.unique(ht * (len(t.elem_geo) + 10 ** 9) + he) if len(ht) else np.zeros(0, np.int64)
    base = len(t.elem_geo) + 10 ** 9
    ht_u, he_u = hkey // base, hkey % base
    h_cnt = np.bincount(ht_u, minlength=n_tiles)
    h_start = np.concatenate([[0], np.cumsum(h_cnt)])
    h_rank = np.arange(len(hkey)) - h_start[ht_u]

    def slot_of(tile, e):
        s = np.full(len(e), SLOT_NONE, dtype=np.int64)
        valid = e >= 0
        own = valid & (e < n_own)
        own &= tile_of_row(np.where(own, e, -1)) == tile
        s[own] = own_slot[e[own]]
        halo = valid & ~own
        if halo.any():
            q = tile[halo] * base + e[halo]
            pos = np.searchsorted(hkey, q)
            assert np.all(hkey[pos] == q)
            s[halo] = own_cnt[tile[halo]] + h_rank[pos]
        return s

    s_in, s_out = slot_of(ent_tile, e_in), slot_of(ent_tile, e_out)
    w_in = np.where((e_code & CODE_WIN) != 0, ent_tile * (te + 1) + s_in, -1)
    w_out = np.where((e_code & CODE_WOUT) != 0, ent_tile * (te + 1) + s_out, -1)
    color = _color(ent_tile, w_in, w_out, n_tiles * (te + 1))
    nc = int(color.max()) + 1 if len(color) else 1
    kind = ((e_code & CODE_WALL) != 0).astype(np.int64)
    sig = e_code & 1023
    eo = np.lexsort((sig, kind, color, ent_tile))
    ent_tile, color = ent_tile[eo], color[eo]
    s_in, s_out, e_code, e_geo = s_in[eo], s_out[eo], e_code[eo], e_geo[eo]
    cnt = np.bincount(ent_tile * nc + color, minlength=n_tiles * nc).reshape(n_tiles, nc)
    cptr = np.zeros((n_tiles, nc + 1), dtype=np.int64)
    cptr[:, 1:] = np.cumsum(cnt, axis=1)
    cptr += np.concatenate([[0], np.cumsum(cnt.sum(axis=1))[:-1]])[:, None]

    rows = []
    tile_ptr = np.zeros(n_tiles + 1, dtype=np.int64)
    own_rows = own_sorted  # element ids grouped by tile, sorted by id
    for k in range(n_tiles):
        r = np.concatenate([own_rows[own_start[k]:own_start[k + 1]],
                            he_u[h_start[k]:h_start[k + 1]]])
        rows.append(r)
        tile_ptr[k + 1] = tile_ptr[k] + len(r)
    rows = np.concatenate(rows) if rows else np.zeros(0, np.int64)
    i32 = lambda x: np.ascontiguousarray(x, dtype=np.int32)
    return TileSet(
        te=te, n_tiles=n_tiles, n_colors=nc,
        max_rows=int(np.diff(tile_ptr).max()) if n_tiles else 0,
        rows=i32(rows), tile_ptr=i32(tile_ptr), tile_nown=i32(own_cnt),
        color_ptr=i32(cptr.reshape(-1)),
        ent_slots=i32(s_in | (s_out << 16)), ent_code=i32(e_code),
        ent_geo=np.ascontiguousarray(e_geo, dtype=np.float64))
