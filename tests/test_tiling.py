"""Host tiling for the fused operator kernel: ownership, write-once face
sides, conflict-free colours, and the fused accumulation order emulated
against the reference golden outputs."""
import numpy as np
import pytest

from paper_1403_1157_b200 import (DGSpace, DiffusionModel, FluxScheme,
                                  PlaqueModel, unit_cube, unit_square)
from paper_1403_1157_b200.tables import build_tables, scheme_constants
from paper_1403_1157_b200.tiling import (CODE_WALL, CODE_WIN, CODE_WOUT,
                                         build_tiles)

from _cases import operator_case
from _device_emulator import DeviceEmulator
from test_oracle_golden import _golden_names


def _check_invariants(t, tiles, n_own):
    owned = np.concatenate([tiles.rows[tiles.tile_ptr[k]:tiles.tile_ptr[k] + tiles.tile_nown[k]]
                            for k in range(tiles.n_tiles)])
    assert np.array_equal(np.sort(owned), np.arange(n_own))
    # every face side that must be written is written exactly once
    writes = {}
    nc = tiles.n_colors
    for k in range(tiles.n_tiles):
        rows = tiles.rows[tiles.tile_ptr[k]:tiles.tile_ptr[k + 1]]
        nown = tiles.tile_nown[k]
        for c in range(nc):
            seen = set()
            b, e = tiles.color_ptr[k * (nc + 1) + c], tiles.color_ptr[k * (nc + 1) + c + 1]
            for j in range(b, e):
                code = int(tiles.ent_code[j])
                si = int(tiles.ent_slots[j]) & 0xFFFF
                so = (int(tiles.ent_slots[j]) >> 16) & 0xFFFF
                for flag, slot in ((CODE_WIN, si), (CODE_WOUT, so)):
                    if code & flag:
                        assert slot < nown
                        assert slot not in seen, "colour conflict"
                        seen.add(slot)
                        writes[(int(rows[slot]), j, flag)] = 1
    n_sides = 0
    for f in range(len(t.if_code)):
        n_sides += 1 + int(not (int(t.if_code[f]) & ((1 << 14) | (1 << 15))))
    n_sides += len(t.bf_code)
    assert len(writes) == n_sides


@pytest.mark.parametrize("name", [n for n in _golden_names() if "_p0_" not in n])
@pytest.mark.parametrize("te", [8, 64])
def test_fused_order_matches_reference(golden, name, te):
    space, model, scheme, U, R, _ = operator_case(golden, name)
    t = build_tables(space, model, scheme)
    tiles = build_tiles(t, space.mesh.centroids, te=te)
    _check_invariants(t, tiles, space.mesh.n_elements)
    em = DeviceEmulator(t, model, scheme.id, *scheme_constants(space, scheme))
    got = em.apply_tiled(U, tiles)
    assert np.abs(got - R).max() <= 1e-12 * np.abs(R).max()


@pytest.mark.parametrize("dirichlet", [0, 1])
def test_fused_order_heat(golden, dirichlet):
    h = golden["heat"]
    space = DGSpace(unit_square(3), 2)
    model = DiffusionModel(0.7, dirichlet=0.4 if dirichlet else None)
    for scheme in ("cdg2", "br2", "ip"):
        key = f"heat_sq3_{scheme}_{dirichlet}"
        sc = FluxScheme(scheme)
        t = build_tables(space, model, sc)
        tiles = build_tiles(t, space.mesh.centroids, te=8)
        _check_invariants(t, tiles, space.mesh.n_elements)
        em = DeviceEmulator(t, model, sc.id, *scheme_constants(space, sc))
        got = em.apply_tiled(h[f"{key}__U"], tiles)
        R = h[f"{key}__R"]
        assert np.abs(got - R).max() <= 1e-12 * np.abs(R).max()


def test_tiles_at_c2_size():
    space = DGSpace(unit_square(512, 128, lengths=(4.0, 1.0)), 2, 6)
    t = build_tables(space, PlaqueModel(), FluxScheme("cdg2"))
    tiles = build_tiles(t, space.mesh.centroids, te=256)
    st = tiles.stats()
    assert st["tiles"] == 512 and st["colors"] <= 6 and st["halo_fraction"] < 0.3
    assert tiles.max_rows < 400


def test_element_bands_order_faces_for_host_pipelined_steps():
    """tables.build_tables bands: contiguous element ranges; interior faces
    ordered (lowest band, straddle, signature): faces [2k, 2k+1) lie in band
    k, faces [2k+1, 2k+2) straddle (k, k+1); walls grouped by band; every
    face exactly once; signatures sorted within each group."""
    space = DGSpace(unit_square(128, 128), 1, 6)
    t = build_tables(space, PlaqueModel(), FluxScheme("cdg2"), bands=4)
    assert t.n_bands == 4
    eb = t.band_elem_ptr
    assert eb[0] == 0 and eb[-1] == space.mesh.n_elements and np.all(np.diff(eb) > 0)
    band = lambda e: np.searchsorted(eb, e, side="right") - 1
    fp = t.band_face_ptr
    assert fp[0] == 0 and fp[-1] == len(t.if_code) and np.all(np.diff(fp) >= 0)
    el = t.if_elems
    for k in range(4):
        a, b, c = fp[2 * k], fp[2 * k + 1], fp[2 * k + 2]
        assert np.all(band(el[a:b, 0]) == k) and np.all(band(el[a:b, 1]) == k)
        lo = np.minimum(band(el[b:c, 0]), band(el[b:c, 1]))
        hi = np.maximum(band(el[b:c, 0]), band(el[b:c, 1]))
        assert np.all(lo == k) and np.all(hi == k + 1)
        for lo_, hi_ in ((a, b), (b, c)):
            sig = t.if_code[lo_:hi_] & 1023
            assert np.all(np.diff(sig) >= 0)
        w0, w1 = t.band_wall_ptr[k], t.band_wall_ptr[k + 1]
        assert np.all(band(t.bf_elem[w0:w1]) == k)
    # small meshes and slab meshes are not banded
    assert build_tables(DGSpace(unit_square(8), 1, 6), PlaqueModel(), FluxScheme("cdg2")).n_bands == 1


@pytest.mark.parametrize("dim", [2, 3])
def test_face_blocks_respect_band_segments(dim):
    """tc_face_blocks never straddles a band segment (nor a signature), and
    tc_band_blocks gives each band exactly the blocks of its faces (those
    straddling (k-1, k) and those internal to k): the 3D host-pipelined
    steps launch the transposed face kernel per band over these blocks."""
    from paper_1403_1157_b200.tables import tc_band_blocks, tc_face_blocks
    mesh = unit_square(128, 128) if dim == 2 else unit_cube(16)
    t = build_tables(DGSpace(mesh, 1, 6), PlaqueModel(), FluxScheme("cdg2"), bands=3)
    assert t.n_bands == 3
    blocks, ncut = tc_face_blocks(t)
    assert ncut == 0
    first, cnt = blocks[:, 0].astype(np.int64), blocks[:, 1].astype(np.int64)
    assert first[0] == 0 and np.array_equal(first[1:], first[:-1] + cnt[:-1])
    assert first[-1] + cnt[-1] == len(t.if_code) and np.all((cnt >= 1) & (cnt <= 8))
    seg = np.searchsorted(t.band_face_ptr, np.arange(len(t.if_code)), side="right")
    sig = t.if_code & 1023
    for f0, c in zip(first, cnt):
        assert len(set(seg[f0:f0 + c])) == 1 and len(set(sig[f0:f0 + c])) == 1
    bb = tc_band_blocks(t, blocks)
    assert bb[0] == 0 and bb[-1] == len(blocks) and np.all(np.diff(bb) >= 0)
    for k in range(3):
        f_lo = 0 if k == 0 else t.band_face_ptr[2 * k - 1]
        f_hi = t.band_face_ptr[2 * k + 1] if k < 2 else len(t.if_code)
        assert first[bb[k]] == f_lo
        last = bb[k + 1] - 1
        assert first[last] + cnt[last] == f_hi


def test_cpu_baseline_sample_is_a_bounded_slab_of_the_config():
    """bench.sample_config: the CPU baseline of large configs is an x-slab
    (then y-slab in 3D) with the config's cell size, order and physics,
    at most ~5M DoFs; small configs are timed whole."""
    import sys
    import os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    from paper_1403_1157_b200.basis import basis_size
    from paper_1403_1157_b200.configs import CONFIGS
    for name in ("c1", "c2", "c3", "c4", "c5"):
        cfg = bench.weak_config(CONFIGS[name], 1)
        smp = bench.sample_config(cfg)
        per = (2 if cfg.dim == 2 else 6) * 6 * basis_size(cfg.dim, cfg.order)
        dofs = int(np.prod(smp.cells)) * per
        if name in ("c1", "c2"):
            assert smp == cfg
        else:
            assert dofs <= 5_000_000 and smp.order == cfg.order and smp.dim == cfg.dim
        for a in range(cfg.dim):    # same cell size
            assert smp.lengths[a] / smp.cells[a] == pytest.approx(cfg.lengths[a] / cfg.cells[a])
