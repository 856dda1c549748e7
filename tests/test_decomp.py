"""x-slab decomposition: slab meshes, ghost ordering and the halo
exchange (world_size 2 with gloo on CPU), checked with the CPU oracle
against the undecomposed operator."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import OracleOperator
from paper_1403_1157_b200 import DGSpace, FluxScheme, PlaqueModel, PlaqueParams
from paper_1403_1157_b200.configs import CONFIGS, Config, make_mesh
from paper_1403_1157_b200.decomp import HaloExchange, build_slab, slab_ranges
from paper_1403_1157_b200.fields import bump_field

from _cases import AMPLIFIED

SMALL = {
    "c2": ((16, 4), {}),
    "c3": ((16, 4), {}),
    "c4": ((6, 3, 3), {}),
    "c5": ((6, 3, 3), {}),
}


def _problem(name, cells, rank=None, nranks=None):
    cfg = CONFIGS[name]
    params = PlaqueParams(**AMPLIFIED)
    if rank is None:
        mesh = make_mesh(cfg, cells=cells)
        gids = np.arange(mesh.n_elements)
        n_own = mesh.n_elements
    else:
        sl = build_slab(cfg, rank, nranks, cells=cells)
        mesh, gids, n_own = sl.mesh, sl.global_ids, sl.n_owned
    order = 1 if cfg.dim == 3 else 2
    space = DGSpace(mesh, order, 6)
    lo = np.zeros(cfg.dim)
    hi = np.asarray(cfg.lengths, dtype=float)
    U = space.project(bump_field(cfg.dim, 6, 3, lo, hi)).coeffs
    return space, PlaqueModel(params), U, gids, n_own


def test_slab_ranges():
    assert slab_ranges(10, 3) == [(0, 3), (3, 6), (6, 10)]
    with pytest.raises(ValueError):
        slab_ranges(2, 3)


@pytest.mark.parametrize("name", sorted(SMALL))
def test_slab_geometry_is_bitwise_global(name):
    cells = SMALL[name][0]
    gspace, _, _, _, _ = _problem(name, cells)
    gm = gspace.mesh
    for r in range(3):
        sl = build_slab(CONFIGS[name], r, 3, cells=cells)
        m = sl.mesh
        assert np.array_equal(m.volumes, gm.volumes[sl.global_ids])
        assert np.array_equal(m.diameters, gm.diameters[sl.global_ids])
        assert np.array_equal(m.vertices[m.elements], gm.vertices[gm.elements[sl.global_ids]])
        assert len(set(sl.global_ids[:sl.n_owned])) == sl.n_owned


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, nranks, port, name, cells, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=nranks)
    try:
        space, model, U, gids, n_own = _problem(name, cells, rank, nranks)
        Ut = torch.from_numpy(np.ascontiguousarray(U))
        Ut[n_own:] = float("nan")          # ghosts must come from the exchange
        sl = build_slab(CONFIGS[name], rank, nranks, cells=cells)
        HaloExchange(sl).exchange(Ut)
        assert not torch.isnan(Ut).any()
        op = OracleOperator(space, model, FluxScheme("cdg2"), global_ids=gids)
        R = op.apply(Ut.numpy())[:n_own]
        out[rank] = (gids[:n_own], R)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["c2", "c4"])
def test_gloo_two_ranks_match_global_operator(name):
    cells = SMALL[name][0]
    space, model, U, _, _ = _problem(name, cells)
    ref = OracleOperator(space, model, FluxScheme("cdg2")).apply(U)
    nranks = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.start_processes(_worker, args=(nranks, port, name, cells, out),
                       nprocs=nranks, start_method="spawn")
    covered = np.zeros(space.mesh.n_elements, dtype=int)
    for r in range(nranks):
        gids, R = out[r]
        covered[gids] += 1
        assert np.abs(R - ref[gids]).max() <= 1e-13 * np.abs(ref).max()
    assert np.all(covered == 1)
