"""Slab-decomposed implicit stepping (SURVEY 8(e) Krylov row): SDIRK3 +
JFNK + GMRES over two gloo ranks on CPU, with the ghost exchange inside
every G(V) and the Krylov dots / norms all-reduced, equals the same
integrator on the undecomposed mesh.  The operator is a CPU test double
that routes the stage algebra through the oracle (test infrastructure);
the device path runs the identical timeint code with the CUDA library."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import OracleOperator
from paper_1403_1157_b200 import DGSpace, FluxScheme, PlaqueModel, PlaqueParams
from paper_1403_1157_b200.configs import CONFIGS, make_mesh
from paper_1403_1157_b200.decomp import HaloExchange, build_slab
from paper_1403_1157_b200.fields import bump_field
from paper_1403_1157_b200.timeint import SlabReductions, integrate

from _cases import AMPLIFIED

CELLS = (12, 4)
DT = 2e-4
NEWTON = dict(rtol=1e-11, atol=1e-13, gmres_rtol=1e-8, gmres_maxiter=400)


class _CpuStageOp:
    """Duck-typed stand-in for DiscreteOperator's stepping surface on CPU
    tensors (apply via the oracle)."""

    def __init__(self, space, model, gids, n_owned):
        self.space = space
        self.n_owned = n_owned
        self.n_rows = space.mesh.n_elements
        self.device = torch.device("cpu")
        self.oracle = OracleOperator(space, model, FluxScheme("cdg2"), global_ids=gids)

    def rk_stage(self, U0, V, out, a, b, c):
        n = self.n_owned
        f = torch.from_numpy(self.oracle.apply_f(V.numpy())[:n])
        res = b * V[:n] + c * f
        if a != 0.0:
            res = res + a * U0[:n]
        out[:n] = res
        return out

    def rk_stage_part(self, U0, V, out, a, b, c, part):
        if part == 2:
            self.rk_stage(U0, V, out, a, b, c)
        return out

    def dot(self, x, y, out=None):
        v = torch.dot(x.reshape(-1), y.reshape(-1))
        if out is None:
            return v.reshape(1)
        out.copy_(v.reshape(out.shape))
        return out

    def norm2(self, x, out=None):
        v = torch.linalg.vector_norm(x.reshape(-1))
        if out is None:
            return v.reshape(1)
        out.copy_(v.reshape(out.shape))
        return out

    def axpy_dev(self, s, alpha, x, y):
        y.add_(x, alpha=float(s * alpha.reshape(-1)[0]))
        return y

    def mgs_pass(self, V, i, j, w, h, n):
        """tdg_mgs_pass semantics on the first n entries (CPU double)."""
        wv = w.reshape(-1)[:n]
        if i > 0:
            wv.sub_(V[i - 1, :n] * h[i - 1])
        h[i] = torch.dot(wv, wv if i == j + 1 else V[i, :n])
        return h


def _problem(rank=None, nranks=None):
    cfg = CONFIGS["c2"]
    if rank is None:
        mesh = make_mesh(cfg, cells=CELLS)
        gids, n_own, sl = np.arange(mesh.n_elements), mesh.n_elements, None
    else:
        sl = build_slab(cfg, rank, nranks, cells=CELLS)
        mesh, gids, n_own = sl.mesh, sl.global_ids, sl.n_owned
    space = DGSpace(mesh, 2, 6)
    U = space.project(bump_field(2, 6, 3, np.zeros(2), np.asarray(cfg.lengths, float))).coeffs
    op = _CpuStageOp(space, PlaqueModel(PlaqueParams(**AMPLIFIED)), gids, n_own)
    return op, torch.from_numpy(np.ascontiguousarray(U)), gids, n_own, sl


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, nranks, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=nranks)
    try:
        op, U, gids, n_own, sl = _problem(rank, nranks)
        U[n_own:] = float("nan")                      # ghosts come from the exchange
        res = integrate(op, U, 0.0, 2 * DT, DT, order=3, newton_kwargs=NEWTON,
                        halo=HaloExchange(sl))
        # the slab reductions see the whole vector: norm == global norm
        red = SlabReductions(op)
        nrm = float(red.norm2(res.U, torch.zeros(1, dtype=torch.float64)))
        out[rank] = (gids[:n_own], res.U[:n_own].numpy(), res.gmres_iterations, nrm)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("nranks", [2, 4])
def test_slab_sdirk3_jfnk_matches_single_domain(nranks):
    """2 and 4 gloo ranks: the slab SDIRK3 + JFNK path (exchange inside
    G(V); the MGS sweep pass by pass with every pass's dot all-reduced,
    SlabReductions.mgs over tdg_mgs_pass semantics) equals the single-domain
    run with the same GMRES iteration count."""
    op, U, _, _, _ = _problem()
    ref = integrate(op, U, 0.0, 2 * DT, DT, order=3, newton_kwargs=NEWTON)
    Uref = ref.U.numpy()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(nranks, _free_port(), out), nprocs=nranks,
                       start_method="spawn")
    covered = np.zeros(len(Uref), dtype=int)
    for r in range(nranks):
        gids, Ur, iters, nrm = out[r]
        covered[gids] += 1
        scale = np.abs(Uref).max()
        assert np.abs(Ur - Uref[gids]).max() <= 1e-10 * scale
        assert iters == ref.gmres_iterations
        assert nrm == pytest.approx(float(np.linalg.norm(Uref)), rel=1e-13)
    assert np.all(covered == 1)
    assert ref.U.shape == U.shape and not np.allclose(Uref, U.numpy())
