"""x-slab domain decomposition for multi-GPU runs (one process per GPU).

SURVEY.md 8(e): the structured configs number cells with x fastest, so
an x-slab owns a strided set of global elements.  Each rank builds only
its slab plus one ghost cell column on each side (``mesh._square_parts``
/ ``_cube_parts`` with the global grid's coordinates, so geometry and the
K- volume ties are bit-identical to the global mesh), numbers its owned
elements first and its ghosts after them, and per operator application
exchanges the ghost elements' coefficient rows with its x-neighbours
(NCCL point-to-point on GPUs, gloo in the CPU tests).  Ghost rows are
laid out in exactly the order the neighbour packs them, so a receive
lands in a contiguous slice of U with no unpack step.

Faces between an owned element and a ghost are evaluated by both ranks,
each writing only its own side; the K- rule uses global element ids, so
both ranks take the same lifting side.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .configs import Config
from .mesh import Mesh, _cube_parts, _square_parts

__all__ = ["Slab", "slab_ranges", "build_slab", "HaloExchange"]


def slab_ranges(nx: int, nranks: int):
    """Balanced contiguous cell-column ranges [i0, i1) per rank."""
    if nranks < 1 or nranks > nx:
        raise ValueError("need 1 <= nranks <= nx")
    cuts = [nx * r // nranks for r in range(nranks + 1)]
    return [(cuts[r], cuts[r + 1]) for r in range(nranks)]


@dataclass
class Slab:
    rank: int
    nranks: int
    cells_x: tuple            # owned cell columns [i0, i1)
    mesh: Mesh                # owned elements first, then ghosts
    n_owned: int
    global_ids: np.ndarray    # global element id of every local element
    send_left: np.ndarray     # local rows sent to rank-1 (its right ghosts)
    send_right: np.ndarray    # local rows sent to rank+1 (its left ghosts)
    recv_left: slice          # ghost rows received from rank-1
    recv_right: slice         # ghost rows received from rank+1

    @property
    def n_ghost(self) -> int:
        return self.mesh.n_elements - self.n_owned


def _column_order(col, gids):
    """Element order of one cell column: by global id (x fastest in the
    global numbering, so this is (k, j, tet) order inside a column)."""
    return np.argsort(gids[col], kind="stable")


def build_slab(cfg: Config, rank: int, nranks: int, cells=None,
               seed: int = 0) -> Slab:
    cells = tuple(cells or cfg.cells)
    nx = cells[0]
    i0, i1 = slab_ranges(nx, nranks)[rank]
    g0, g1 = max(i0 - 1, 0), min(i1 + 1, nx)
    if cfg.dim == 2:
        verts, elems, gids, tag_fn = _square_parts(
            nx, cells[1], (0.25, 0.75), cfg.lengths, cfg.jitter, seed, (g0, g1))
        per_cell = 2
        cell_x = (gids // 2) % nx
    else:
        gamma1_in = None if cfg.tags == "z0_gamma1" else (0.25, 0.75, 0.25, 0.75)
        from .mesh import BoundaryTag
        top = BoundaryTag.NO_FLOW if cfg.tags == "z0_gamma1" else BoundaryTag.GAMMA2
        verts, elems, gids, tag_fn = _cube_parts(
            nx, cells[1], cells[2], gamma1_in, top, cfg.lengths, (g0, g1))
        per_cell = 6
        cell_x = (gids // 6) % nx
    owned = (cell_x >= i0) & (cell_x < i1)
    left = cell_x == i0 - 1
    right = cell_x == i1
    own_idx = np.flatnonzero(owned)
    left_idx = np.flatnonzero(left)[_column_order(np.flatnonzero(left), gids)]
    right_idx = np.flatnonzero(right)[_column_order(np.flatnonzero(right), gids)]
    order = np.concatenate([own_idx, left_idx, right_idx])
    mesh = Mesh(verts, elems[order], tag_fn=tag_fn)
    gl = gids[order]
    n_own = len(own_idx)
    # rows this rank sends: its first / last owned cell column, packed in
    # the same (global id) order the neighbour stores its ghosts in
    own_x = cell_x[own_idx]
    first = np.flatnonzero(own_x == i0)
    last = np.flatnonzero(own_x == i1 - 1)
    send_left = first[np.argsort(gl[first], kind="stable")] if rank > 0 else np.zeros(0, np.int64)
    send_right = last[np.argsort(gl[last], kind="stable")] if rank < nranks - 1 else np.zeros(0, np.int64)
    nl, nr = len(left_idx), len(right_idx)
    del per_cell
    return Slab(rank, nranks, (i0, i1), mesh, n_own, gl,
                send_left.astype(np.int64), send_right.astype(np.int64),
                slice(n_own, n_own + nl), slice(n_own + nl, n_own + nl + nr))


class HaloExchange:
    """Ghost-row exchange with the x-neighbours through torch.distributed
    point-to-point ops.  ``start`` packs the two boundary columns and
    posts the sends/receives; ``wait`` makes the caller's stream (NCCL) or
    thread (gloo) wait until the ghost rows of U are filled.

    With NCCL the device rows travel directly (GPU to GPU).  With gloo
    (CPU tests, and several ranks sharing one GPU in the one-GPU slab
    tests) device tensors are staged through host buffers: gloo cannot
    address device memory, and no device kernel ever waits on another
    rank -- the host does."""

    def __init__(self, slab: Slab, device=None):
        import torch
        self.slab = slab
        self.dev = device
        self.idx_l = torch.as_tensor(slab.send_left, device=device)
        self.idx_r = torch.as_tensor(slab.send_right, device=device)
        self._works = []
        self._recv = []

    def _staged(self, U):
        import torch.distributed as dist
        return U.is_cuda and dist.get_backend() == "gloo"

    def start(self, U):
        import torch.distributed as dist
        s = self.slab
        ops = []
        self._bufs = []
        self._recv = []
        staged = self._staged(U)
        for nb, idx, rsl in ((s.rank - 1, self.idx_l, s.recv_left),
                             (s.rank + 1, self.idx_r, s.recv_right)):
            if nb < 0 or nb >= s.nranks:
                continue
            buf = U.index_select(0, idx)
            rv = U[rsl]
            if staged:
                buf = buf.cpu()
                host_rv = rv.new_empty(rv.shape, device="cpu")
                self._recv.append((rv, host_rv))
                rv = host_rv
            self._bufs.append(buf)
            ops.append(dist.P2POp(dist.isend, buf, nb))
            ops.append(dist.P2POp(dist.irecv, rv, nb))
        try:
            self._works = dist.batch_isend_irecv(ops) if ops else []
        except Exception as err:  # noqa: BLE001 -- re-raised with the slab attached
            raise RuntimeError(f"ghost exchange post failed on rank {s.rank}/{s.nranks} "
                               f"(neighbours {s.rank - 1}, {s.rank + 1}, backend "
                               f"{dist.get_backend()}): {err}") from err

    def wait(self):
        for w in self._works:
            try:
                w.wait()
            except Exception as err:  # noqa: BLE001 -- re-raised with the slab attached
                s = self.slab
                raise RuntimeError(f"ghost exchange failed on rank {s.rank}/{s.nranks}: "
                                   f"{err}") from err
        for dev_rows, host_rows in self._recv:
            dev_rows.copy_(host_rows)
        self._works = []
        self._bufs = []
        self._recv = []

    def exchange(self, U):
        self.start(U)
        self.wait()
