"""Run diagnostics from device buffers.

The reference writes, per run, ``balance.csv`` (species totals per step,
``scenarios.py:235-239``) and legacy-ASCII VTK snapshots of cell means and
vertex averages (``vtkio.py:26-77``), both from host arrays
(``DiscreteFunction.species_totals / cell_means / vertex_values``,
``fespace.py:150-174``).  Here the reductions run on the device -- species
totals through the library's deterministic ``tdg_species_totals``, cell
means and vertex averages as device gathers / scatter-adds -- and only the
small results cross to the host, in the reference's file formats:

* ``BalanceRecorder``: a step callback (``integrate(..., callback=...)``
  or any stepping loop) that keeps one row of totals per step on the
  device and writes ``balance.csv`` at the end (header ``time,
  total_<species>``, time ``%.10g``, totals ``%.16e``);
* ``write_vtk``: one snapshot (``# vtk DataFile Version 3.0``, POINTS,
  CELLS, CELL_TYPES 5 / 10, CELL_DATA per species, POINT_DATA
  ``<species>_vertex``; values ``%.10g``).
"""

from __future__ import annotations

import csv

import numpy as np

from .mesh import REF_VERTICES

__all__ = ["BalanceRecorder", "device_cell_means", "device_vertex_values", "write_vtk"]

_CELL_TYPE = {2: 5, 3: 10}
_REF_MEASURE = {2: 0.5, 3: 1.0 / 6.0}


def _torch():
    import torch
    return torch


def _as_device(op, U):
    torch = _torch()
    if isinstance(U, torch.Tensor):
        return U[:op.n_owned]
    U = np.asarray(getattr(U, "coeffs", U), dtype=float)
    return torch.from_numpy(np.ascontiguousarray(U[:op.n_owned])).to(op.device)


def device_cell_means(op, U):
    """(ne, S) element averages on the device (reference
    ``DiscreteFunction.cell_means``, ``fespace.py:150-153``)."""
    Ud = _as_device(op, U)
    return Ud[:, :, 0] / np.sqrt(_REF_MEASURE[op.mesh.dim])


def device_vertex_values(op, U):
    """(nv, S) vertex averages over the incident elements on the device
    (reference ``DiscreteFunction.vertex_values``, ``fespace.py:155-168``)."""
    torch = _torch()
    Ud = _as_device(op, U)
    mesh = op.mesh
    d = mesh.dim
    basis = getattr(op.space, "basis")
    phi = torch.as_tensor(basis.eval(REF_VERTICES[d]), dtype=Ud.dtype, device=Ud.device)
    vals = torch.einsum("esi,ci->ecs", Ud, phi)                  # (ne, d+1, S)
    elems = torch.as_tensor(np.asarray(mesh.elements[:op.n_owned]), device=Ud.device)
    nv = len(mesh.vertices)
    out = torch.zeros((nv, Ud.shape[1]), dtype=Ud.dtype, device=Ud.device)
    count = torch.zeros(nv, dtype=Ud.dtype, device=Ud.device)
    ones = torch.ones(elems.shape[0], dtype=Ud.dtype, device=Ud.device)
    for c in range(d + 1):
        out.index_add_(0, elems[:, c], vals[:, c, :])
        count.index_add_(0, elems[:, c], ones)
    return out / count.clamp(min=1.0)[:, None]


class BalanceRecorder:
    """Species totals per step, kept on the device; ``write_csv`` emits the
    reference's ``balance.csv``.  Usable directly as the ``callback`` of
    ``timeint.integrate`` (numpy or device states)."""

    def __init__(self, op, names=None, capacity: int = 1024):
        torch = _torch()
        self.op = op
        S = op.space.n_species
        self.names = list(names) if names is not None else list(
            getattr(op.model, "species", [f"f{s}" for s in range(S)]))
        self._rows = torch.empty((capacity, S), dtype=torch.float64, device=op.device)
        self._times = []

    def record(self, t: float, U):
        torch = _torch()
        k = len(self._times)
        if k == self._rows.shape[0]:
            self._rows = torch.cat([self._rows, torch.empty_like(self._rows)])
        Ud = U if isinstance(U, torch.Tensor) else _as_device(self.op, U).contiguous()
        self.op.species_totals(Ud, out=self._rows[k])
        self._times.append(float(t))

    def __call__(self, step, t, U):
        self.record(t, U)

    def totals(self) -> np.ndarray:
        return self._rows[:len(self._times)].cpu().numpy()

    def write_csv(self, path):
        totals = self.totals()
        with open(path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["time"] + [f"total_{s}" for s in self.names])
            for t, row in zip(self._times, totals):
                w.writerow([f"{t:.10g}"] + [f"{v:.16e}" for v in row])
        return path


def _data_name(name: str) -> str:
    return "".join(ch if ch.isalnum() or ch in "_-" else "_" for ch in name) or "field"


def write_vtk(path, op, U, names=None, title: str = "taxisdg snapshot"):
    """One legacy-ASCII VTK snapshot of a state (device tensor or host
    array), cell means and vertex averages reduced on the device (format
    of reference ``vtkio.write_vtk``, ``vtkio.py:26-77``)."""
    S = op.space.n_species
    if names is None:
        names = [f"f{s}" for s in range(S)]
    if len(names) != S:
        raise ValueError(f"{len(names)} names for {S} species")
    names = [_data_name(n) for n in names]
    cell = device_cell_means(op, U).cpu().numpy()
    point = device_vertex_values(op, U).cpu().numpy()
    if not (np.isfinite(cell).all() and np.isfinite(point).all()):
        raise ValueError("refusing to write non-finite field data")
    mesh = op.mesh
    verts = np.asarray(mesh.vertices)
    if mesh.dim == 2:
        verts = np.column_stack([verts, np.zeros(len(verts))])
    elems = np.asarray(mesh.elements)[:op.n_owned]
    npe = elems.shape[1]
    lines = ["# vtk DataFile Version 3.0", title[:255], "ASCII", "DATASET UNSTRUCTURED_GRID",
             f"POINTS {len(verts)} double"]
    lines += [" ".join(f"{c:.10g}" for c in v) for v in verts]
    lines.append(f"CELLS {len(elems)} {len(elems) * (npe + 1)}")
    lines += [f"{npe} " + " ".join(map(str, e)) for e in elems]
    lines.append(f"CELL_TYPES {len(elems)}")
    lines += [str(_CELL_TYPE[mesh.dim])] * len(elems)
    lines.append(f"CELL_DATA {len(elems)}")
    for s, name in enumerate(names):
        lines += [f"SCALARS {name} double 1", "LOOKUP_TABLE default"]
        lines += [f"{v:.10g}" for v in cell[:, s]]
    lines.append(f"POINT_DATA {len(verts)}")
    for s, name in enumerate(names):
        lines += [f"SCALARS {name}_vertex double 1", "LOOKUP_TABLE default"]
        lines += [f"{v:.10g}" for v in point[:, s]]
    with open(path, "w") as fh:
        fh.write("\n".join(lines))
        fh.write("\n")
    return path
