"""Diagnostics from device buffers against the
reference's own outputs: the VTK snapshot of reference vtkio.write_vtk
(vtkio.py:26-77) and DiscreteFunction.species_totals (fespace.py:170-174),
and the balance.csv layout of scenarios.py:235-239."""
import csv
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_1403_1157_b200 import DGSpace, FluxScheme, PlaqueModel, unit_cube, unit_square  # noqa: E402

pytestmark = pytest.mark.gpu
NAMES = ["n1", "n2", "n3", "c1", "c2", "c3"]


def _op(space):
    from paper_1403_1157_b200.operator import DiscreteOperator
    return DiscreteOperator(space, PlaqueModel(), FluxScheme("cdg2"))


def _parse(text):
    """Section name -> list of numbers (and the non-numeric header lines)."""
    out, key = {}, None
    for ln in text.strip().split("\n"):
        head = ln.split()[0] if ln.split() else ""
        if head in ("POINTS", "CELLS", "CELL_TYPES", "CELL_DATA", "POINT_DATA", "SCALARS"):
            key = ln
            out[key] = []
            continue
        if key is None or head == "LOOKUP_TABLE":
            out.setdefault("header", []).append(ln)
            continue
        out[key].extend(float(x) for x in ln.split())
    return out


@pytest.mark.parametrize("key,mesh,k", [("sq3", lambda: unit_square(3), 2),
                                        ("cube1", lambda: unit_cube(1), 1)])
def test_vtk_from_device_buffers_matches_reference_writer(golden, tmp_path, key, mesh, k):
    from paper_1403_1157_b200.diagnostics import write_vtk
    g = golden["diagnostics"]
    space = DGSpace(mesh(), k, 6)
    op = _op(space)
    U = torch.from_numpy(g[f"{key}__U"]).cuda()
    path = write_vtk(os.path.join(tmp_path, "s.vtk"), op, U, names=NAMES)
    got, ref = _parse(open(path).read()), _parse(str(g[f"{key}__vtk"]))
    assert got.keys() == ref.keys()
    for sec in ref:
        if sec == "header":
            assert got[sec] == ref[sec]
        else:
            assert np.allclose(got[sec], ref[sec], rtol=1e-9, atol=1e-12), sec


def test_balance_csv_from_device_totals(golden, tmp_path):
    from paper_1403_1157_b200.diagnostics import BalanceRecorder
    from paper_1403_1157_b200.timeint import integrate
    g = golden["diagnostics"]
    space = DGSpace(unit_square(3), 2, 6)
    op = _op(space)
    rec = BalanceRecorder(op, capacity=2)
    rec.record(0.0, g["sq3__U"])
    assert np.allclose(rec.totals()[0], g["sq3__totals"], rtol=1e-13, atol=1e-15)
    res = integrate(op, g["sq3__U"], 0.0, 1.0, 0.01, order=3, n_steps=3, callback=rec)
    path = rec.write_csv(os.path.join(tmp_path, "balance.csv"))
    rows = list(csv.reader(open(path)))
    assert rows[0] == ["time"] + [f"total_{s}" for s in NAMES]
    assert len(rows) == 5 and float(rows[-1][0]) == pytest.approx(0.03)
    last = np.array([float(x) for x in rows[-1][1:]])
    assert np.allclose(last, space.function(res.U).species_totals(), rtol=1e-13, atol=1e-15)
