"""Per-kernel timing of one 3D configuration (A/B of kernel changes).
usage: python tools/face_bench.py [nx ny nz] [k] [reps] [variant]
Prints ms per application and algorithmic TFLOP/s per kernel class."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1403_1157_b200 import DGSpace, FluxScheme, PlaqueModel  # noqa: E402
from paper_1403_1157_b200.mesh import unit_cube  # noqa: E402
from paper_1403_1157_b200.operator import DiscreteOperator  # noqa: E402
from paper_1403_1157_b200.roofline import apply_flops  # noqa: E402

a = [int(x) for x in sys.argv[1:]]
nx, ny, nz = (a + [48, 48, 48])[:3] if len(a) >= 3 else (48, 48, 48)
k = a[3] if len(a) > 3 else 3
reps = a[4] if len(a) > 4 else 5
var = a[5] if len(a) > 5 else 0
space = DGSpace(unit_cube(nx, ny, nz, lengths=(2.0 * nx / 256, ny / 128, nz / 128)), k, 6)
op = DiscreteOperator(space, PlaqueModel(), FluxScheme("cdg2"))
if var:
    op.lib.tdg_set_variant(op._ctx, var)
t = op.tables
rng = np.random.default_rng(0)
U = torch.from_numpy(0.1 + 0.01 * rng.random((space.mesh.n_elements, 6, space.nb))).cuda()
out = torch.empty_like(U)
for _ in range(3):
    op.rk_stage(U, U, out, 0.5, 0.5, 1e-6)
torch.cuda.synchronize()
op.profile(True)
for _ in range(reps):
    op.rk_stage(U, U, out, 0.5, 0.5, 1e-6)
torch.cuda.synchronize()
op.profile(False)
kt = op.profile_read()
fv, ff, fb = apply_flops(3, t.nb, t.nq_vol, t.nq_face, op.n_owned, len(t.if_code), len(t.bf_code))
for name, fl in (("faces", ff), ("wall", fb), ("volume", fv)):
    ms, n = kt[name]
    if n:
        print(f"{name:7s} {ms / reps:9.3f} ms/app  {fl / (ms / reps * 1e-3) / 1e12:6.2f} TF/s alg  "
              f"({n // reps} launches/app)")
print(f"elements {op.n_owned}, faces {len(t.if_code)}, segments {t.n_seg}")
