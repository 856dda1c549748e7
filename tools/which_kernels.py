"""One 3D application (unit_cube(n), p=k) for kernel-name / timing checks under ncu.
usage: python tools/which_kernels.py [n] [k] [variant]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1403_1157_b200 import DGSpace, FluxScheme, PlaqueModel  # noqa: E402
from paper_1403_1157_b200.mesh import unit_cube  # noqa: E402
from paper_1403_1157_b200.operator import DiscreteOperator  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
k = int(sys.argv[2]) if len(sys.argv) > 2 else 2
var = int(sys.argv[3]) if len(sys.argv) > 3 else 0
space = DGSpace(unit_cube(n), k, 6)
op = DiscreteOperator(space, PlaqueModel(), FluxScheme("cdg2"))
if var:
    op.lib.tdg_set_variant(op._ctx, var)
U = torch.from_numpy(np.random.default_rng(0).random((space.mesh.n_elements, 6, space.nb))).cuda()
for _ in range(3):
    R = op.apply_f(U)
torch.cuda.synchronize()
print("ok", float(R.abs().sum()))
