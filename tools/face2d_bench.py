"""A/B of the 2D face kernels (k_faces_sig vs k_faces_fast): ms per
application per kernel class and the difference between the two kernels at
size (parity against the oracle: tests/test_gpu_operator.py).
usage: python tools/face2d_bench.py [nx ny] [k] [reps] [jitter]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1403_1157_b200 import (DGSpace, FluxScheme, PlaqueModel, PlaqueParams,  # noqa: E402
                                  unit_square)
from paper_1403_1157_b200.operator import DiscreteOperator  # noqa: E402
from paper_1403_1157_b200.roofline import apply_flops  # noqa: E402

a = sys.argv[1:]
nx, ny = (int(a[0]), int(a[1])) if len(a) >= 2 else (512, 128)
k = int(a[2]) if len(a) > 2 else 2
reps = int(a[3]) if len(a) > 3 else 20
jit = float(a[4]) if len(a) > 4 else 0.0
model = PlaqueModel(PlaqueParams(chi11_a=1.0, chi13_a=0.6, chi21_a=0.8, chi2n_a=0.7,
                                 c1_star=0.12, c1_starstar=0.13))


def mesh(nx, ny):
    kw = dict(lengths=(4.0, 1.0))
    if jit:
        kw.update(jitter=jit, seed=3)
    return unit_square(nx, ny, **kw)


space = DGSpace(mesh(nx, ny), k, 6)
op = DiscreteOperator(space, model, FluxScheme("cdg2"))
t = op.tables
rng = np.random.default_rng(0)
U = torch.from_numpy(0.1 + 0.01 * rng.random((space.mesh.n_elements, 6, space.nb))).cuda()
out = torch.empty_like(U)
res = {}
cps = int(os.environ.get("TDG_FACE_CTAS", "0"))
for name, kw in (("sig", {"face_ctas_per_sm": cps}), ("fast", {"no_sig": True})):
    op.set_variant(**kw)
    for _ in range(3):
        op.rk_stage(U, U, out, 0.5, 0.5, 1e-6)
    torch.cuda.synchronize()
    op.profile(True)
    for _ in range(reps):
        op.rk_stage(U, U, out, 0.5, 0.5, 1e-6)
    torch.cuda.synchronize()
    op.profile(False)
    kt = op.profile_read()
    res[name] = out.clone()
    fv, ff, fb = apply_flops(2, t.nb, t.nq_vol, t.nq_face, op.n_owned, len(t.if_code), len(t.bf_code))
    for kn, fl in (("faces", ff), ("wall", fb), ("volume", fv)):
        ms, n = kt[kn]
        if n:
            print(f"{name:5s} {kn:7s} {ms / reps * 1e3:9.1f} us/app  {fl / (ms / reps * 1e-3) / 1e12:6.2f} "
                  f"TF/s alg  ({n // reps} launches/app)")
d = (res["sig"] - res["fast"]).abs().max().item() / res["fast"].abs().max().item()
print(f"elements {op.n_owned}, faces {len(t.if_code)}, segments {t.n_seg}; sig vs fast rel {d:.2e}")
