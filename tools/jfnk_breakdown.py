"""Where the time of one GMRES(30) cycle goes at C2 (device): matvec
(Jacobian-free G evaluations), the fused MGS sweep, and the host round
trip per Arnoldi step.  Prints ms per Arnoldi step for each part."""
import time

import numpy as np
import torch

from paper_1403_1157_b200.configs import CONFIGS, make_mesh
from paper_1403_1157_b200 import DGSpace, FluxScheme, PlaqueModel
from paper_1403_1157_b200.fields import initial_state
from paper_1403_1157_b200.operator import DiscreteOperator

cfg = CONFIGS["c2"]
space = DGSpace(make_mesh(cfg), cfg.order, 6)
op = DiscreteOperator(space, PlaqueModel(), FluxScheme("cdg2"))
U = torch.from_numpy(initial_state(space, 1)).cuda()
n = U.numel()
m = 30
V = torch.randn(m + 1, n, dtype=torch.float64, device="cuda")
V /= V.norm(dim=1, keepdim=True)
h = torch.zeros(m + 2, dtype=torch.float64, device="cuda")
r = torch.empty_like(U)
dt, aii = 0.01, 0.4358665215


def G(v):
    op.rk_stage(U, v.reshape(U.shape), r, -1.0, 1.0, -dt * aii)
    return r


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def matvecs():
    for j in range(m):
        G(V[j])


def mgs_all():
    for j in range(m):
        w = V[m].clone()
        op.mgs(V, j, w, h)


def mgs_sync():
    for j in range(m):
        w = V[m].clone()
        op.mgs(V, j, w, h)
        h[:j + 2].cpu()


def full():
    for j in range(m):
        w = G(V[j]).reshape(-1).clone()
        op.mgs(V, j, w, h)
        hv = h[:j + 2].cpu().numpy()
        torch.mul(w, 1.0 / max(hv[j + 1], 1e-300), out=V[m])


for name, fn in [("matvec (G only)", matvecs), ("fused MGS", mgs_all),
                 ("fused MGS + host sync", mgs_sync), ("Arnoldi step", full)]:
    print(f"{name:24s} {timeit(fn) / m:8.3f} ms per Arnoldi step")
