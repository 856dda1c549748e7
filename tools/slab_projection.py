"""One rank's share of an N-way strong-scaling run of C5, timed on ONE GPU.

Builds rank R's x-slab of the fixed C5 mesh split N ways (owned rows + one
ghost cell column per side, decomp.build_slab), and steps it with the slab
stepper (stepping.SSPRK3: part 1 = faces on owned rows, exchange, part 2 =
cut faces + volume kernel).  The exchange is replaced by a LOCAL stand-in of
the same shape: the boundary rows are packed as in HaloExchange.start and
copied into the ghost rows on a side stream (device-to-device, so the copy
runs at HBM speed, not NVLink speed; no second GPU, no kernel waits on
another rank).  What this measures: the per-rank kernel time of the N-way
split (smaller launches, the extra cut-face segments, the ghost columns) and
the pack cost.  What it does not: NVLink transfer time and NCCL launch
latency -- printed as a bytes / 900 GB/s estimate beside the overlap window.

usage: python tools/slab_projection.py [N] [rank] [steps]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_problem  # noqa: E402
from paper_1403_1157_b200.operator import DiscreteOperator  # noqa: E402
from paper_1403_1157_b200.stepping import SSPRK3  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
R = int(sys.argv[2]) if len(sys.argv) > 2 else N // 2
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
cfg_name = os.environ.get("TDG_CONFIG", "c5")
dev = torch.device("cuda", 0)


class LocalHalo:
    """Same packing and ghost-row writes as decomp.HaloExchange, the transfer
    replaced by a device-to-device copy on a side stream."""

    def __init__(self, slab, device):
        self.slab = slab
        self.idx_l = torch.as_tensor(slab.send_left, device=device)
        self.idx_r = torch.as_tensor(slab.send_right, device=device)
        self.side = torch.cuda.Stream(device=device)
        self.bytes = 0

    def start(self, U):
        s = self.slab
        self.side.wait_stream(torch.cuda.current_stream())
        self.bytes = 0
        with torch.cuda.stream(self.side):
            for nb, idx, rsl in ((s.rank - 1, self.idx_l, s.recv_left),
                                 (s.rank + 1, self.idx_r, s.recv_right)):
                if nb < 0 or nb >= s.nranks:
                    continue
                buf = U.index_select(0, idx)          # the pack kernel
                rv = U[rsl]
                n = min(len(buf), len(rv))
                rv[:n].copy_(buf[:n])                 # stands in for isend / irecv
                self.bytes += 2 * buf.numel() * 8     # sent + received

    def wait(self):
        torch.cuda.current_stream().wait_stream(self.side)

    def exchange(self, U):
        self.start(U)
        self.wait()


t0 = time.time()
cfg, space, model, scheme, U, slab = build_problem(cfg_name, "cdg2", R, N, "strong", True, dev)
op = DiscreteOperator(space, model, scheme, device=dev, n_owned=slab.n_owned,
                      global_ids=slab.global_ids)
halo = LocalHalo(slab, dev)
stepper = SSPRK3(op, halo)
halo.exchange(U)
dt = float(os.environ.get("TDG_DT", "2.2366e-06"))
for _ in range(3):
    stepper.step(U, dt)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(steps):
    stepper.step(U, dt)
b.record()
b.synchronize()
ms = a.elapsed_time(b) / steps
# part 1 alone (the window the exchange overlaps with), one stage
W = torch.empty_like(U)
torch.cuda.synchronize()
a.record()
for _ in range(steps):
    op.rk_stage_part(None, U, W, 0.0, 1.0, dt, 1)
b.record()
b.synchronize()
p1 = a.elapsed_time(b) / steps
n_dofs = slab.n_owned * 6 * space.nb
print(json.dumps({
    "what": f"rank {R} of {N}: one-GPU timing of its x-slab of {cfg_name} (local stand-in for "
            "the exchange)",
    "owned_elements": int(slab.n_owned), "ghost_elements": int(space.mesh.n_elements - slab.n_owned),
    "colour_segments": int(op.tables.n_seg), "cut_segments": int(op.tables.n_seg_cut),
    "ms_per_step": ms, "dof_updates_per_s_rank": n_dofs * 3 / (ms * 1e-3),
    "projected_job_dof_updates_per_s": N * n_dofs * 3 / (ms * 1e-3),
    "exchange_bytes_per_stage": halo.bytes,
    "nvlink_ms_per_stage_at_900GBs_per_direction": halo.bytes / 2 / 900e9 * 1e3,
    "overlap_window_ms_per_stage (part 1: owned-row faces)": p1,
    "setup_s": time.time() - t0,
    "finite": bool(torch.isfinite(U[:slab.n_owned]).all().item()),
}))
