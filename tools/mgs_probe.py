"""Time one tdg_mgs sweep (GMRES Arnoldi step) at C2 / C3 vector sizes.

usage: python tools/mgs_probe.py [n] > gpurun_out/mgs.json
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1403_1157_b200 import DGSpace, FluxScheme, PlaqueModel, unit_square  # noqa: E402
from paper_1403_1157_b200.operator import DiscreteOperator  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4718592
if len(sys.argv) > 2 and sys.argv[2] == "persist":
    # set aside the device's maximum persisting-L2 size (evict-last lines)
    import ctypes
    import glob
    torch.cuda.init()
    libs = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*")) + \
        glob.glob("/usr/local/cuda/lib64/libcudart.so*")
    rt = ctypes.CDLL(libs[0])
    mx = ctypes.c_int()
    rt.cudaDeviceGetAttribute(ctypes.byref(mx), 108, 0)  # cudaDevAttrMaxPersistingL2CacheSize
    rc = rt.cudaDeviceSetLimit(6, ctypes.c_size_t(mx.value))  # cudaLimitPersistingL2CacheSize
    print(json.dumps({"persist_max": mx.value, "rc": rc}), file=sys.stderr)
m = 31
dev = torch.device("cuda:0")
op = DiscreteOperator(DGSpace(unit_square(4), 1, 6), PlaqueModel(), FluxScheme("cdg2"), device=dev)
g = torch.Generator(device=dev).manual_seed(5)
V = torch.randn((m, n), dtype=torch.float64, device=dev, generator=g)
V /= torch.linalg.norm(V, dim=1, keepdim=True)
w0 = torch.randn(n, dtype=torch.float64, device=dev, generator=g)
w = w0.clone()
h = torch.zeros(m + 2, dtype=torch.float64, device=dev)
res = {"n": n}
for j in (0, 4, 14, 29):
    for _ in range(3):
        w.copy_(w0)
        op.mgs(V, j, w, h)
    ts = []
    for _ in range(10):
        w.copy_(w0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        op.mgs(V, j, w, h)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    res[f"j{j}"] = {"ms": ms, "us_per_pass": ms * 1e3 / (j + 2),
                    "hbm_min_GBps": (j + 1) * n * 8 / (ms * 1e-3) / 1e9}
print(json.dumps(res))
