"""FP64 throughput probes on the GPU: DFMA (SIMT) vs DMMA (mma.sync m8n8k4 f64)."""
import ctypes, torch, sys
sys.path.insert(0, '.')
from paper_1403_1157_b200 import _native
lib = _native.load()
n = lib.tdg_fp64_probe_threads()
out = torch.empty(n, dtype=torch.float64, device='cuda')
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for name, fn, per in (("dfma", lib.tdg_fp64_probe, lambda it: n*16*2*it), ("dmma", lib.tdg_dmma_probe, lambda it: n/32*it*4*512)):
    it = 20000
    for _ in range(2): fn(out.data_ptr(), it, st)
    best = 0
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(out.data_ptr(), it, st); b.record(); b.synchronize()
        best = max(best, per(it) / (a.elapsed_time(b)*1e-3) / 1e12)
    print(name, f"{best:.2f} TFLOP/s")
