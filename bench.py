#!/usr/bin/env python
"""Benchmark: fp64 DG-operator DoF-updates/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2]
                    [--impl native|reference]

A step is one Shu-Osher SSP-RK3 step = 3 applications of f = M^-1 L_h,
each fused with its Runge-Kutta stage update, over the whole mesh.
Unit of work: one DoF receiving one f evaluation, so
value = n_dofs * 3 * K / (device time of K steps), max over ranks.

Default workload: config C2 (BASELINE configs[1], 4.7M DoFs, p=2 2D) at
the explicit CFL step dt = 0.8 * 2.51 / rho(J), rho by device power
iteration.  Inputs are resident in HBM; L2 (126 MB) is flushed between
timed steps by writing a 256 MiB buffer outside the timed events.

``--impl reference`` times the CPU oracle port of the reference
(oracle/, numpy, all host threads) on the same config: the reference
itself is pure Python and cannot travel to the GPU box.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 DG-operator DoF-updates/s at 1/2/4/8 B200; % of HBM/FP64 roofline"
UNIT = "DoF-updates/s"
FP64_NOMINAL_TFLOPS = 37.0  # HGX B200 datasheet FP64 / FP64 tensor


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--scheme", default="cdg2")
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: testing only (host-staged exchange; ranks may share a GPU)")
    ap.add_argument("--bands", type=int, default=8,
                    help="element bands of the host-pipelined e2e stepping")
    ap.add_argument("--no-implicit", action="store_true",
                    help="skip the extra SDIRK3+JFNK figure of the explicit C2 run")
    ap.add_argument("--power-iters", type=int, default=200)
    ap.add_argument("--integrator", default="ssprk3", choices=["ssprk3", "sdirk3"],
                    help="sdirk3: the reference's default SDIRK3 + JFNK at --dt")
    ap.add_argument("--dt", type=float, default=0.01)
    ap.add_argument("--force-slab", action="store_true",
                    help="use the slab/halo code path even at N=1 (testing)")
    ap.add_argument("--variant", type=int, default=0,
                    help="kernel variant bits (tdg_set_variant), for A/B timing")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self._t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self._t is not None:
            self._t.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": smax, "samples": len(sm),
                "reasons": sorted(reasons)}


# -------------------------------------------------------------- workload

def weak_config(cfg, world):
    """Weak scaling: every rank owns one x-slab of cfg.cells[0] /
    cfg.weak_div cell columns (same cell size) of a domain N times that
    long in x -- C2 at N GPUs is N side-by-side C2 domains; C5 (weak_div
    8) at N = 8 is exactly C5."""
    import dataclasses
    if world == 1 and cfg.weak_div == 1:
        return cfg
    cx = cfg.cells[0] // cfg.weak_div
    lx = cfg.lengths[0] / cfg.weak_div
    cells = (cx * world,) + tuple(cfg.cells[1:])
    lengths = (lx * world,) + tuple(cfg.lengths[1:])
    desc = cfg.description
    if cfg.weak_div > 1:
        desc += f" -- weak unit {cx}x" + "x".join(map(str, cfg.cells[1:])) + \
            f" cells per GPU ({world}/{cfg.weak_div} of the config)"
    return dataclasses.replace(cfg, cells=cells, lengths=lengths, description=desc)


def sample_config(cfg, max_dofs=5_000_000):
    """The CPU baseline's bounded sample: an x-slab of the config with the
    same cell size, order and physics, cut to about ``max_dofs`` DoFs (the
    config itself when it is smaller)."""
    import dataclasses
    from paper_1403_1157_b200.basis import basis_size
    per_cell = (2 if cfg.dim == 2 else 6) * 6 * basis_size(cfg.dim, cfg.order)
    cells, lengths = list(cfg.cells), list(cfg.lengths)
    for ax in range(cfg.dim - 1):       # shrink x first, then y (3D), same cell size
        rest = int(np.prod(cells)) // cells[ax]
        c = max(1, min(cells[ax], max_dofs // (per_cell * rest)))
        lengths[ax] *= c / cells[ax]
        cells[ax] = c
    if tuple(cells) == tuple(cfg.cells):
        return cfg
    return dataclasses.replace(cfg, cells=tuple(cells), lengths=tuple(lengths))


def build_problem(cfg_name, scheme_name, rank=0, world=1, force_slab=False, device=None,
                  cpu_sample=False):
    """(cfg, space, model, scheme, U0, slab); the slab is None at N=1
    unless ``force_slab``; ``cpu_sample``: the CPU baseline's bounded
    x-slab of the config (sample_config)."""
    from paper_1403_1157_b200 import DGSpace, FluxScheme, PlaqueModel
    from paper_1403_1157_b200.configs import CONFIGS, make_mesh
    from paper_1403_1157_b200.decomp import build_slab
    from paper_1403_1157_b200.fields import bump_field
    cfg = weak_config(CONFIGS[cfg_name], world)
    if cpu_sample:
        cfg = sample_config(cfg)
    slab = None
    if world == 1 and not force_slab:
        mesh = make_mesh(cfg)
    else:
        slab = build_slab(cfg, rank, world)
        mesh = slab.mesh
    space = DGSpace(mesh, cfg.order, 6)
    lo = np.zeros(cfg.dim)
    hi = np.asarray(cfg.lengths, dtype=float)
    fn = bump_field(cfg.dim, 6, 1, lo, hi)
    if device is not None and (cfg.dim == 3 or mesh.n_elements > 500_000):
        # host projection is slow at scale (~0.4 ms/tet at 3D p=3): on the GPU
        from paper_1403_1157_b200.fields import project_bumps_device
        U0 = project_bumps_device(space, fn, device).cpu().numpy()
    else:
        U0 = np.ascontiguousarray(space.project(fn).coeffs)
    return cfg, space, PlaqueModel(), FluxScheme(scheme_name), U0, slab


def spectral_radius(op, U, iters):
    """rho of the FD Jacobian of f at U by power iteration.
    Slab runs (ghost rows after the owned ones) iterate on the owned rows
    with the ghost rows held at U (a per-slab estimate; the caller takes
    the max over ranks)."""
    import torch
    n_own = op.n_owned
    g = torch.Generator(device=U.device).manual_seed(1234)
    v = torch.randn((n_own,) + tuple(U.shape[1:]), dtype=torch.float64, device=U.device,
                    generator=g)
    v /= torch.linalg.norm(v)
    fU = op.apply_f(U)
    eps = math.sqrt(np.finfo(float).eps) * (1.0 + torch.linalg.norm(U[:n_own]).item())
    rho = 0.0
    Up = U.clone()
    for _ in range(iters):
        Up[:n_own] = U[:n_own] + eps * v
        Jv = (op.apply_f(Up) - fU) / eps
        n = torch.linalg.norm(Jv)
        rho = n.item()
        v = Jv / n
    return rho


def measured_hbm_gbs():
    """Driver-measured HBM copy bandwidth (MEASURED_PEAKS.json), or None."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return None


def fp64_peak(op):
    """Measured DFMA throughput (TFLOP/s) of this GPU; the roofline
    denominator for the FP64-bound operator kernels."""
    import ctypes
    import torch
    lib = op.lib
    nthr = lib.tdg_fp64_probe_threads()
    out = torch.empty(nthr, dtype=torch.float64, device=op.device)
    iters = 20000
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for _ in range(2):
        lib.tdg_fp64_probe(out.data_ptr(), iters, st)
    best = 0.0
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        lib.tdg_fp64_probe(out.data_ptr(), iters, st)
        b.record()
        b.synchronize()
        best = max(best, nthr * 16 * 2 * iters / (a.elapsed_time(b) * 1e-3) / 1e12)
    return best


def cpu_reference(cfg_name, scheme_name, steps, warmup, nthreads, dt=None):
    """Time the CPU oracle port on the same config; returns (DoF-upd/s,
    sample description, n_dofs)."""
    from oracle import OracleOperator
    cfg, space, model, scheme, U0, _ = build_problem(cfg_name, scheme_name, cpu_sample=True)
    op = OracleOperator(space, model, scheme, nthreads=nthreads)
    if dt is None:
        from paper_1403_1157_b200.configs import rho_constant
        h = float(space.mesh.diameters.min())
        dt = 0.8 * 2.51 / (rho_constant(cfg.dim, cfg.order) * 1e-2 / h ** 2)
    U = U0.copy()

    def step(U):
        U1 = U + dt * op.apply_f(U)
        U2 = 0.75 * U + 0.25 * (U1 + dt * op.apply_f(U1))
        return U / 3.0 + (2.0 / 3.0) * (U2 + dt * op.apply_f(U2))

    for _ in range(warmup):
        U = step(U)
    tic = time.perf_counter()
    for _ in range(steps):
        U = step(U)
    el = time.perf_counter() - tic
    return space.n_dofs * 3 * steps / el, el, cfg.cells, space.n_dofs


# ---------------------------------------------------------------- arms

def run_reference_arm(args, rank):
    if rank != 0:
        return
    nthreads = os.cpu_count() or 1
    steps = max(1, args.steps)
    warm = max(0, min(args.warmup, 1))
    val, el, cells, ndofs = cpu_reference(args.config, args.scheme, steps, warm, nthreads)
    full = tuple(weak_config(__import__("paper_1403_1157_b200.configs", fromlist=["CONFIGS"])
                             .CONFIGS[args.config], 1).cells)
    where = ("one full " + args.config + "-sized mesh (= one rank's weak-scaling slab)"
             if tuple(cells) == full else
             "a " + "x".join(map(str, cells)) + "-cell x-slab of the " + args.config
             + " mesh (same cells, order, physics; bounded CPU sample)")
    from paper_1403_1157_b200.configs import CONFIGS
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT,
        "n_gpus": args.gpus, "steps": steps, "warmup": warm,
        "ms_per_step": el / steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Gaussian bumps, L2-projected)",
        "config": {"workload": CONFIGS[args.config].description
                   + f", {args.scheme}, SSP-RK3 steps (3 f-evals each)",
                   "n_dofs": ndofs},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": nthreads,
                         "kind": "port",
                         "sample": f"{steps} SSP-RK3 steps of {where}, numpy oracle "
                                   f"port of the reference (oracle/), {nthreads} threads"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


_T0 = time.time()


def log(msg):
    print(f"[bench {time.time() - _T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


def run_native_arm(args, rank, world, local):
    import torch
    from paper_1403_1157_b200.operator import DiscreteOperator
    from paper_1403_1157_b200.roofline import apply_bytes, apply_flops, executed_flops

    local = local % max(torch.cuda.device_count(), 1)  # testing: ranks may share a GPU
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or "RANK" in os.environ:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:  # testing only: host-staged exchange, several ranks per GPU
            dist.init_process_group("gloo")
    dist_on = torch.distributed.is_available() and torch.distributed.is_initialized()
    cfg, space, model, scheme, U0h, slab = build_problem(args.config, args.scheme, rank, world,
                                                         args.force_slab, dev)
    log(f"problem built: {space.mesh.n_elements} elements")
    op = DiscreteOperator(space, model, scheme, device=dev,
                          n_owned=None if slab is None else slab.n_owned,
                          global_ids=None if slab is None else slab.global_ids,
                          bands=args.bands)
    log("operator created")
    if args.variant:
        op.set_variant(generic=bool(args.variant & 1), vol4=bool(args.variant & 2),
                       serial=bool(args.variant & 4), flip_mma=bool(args.variant & 8),
                       mma_volume=bool(args.variant & 16),
                       no_graph=bool(args.variant & 32),
                       tc_volume=bool(args.variant & 4096),
                       no_tc_faces=bool(args.variant & 8192),
                       volume_first=bool(args.variant & 16384),
                       face_rows_tc=bool(args.variant & 32768),
                       one_copy_stream=bool(args.variant & 65536),
                       walls_first=bool(args.variant & 131072),
                       copy_streams=(args.variant >> 18) & 7,
                       face_ctas_per_sm=(args.variant >> 8) & 15)
    t = op.tables
    d, nb = t.dim, t.nb
    ne, n_int, n_bnd = op.n_owned, len(t.if_code), len(t.bf_code)
    n_dofs = ne * 6 * nb          # owned DoFs of this rank

    from paper_1403_1157_b200.stepping import SSPRK3
    halo = None
    if slab is not None:
        from paper_1403_1157_b200.decomp import HaloExchange
        halo = HaloExchange(slab, dev)
    stepper = SSPRK3(op, halo)
    U = torch.from_numpy(U0h).to(dev)
    if dist_on:
        # initialise the NCCL communicator with a collective before the
        # first batched point-to-point exchange
        torch.distributed.barrier()
    if halo is not None:
        halo.exchange(U)
    rho = spectral_radius(op, U, args.power_iters)
    if dist_on:
        rr = torch.tensor([rho], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(rr, op=torch.distributed.ReduceOp.MAX)
        rho = rr.item()
    dt = 0.8 * 2.51 / rho
    log(f"rho {rho:.4e}")

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def barrier():
        if dist_on:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        stepper.step(U, dt)
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    for a, b in evs:
        flush.fill_(1.0)
        a.record()
        stepper.step(U, dt)
        b.record()
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    ms = sum(a.elapsed_time(b) for a, b in evs)
    if dist_on:
        tt = torch.tensor([ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms = tt.item()
    # per-kernel times: a separate, untimed profiling pass (per-launch CUDA
    # events on the launching streams; the timed steps above replay the
    # step's CUDA graph, which per-kernel events would break up)
    nprof = max(1, min(args.steps, 5))
    op.profile(True)
    pevs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(nprof)]
    for a, b in pevs:
        flush.fill_(1.0)
        a.record()
        stepper.step(U, dt)
        b.record()
    torch.cuda.synchronize()
    op.profile(False)
    kt = op.profile_read()
    ms_prof = sum(a.elapsed_time(b) for a, b in pevs)
    total_dofs = n_dofs
    if dist_on:  # whole-job DoFs (owned rows of every rank)
        td = torch.tensor([float(n_dofs)], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(td, op=torch.distributed.ReduceOp.SUM)
        total_dofs = int(td.item())
    value = total_dofs * 3 * args.steps / (ms * 1e-3)

    # per-kernel roofline (algorithmic flops of the reference sequence)
    Q, F = t.nq_vol, t.nq_face
    fv, ff, fb = apply_flops(d, nb, Q, F, ne, n_int, n_bnd)
    per = {}
    for name, flops in (("faces", ff), ("wall", fb), ("volume", fv), ("fc_add", 0.0)):
        tms, nl = kt[name]
        if nl:
            per[name] = {"avg_ms": tms / nl, "launches": nl * args.steps // nprof,
                         "algorithmic_tflops": flops / (tms / nl * 1e-3) / 1e12,
                         "share_of_step": tms / ms_prof}
    if "fc_add" in per and "volume" in per:
        # overlapped schedule: the volume part is launched on a second
        # stream beside the face kernel; its event span includes waiting for
        # SM resources the face kernel holds
        per["volume"]["note"] = "launched concurrently with faces; span includes co-scheduling"
    peak = fp64_peak(op)
    if "fc_add" in per:  # streaming kernel: report its bandwidth instead
        per["fc_add"]["gbs"] = (t.dim + 3) * n_dofs * 8 / (per["fc_add"]["avg_ms"] * 1e-3) / 1e9
        hbm = measured_hbm_gbs()
        if hbm:
            per["fc_add"]["hbm_peak_gbs"] = hbm
            per["fc_add"]["hbm_frac"] = per["fc_add"]["gbs"] / hbm
            per["fc_add"]["note"] = ("algorithmic bytes (d+1 slots + out read + out write) per "
                                     "launch / time; MEASURED_PEAKS.json copy bandwidth; >1 means "
                                     "part of the slots were still in L2")
    # the face kernel starts first and runs alone on the SMs it holds: its
    # span is its own duration; in the serial schedule take the longest
    dom = "faces" if ("faces" in per and "fc_add" in per) else \
        max((k for k in per if k != "fc_add"), key=lambda k: per[k]["avg_ms"])
    traffic = None
    try:  # dram read+write bytes per launch from the committed ncu capture
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            traffic = json.load(fh)["bytes_per_launch"].get(f"k_{dom}")
    except (OSError, ValueError, KeyError):
        traffic = None
    step_flops = 3 * (fv + ff + fb)
    roof = {"bound": "fp64", "kernel": f"k_{dom}",
            "bound_note": "fp64 workload (north_star: achieved FP64 throughput against the B200 "
                          "FP64 peak); DFMA and DMMA share the 37 TFLOP/s FP64 datapath, so "
                          "neither 'hbm' (<= 0.6 TB/s compulsory per step) nor the bf16 "
                          "tensor peak bounds it",
            "achieved": per[dom]["algorithmic_tflops"], "peak": peak,
            "unit": "TFLOP/s", "frac": per[dom]["algorithmic_tflops"] / peak,
            "traffic": traffic,
            "traffic_source": "profiles/ncu_traffic.json (ncu --set full dram bytes/launch)",
            "peak_source": "measured DFMA loop (tdg_fp64_probe) on this GPU; "
                           f"nominal {FP64_NOMINAL_TFLOPS} TFLOP/s; "
                           "MEASURED_PEAKS.json has no fp64 figure",
            "per_kernel": per,
            "step_algorithmic_tflops": step_flops / (ms / args.steps * 1e-3) / 1e12,
            "step_frac": step_flops / (ms / args.steps * 1e-3) / 1e12 / peak,
            "step_executed_tflops": 3 * executed_flops(d, nb, Q, F, ne, n_int, n_bnd)
            / (ms / args.steps * 1e-3) / 1e12,
            "step_hbm_gbs_compulsory": 3 * apply_bytes(d, n_dofs, ne, n_int, n_bnd)
            / (ms / args.steps * 1e-3) / 1e9}

    # end to end through the public API: pinned host U -> device, one
    # SSP-RK3 step, result back to host, every step
    e2e = None
    if not args.no_e2e:
        # the public host-data call: every step copies the state in from
        # pinned host memory and the result back out (undecomposed runs:
        # DiscreteOperator.ssprk3_steps_host, copies pipelined by element
        # bands; slab runs: copy-in, SSPRK3 step with the exchange, copy-out)
        Uh = torch.from_numpy(U0h).pin_memory()
        host_api = slab is None
        if host_api:
            op.ssprk3_steps_host(Uh, 2, dt)
        else:
            Ud = torch.empty_like(U)
            for _ in range(2):
                Ud.copy_(Uh, non_blocking=True)
                stepper.step(Ud, dt)
                Uh.copy_(Ud, non_blocking=True)
        torch.cuda.synchronize()
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        t_enq = time.perf_counter()
        if host_api:
            op.ssprk3_steps_host(Uh, args.steps, dt)
        else:
            for _ in range(args.steps):
                Ud.copy_(Uh, non_blocking=True)
                stepper.step(Ud, dt)
                Uh.copy_(Ud, non_blocking=True)
        b.record()
        t_enq = time.perf_counter() - t_enq
        b.synchronize()
        ems = a.elapsed_time(b)
        if dist_on:
            tt = torch.tensor([ems], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            ems = tt.item()
        e2e = {"value": total_dofs * 3 * args.steps / (ems * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": Uh.numel() * 8, "d2h_bytes_per_step": Uh.numel() * 8,
               "ms_per_step": ems / args.steps, "host_issue_ms_per_step": t_enq * 1e3 / args.steps,
               "api": "DiscreteOperator.ssprk3_steps_host (tdg_ssprk3_steps_host): per-step "
                      "copy-in / copy-out pipelined by element bands" if host_api else
                      "copy-in, SSPRK3.step with the halo exchange, copy-out per step"}

    # the reference's default integrator on the same state:
    # one SDIRK3 + JFNK step at dt 0.01 (C2) with the reference's Newton /
    # GMRES settings; DoF-updates counted per actual f evaluation
    implicit = None
    if world == 1 and slab is None and not args.no_implicit and cfg.dim == 2 and cfg.order == 2:
        from paper_1403_1157_b200.timeint import integrate
        nk = {"rtol": 1e-8, "atol": 1e-12, "maxiter": 25, "gmres_rtol": 1e-4,
              "gmres_restart": 30, "gmres_maxiter": 200}
        Ui = torch.from_numpy(U0h).to(dev)
        integrate(op, Ui, 0.0, 1.0, 0.01, order=3, n_steps=1, newton_kwargs=nk)  # warm-up
        torch.cuda.synchronize()
        ia, ib = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ia.record()
        res = integrate(op, Ui, 0.0, 1.0, 0.01, order=3, n_steps=1, newton_kwargs=nk)
        ib.record()
        ib.synchronize()
        ims = ia.elapsed_time(ib)
        implicit = {"value": n_dofs * res.f_evaluations / (ims * 1e-3), "unit": UNIT,
                    "integrator": "SDIRK3 + JFNK (reference defaults: Newton 1e-8/1e-12/25, "
                                  "GMRES(30) 1e-4/200), dt 0.01, 1 step from U0 after 1 warm-up step",
                    "ms_per_step": ims, "f_evaluations": res.f_evaluations,
                    "newton_iterations": res.newton_iterations,
                    "gmres_iterations": res.gmres_iterations}
        del Ui

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        nthreads = os.cpu_count() or 1
        val, el, cells, _ = cpu_reference(args.config, args.scheme, 1, 0, nthreads, dt=dt)
        where = (f"the full {args.config} mesh" if tuple(cells) == tuple(cfg.cells) else
                 "a " + "x".join(map(str, cells)) + f"-cell x-slab of the {args.config} mesh "
                 "(same cells, order, physics; bounded CPU sample)")
        cpu = {"value": val, "unit": UNIT, "cores": nthreads, "kind": "port",
               "sample": f"1 SSP-RK3 step (3 apply_f) of {where}, "
                         f"numpy oracle port, {nthreads} threads, {el:.1f} s"}

    launches = sum(v["launches"] for v in per.values())
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Gaussian bumps, L2-projected on host)",
            "config": {"workload": cfg.description + f", {args.scheme}, SSP-RK3 "
                       "steps (3 fused f-evals + stage updates each)",
                       "n_elements": ne, "n_dofs": n_dofs, "interior_faces": n_int,
                       "boundary_faces": n_bnd, "dt": dt, "rho": rho,
                       "l2": "flushed between timed steps (256 MiB write outside "
                             "the timed events)",
                       "parallelism": (f"x-slabs x{world}, NCCL ghost-row exchange per stage, "
                            "weak scaling (one config-sized slab per GPU)")
                           if world > 1 else "1 GPU"},
            "roofline": roof, "clocks": clocks, "gpu_launches": launches,
            **({"implicit": implicit} if implicit else {}),
        }
        if cpu:
            line["cpu_baseline"] = cpu
        if e2e:
            line["e2e"] = e2e
        print(json.dumps(line), flush=True)
    if dist_on:
        torch.distributed.destroy_process_group()


def run_implicit(args, rank, world, local):
    """C2 with the reference's default integrator: SDIRK3 + JFNK (dt 0.01,
    Newton 1e-8/1e-12/25, GMRES 1e-4/30/200; reference config.py:74-83).
    DoF-updates counted per actual f evaluation.  N > 1:
    weak-scaled slabs, ghost exchange inside every G(V) and the Krylov
    scalars all-reduced over NCCL (timeint.SlabReductions)."""
    import torch
    from paper_1403_1157_b200.operator import DiscreteOperator
    from paper_1403_1157_b200.timeint import integrate
    local = local % max(torch.cuda.device_count(), 1)  # testing: ranks may share a GPU
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or "RANK" in os.environ:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:  # testing only: host-staged exchange, several ranks per GPU
            dist.init_process_group("gloo")
    dist_on = torch.distributed.is_available() and torch.distributed.is_initialized()
    cfg, space, model, scheme, U0h, slab = build_problem(args.config, args.scheme, rank, world,
                                                         args.force_slab, dev)
    op = DiscreteOperator(space, model, scheme, device=dev,
                          n_owned=None if slab is None else slab.n_owned,
                          global_ids=None if slab is None else slab.global_ids)
    halo = None
    if slab is not None:
        from paper_1403_1157_b200.decomp import HaloExchange
        halo = HaloExchange(slab, dev)
    U = torch.from_numpy(U0h).to(dev)
    if dist_on:
        torch.distributed.barrier()
    nk = {"rtol": 1e-8, "atol": 1e-12, "maxiter": 25, "gmres_rtol": 1e-4,
          "gmres_restart": 30, "gmres_maxiter": 200}
    integrate(op, U, 0.0, 1.0, args.dt, order=3, n_steps=max(1, args.warmup),
              newton_kwargs=nk, halo=halo)
    torch.cuda.synchronize()
    if dist_on:
        torch.distributed.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    res = integrate(op, U, 0.0, 1.0, args.dt, order=3, n_steps=args.steps, newton_kwargs=nk,
                    halo=halo)
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b)
    n_dofs = op.n_owned * 6 * space.nb
    if dist_on:
        v = torch.tensor([ms, float(n_dofs)], dtype=torch.float64, device=dev)
        mx = v.clone()
        torch.distributed.all_reduce(mx, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(v, op=torch.distributed.ReduceOp.SUM)
        ms, n_dofs = float(mx[0]), int(v[1])
    if rank == 0:
        line = {"metric": METRIC, "value": n_dofs * res.f_evaluations / (ms * 1e-3),
                "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": cfg.description + f", {args.scheme}, SDIRK3 + JFNK "
                           f"(reference defaults), dt {args.dt}",
                           "f_evaluations": res.f_evaluations,
                           "newton_iterations": res.newton_iterations,
                           "gmres_iterations": res.gmres_iterations,
                           "parallelism": f"{world} x-slab(s)" if slab is not None else "1 GPU"}}
        print(json.dumps(line), flush=True)
    if dist_on:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference_arm(args, rank)
        return
    if args.integrator == "sdirk3":
        run_implicit(args, rank, world, local)
        return
    run_native_arm(args, rank, world, local)


if __name__ == "__main__":
    main()
