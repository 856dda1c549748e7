#!/usr/bin/env python
"""Benchmark: fp64 DG-operator DoF-updates/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5]
                    [--scaling strong|weak] [--impl native|reference]

A step is one Shu-Osher SSP-RK3 step = 3 applications of f = M^-1 L_h,
each fused with its Runge-Kutta stage update, over the whole mesh.
Unit of work: one DoF receiving one f evaluation, so
value = n_dofs * 3 * K / (device time of K steps), max over ranks.

Default workload: config C5 (BASELINE configs[4], the configuration the
metric is quoted on "at 1/2/4/8 B200"): [0,2]x[0,1]^2, 256x128x128 cells
x 6 Kuhn tetrahedra = 25.2M tets, p=3, 3.02e9 DoFs, cdg2, the explicit
CFL step dt = 0.8 * 2.51 / rho(J).  N > 1: the fixed C5 mesh split into
N x-slabs (strong scaling, NCCL ghost-row exchange per stage);
``--scaling weak`` gives every GPU a config-sized slab instead.  Inputs
are resident in HBM; the 24 GB state is far larger than L2 (small
configs flush L2 between timed steps).

``--impl reference`` times the CPU oracle port of the reference
(oracle/, numpy, all physical host cores, BLAS pinned to one thread)
on a bounded x-slab sample of the same config: the reference itself is
pure Python and cannot travel to the GPU box.
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
BIG_DOFS = 400_000_000      # above this: dt from a same-h replica, no L2 flush


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: 5 for c5, 20 otherwise)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N > 1: strong = the fixed config split into N x-slabs; "
                         "weak = one config-sized slab per GPU")
    ap.add_argument("--scheme", default="cdg2")
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: testing only (host-staged exchange; ranks may share a GPU)")
    ap.add_argument("--no-implicit", action="store_true",
                    help="skip the extra SDIRK3+JFNK figure of the explicit C2 run")
    ap.add_argument("--power-iters", type=int, default=200)
    ap.add_argument("--integrator", default="ssprk3", choices=["ssprk3", "sdirk3"],
                    help="sdirk3: the reference's default SDIRK3 + JFNK at --dt")
    ap.add_argument("--dt", type=float, default=None,
                    help="implicit step (default: the reference's 0.01; C3: the stiffness "
                         "ratio dt a_ii rho = 500, SURVEY 8(d) -- at 0.01 the reference's "
                         "own GMRES(30) stalls)")
    ap.add_argument("--force-slab", action="store_true",
                    help="use the slab/halo code path even at N=1 (testing)")
    ap.add_argument("--variant", type=int, default=0,
                    help="kernel variant bits (tdg_set_variant), for A/B timing")
    ap.add_argument("--cells", default=None,
                    help="override the config's cell counts, e.g. 64x32x32 (testing)")
    a = ap.parse_args()
    if a.steps is None:
        a.steps = 5 if a.config == "c5" else 20
    return a


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

def scaled_config(cfg, world, scaling, cells=None):
    """The job's mesh: the config itself (strong scaling; N ranks split it
    into x-slabs), or for weak scaling N config-sized x-slabs side by side
    (domain N times as long in x, same cell size)."""
    import dataclasses
    if cells:
        cfg = dataclasses.replace(
            cfg, cells=tuple(cells),
            description=cfg.description + " -- TEST OVERRIDE: " + "x".join(map(str, cells))
            + " cells (same cell aspect, order, physics)")
    if world == 1 or scaling == "strong":
        return cfg
    cells = (cfg.cells[0] * world,) + tuple(cfg.cells[1:])
    lengths = (cfg.lengths[0] * world,) + tuple(cfg.lengths[1:])
    desc = cfg.description + f" -- weak scaling: {world} config-sized x-slabs side by side"
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


def replica_config(cfg, max_cells=20_000):
    """A small mesh with the config's cell size (h), order, tags and
    physics: the stiffness (rho ~ C nu / h^2) of the full
    config, at a size the power iteration can afford next to a 24 GB
    state."""
    import dataclasses
    cells, lengths = list(cfg.cells), list(cfg.lengths)
    while int(np.prod(cells)) > max_cells:
        ax = int(np.argmax(cells))
        half = max(1, cells[ax] // 2)
        lengths[ax] *= half / cells[ax]
        cells[ax] = half
    return dataclasses.replace(cfg, cells=tuple(cells), lengths=tuple(lengths))


def build_problem(cfg_name, scheme_name, rank=0, world=1, scaling="strong", force_slab=False,
                  device=None, cpu_sample=False, cells=None, cfg=None):
    """(cfg, space, model, scheme, U0, slab).  U0 is a device tensor when
    ``device`` is given (projected on the device at scale), else numpy.
    The slab is None at N=1 unless ``force_slab``; ``cpu_sample``: the CPU
    baseline's bounded x-slab of the config (sample_config)."""
    from paper_1403_1157_b200 import DGSpace, FluxScheme, PlaqueModel
    from paper_1403_1157_b200.configs import CONFIGS, make_mesh
    from paper_1403_1157_b200.decomp import build_slab
    from paper_1403_1157_b200.fields import bump_field
    if cfg is None:
        cfg = scaled_config(CONFIGS[cfg_name], world, scaling, cells)
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
    if device is not None:
        if cfg.dim == 3 or mesh.n_elements > 500_000:
            # host projection is slow at scale (~0.4 ms/tet at 3D p=3)
            from paper_1403_1157_b200.fields import project_bumps_device
            U0 = project_bumps_device(space, fn, device)
        else:
            import torch
            U0 = torch.from_numpy(np.ascontiguousarray(space.project(fn).coeffs)).to(device)
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


def replica_rho(cfg, scheme_name, device, iters):
    """rho on a same-h replica (replica_config) of the config."""
    from paper_1403_1157_b200.operator import DiscreteOperator
    rc = replica_config(cfg)
    _, space, model, scheme, U0, _ = build_problem(None, scheme_name, device=device, cfg=rc)
    op = DiscreteOperator(space, model, scheme, device=device)
    return spectral_radius(op, U0, iters), rc


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return {}


def fp64_peak(op):
    """Measured DFMA throughput (TFLOP/s) of this GPU; the roofline
    denominator for the FP64-bound operator kernels (MEASURED_PEAKS.json
    has HBM and bf16 figures only)."""
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


def host_cpu():
    """(physical cores, CPU model) of this host."""
    cores = None
    try:
        import psutil
        cores = psutil.cpu_count(logical=False)
    except ImportError:
        pass
    cores = cores or os.cpu_count() or 1
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return int(cores), model


def cpu_reference(cfg_name, scheme_name, steps, warmup, dt=None, repeats=1, cells=None,
                  budget_s=None):
    """Time the CPU oracle port on a bounded sample of the config, under
    the reference's own scaling protocol (analysis.scaling_study,
    reference analysis.py:211-242: BLAS pinned to one thread, one worker
    thread per physical core, best of ``repeats``).  Returns (DoF-upd/s,
    best seconds, sample cells, sample DoFs, cores, cpu model)."""
    from threadpoolctl import threadpool_limits
    from oracle import OracleOperator
    cfg, space, model, scheme, U0, _ = build_problem(cfg_name, scheme_name, cpu_sample=True,
                                                     cells=cells)
    cores, cpu_model = host_cpu()
    op = OracleOperator(space, model, scheme, nthreads=cores)
    if dt is None:
        from paper_1403_1157_b200.configs import rho_constant
        h = float(space.mesh.diameters.min())
        dt = 0.8 * 2.51 / (rho_constant(cfg.dim, cfg.order) * 1e-2 / h ** 2)

    def step(U):
        U1 = U + dt * op.apply_f(U)
        U2 = 0.75 * U + 0.25 * (U1 + dt * op.apply_f(U1))
        return U / 3.0 + (2.0 / 3.0) * (U2 + dt * op.apply_f(U2))

    best = None
    with threadpool_limits(1):
        U = U0.copy()
        for _ in range(warmup):
            U = step(U)
        done, spent = 0, 0.0
        while done < max(1, repeats):
            tic = time.perf_counter()
            for _ in range(steps):
                U = step(U)
            el = time.perf_counter() - tic
            best = el if best is None else min(best, el)
            done += 1
            spent += el
            # best of `repeats`, cut short when another pass would push the
            # whole timing leg past the budget
            if budget_s is not None and spent + el > budget_s:
                break
    return space.n_dofs * 3 * steps / best, best, cfg.cells, space.n_dofs, cores, cpu_model


# ---------------------------------------------------------------- arms

def run_reference_arm(args, rank):
    if rank != 0:
        return
    # the driver's --steps K --warmup W, as given: each step is one SSP-RK3
    # step of the bounded sample (a few seconds on 16 cores at C5), best of
    # up to 3 passes within about two minutes
    steps = max(1, args.steps)
    warm = max(0, args.warmup)
    cells = tuple(int(c) for c in args.cells.split("x")) if args.cells else None
    val, el, scells, ndofs, cores, cpu_model = cpu_reference(
        args.config, args.scheme, steps, warm, repeats=3, cells=cells, budget_s=120.0)
    from paper_1403_1157_b200.configs import CONFIGS
    cfg = scaled_config(CONFIGS[args.config], 1, "strong", cells)
    where = ("the full " + args.config + " mesh" if tuple(scells) == tuple(cfg.cells) else
             "a " + "x".join(map(str, scells)) + "-cell x-slab of the " + args.config
             + " mesh (same cells, order, physics; bounded CPU sample)")
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT,
        "n_gpus": args.gpus, "steps": steps, "warmup": warm,
        "ms_per_step": el / steps * 1e3, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Gaussian bumps, L2-projected)",
        # the same workload string as the native arm's line; the CPU arm times
        # a bounded sample of it (cpu_baseline.sample)
        "config": {"workload": cfg.description + f", {args.scheme}, SSP-RK3 "
                   "steps (3 fused f-evals + stage updates each)",
                   "n_elements": int(np.prod(cfg.cells)) * (2 if cfg.dim == 2 else 6),
                   "n_dofs_sample": ndofs,
                   "parallelism": f"{cores} host threads (reference CPU path)"},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "port",
                         "cpu_model": cpu_model,
                         "sample": f"{steps} SSP-RK3 step(s) of {where}, numpy oracle port "
                                   f"of the reference (oracle/), {cores} worker threads "
                                   f"(physical cores), BLAS pinned to 1 thread, best of up "
                                   f"to 3 passes"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


_T0 = time.time()


def log(msg):
    print(f"[bench {time.time() - _T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


def _init_dist(args, world, dev):
    """One process per GPU; NCCL over NVLink for the ghost-row exchange and
    the Krylov all-reduces.  Logs one line per rank (rank, world, device,
    backend, NCCL version) so a failing rank is identifiable."""
    import torch
    if world > 1 or "RANK" in os.environ:
        import torch.distributed as dist
        os.environ.setdefault("NCCL_DEBUG", "WARN")
        try:
            if args.dist_backend == "nccl":
                dist.init_process_group("nccl", device_id=dev)
            else:  # testing only: host-staged exchange, several ranks per GPU
                dist.init_process_group("gloo")
        except Exception as err:  # noqa: BLE001 -- re-raised with the rank attached
            raise RuntimeError(f"rank {os.environ.get('RANK')}/{world} on {dev}: "
                               f"{args.dist_backend} process-group init failed: {err}") from err
        nccl = ".".join(map(str, torch.cuda.nccl.version())) if args.dist_backend == "nccl" \
            else "-"
        log(f"rank {dist.get_rank()}/{dist.get_world_size()} on {dev} "
            f"({torch.cuda.get_device_name(dev)}), backend {dist.get_backend()}, nccl {nccl}, "
            f"master {os.environ.get('MASTER_ADDR')}:{os.environ.get('MASTER_PORT')}")
    return torch.distributed.is_available() and torch.distributed.is_initialized()


def run_native_arm(args, rank, world, local):
    import torch
    from paper_1403_1157_b200.operator import DiscreteOperator
    from paper_1403_1157_b200.roofline import apply_bytes, apply_flops, executed_split

    local = local % max(torch.cuda.device_count(), 1)  # testing: ranks may share a GPU
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist_on = _init_dist(args, world, dev)
    cells = tuple(int(c) for c in args.cells.split("x")) if args.cells else None
    cfg, space, model, scheme, U, slab = build_problem(args.config, args.scheme, rank, world,
                                                       args.scaling, args.force_slab, dev,
                                                       cells=cells)
    log(f"problem built: {space.mesh.n_elements} elements")
    op = DiscreteOperator(space, model, scheme, device=dev,
                          n_owned=None if slab is None else slab.n_owned,
                          global_ids=None if slab is None else slab.global_ids)
    log(f"operator created: {op.tables.n_seg} colour segments")
    if args.variant:
        op.lib.tdg_set_variant(op._ctx, args.variant)
    t = op.tables
    d, nb = t.dim, t.nb
    ne, n_int, n_bnd = op.n_owned, len(t.if_code), len(t.bf_code)
    n_dofs = ne * 6 * nb          # owned DoFs of this rank
    big = cfg.dim == 3 and np.prod(cfg.cells) * 6 * 6 * nb > BIG_DOFS

    from paper_1403_1157_b200.stepping import SSPRK3
    halo = None
    if slab is not None:
        from paper_1403_1157_b200.decomp import HaloExchange
        halo = HaloExchange(slab, dev)
    stepper = SSPRK3(op, halo)
    if dist_on:
        # initialise the NCCL communicator with a collective before the
        # first batched point-to-point exchange
        torch.distributed.barrier()
    if halo is not None:
        halo.exchange(U)
    if big:   # a 24 GB state leaves no room for the power iteration's vectors
        rho, rcfg = replica_rho(cfg, args.scheme, dev, args.power_iters)
        rho_src = ("power iteration on a same-h replica (" + "x".join(map(str, rcfg.cells))
                   + " cells)")
    else:
        rho = spectral_radius(op, U, args.power_iters)
        rho_src = "power iteration on the benchmark state"
    if dist_on:
        rr = torch.tensor([rho], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(rr, op=torch.distributed.ReduceOp.MAX)
        rho = rr.item()
    dt = 0.8 * 2.51 / rho
    log(f"rho {rho:.4e} ({rho_src}), dt {dt:.3e}")

    flush = None if big else torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def barrier():
        if dist_on:
            torch.distributed.barrier()

    # full-size property check (size-independent): the lipid
    # budget c2 + c3 changes only through the GAMMA1_IN influx, at exactly
    # nu2 sigma |GAMMA1_IN| per unit time (oxidation moves c2 to c3; the
    # face terms conserve; reference tests/test_operator.py:101-110)
    def lipid_total(V):
        tot = op.species_totals(V)
        if dist_on:
            torch.distributed.all_reduce(tot)
        return float(tot[4] + tot[5])
    gamma1_in = float(op.tables.bf_geo[((op.tables.bf_code >> 11) & 7) == 2].sum()) * \
        (1.0 if cfg.dim == 2 else 0.5)
    if dist_on:
        gi = torch.tensor([gamma1_in], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(gi)
        gamma1_in = float(gi)
    lipid0, steps_taken = lipid_total(U), 0

    for _ in range(args.warmup):
        stepper.step(U, dt)
    steps_taken += args.warmup
    torch.cuda.synchronize()
    log("warm-up done")

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    for a, b in evs:
        if flush is not None:
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
    log(f"timed: {ms / args.steps:.3f} ms/step")
    # per-kernel times: a separate, untimed profiling pass (per-launch CUDA
    # events on the launching stream; the timed steps above replay the
    # step's CUDA graph, which per-kernel events would break up)
    nprof = 1 if big else max(1, min(args.steps, 5))
    op.profile(True)
    pevs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(nprof)]
    for a, b in pevs:
        if flush is not None:
            flush.fill_(1.0)
        a.record()
        stepper.step(U, dt)
        b.record()
    torch.cuda.synchronize()
    op.profile(False)
    kt = op.profile_read()
    steps_taken += args.steps + nprof
    lipid1 = lipid_total(U)
    p = model.params
    expect = steps_taken * dt * p.nu2 * p.sigma * gamma1_in
    checks = {"lipid_budget_change": lipid1 - lipid0, "expected": expect,
              "rel_err": abs(lipid1 - lipid0 - expect) / abs(expect) if expect else None,
              "steps": steps_taken, "finite": bool(torch.isfinite(U[:op.n_owned]).all()),
              "what": "full-size size-independent check: the c2 + c3 total after the run's "
                      "SSP-RK3 steps changed by steps * dt * nu2 * sigma * |GAMMA1_IN| "
                      "(reference tests/test_operator.py:101-110), device totals"}
    log(f"lipid budget check: rel err {checks['rel_err']}")
    if slab is None and stepper._work is not None:
        # bitwise run-to-run reproducibility at full size (the reference's
        # determinism contract, tests/test_operator.py:113-119): one fused
        # stage evaluated twice into the two work vectors
        W = stepper._work
        op.rk_stage(U, U, W[0], 0.75, 0.25, 0.25 * dt)
        op.rk_stage(U, U, W[1], 0.75, 0.25, 0.25 * dt)
        checks["stage_bitwise_reproducible"] = bool(torch.equal(W[0], W[1]))
        log(f"stage reproducibility check: {checks['stage_bitwise_reproducible']}")
    ms_prof = sum(a.elapsed_time(b) for a, b in pevs)
    total_dofs = n_dofs
    if dist_on:  # whole-job DoFs (owned rows of every rank)
        td = torch.tensor([float(n_dofs)], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(td, op=torch.distributed.ReduceOp.SUM)
        total_dofs = int(td.item())
    value = total_dofs * 3 * args.steps / (ms * 1e-3)

    # per-kernel roofline (algorithmic flops of the reference sequence,
    # per application; every kernel class runs once per colour segment)
    Q, F = t.nq_vol, t.nq_face
    fv, ff, fb = apply_flops(d, nb, Q, F, ne, n_int, n_bnd)
    names = op.kernel_names()
    per = {}
    xv, xf, xb = executed_split(d, nb, Q, F, ne, n_int, n_bnd,
                                face_classes=op.n_face_classes > 0,
                                vol_classes=op.n_volume_classes > 0,
                                modal_order=t.order if names["faces"] == "k_faces_tcm" else None)
    peak = fp64_peak(op)
    for name, flops, xfl in (("faces", ff, xf), ("wall", fb, xb), ("volume", fv, xv)):
        tms, nl = kt[name]
        if nl:
            apps = 3 * nprof
            sec = tms / apps * 1e-3
            per[name] = {"kernel": names[name], "ms_per_application": tms / apps,
                         "launches_per_application": nl / apps,
                         "algorithmic_tflops": flops / sec / 1e12,
                         "executed_tflops": xfl / sec / 1e12,
                         "executed_frac": xfl / sec / 1e12 / peak,
                         "share_of_step": tms / ms_prof}
    pk = measured_peaks()
    dom = max(per, key=lambda k: per[k]["share_of_step"])
    traffic = None
    try:  # dram read+write bytes per application from the committed ncu capture
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            tr = json.load(fh)
        ent = tr["bytes_per_application"].get(f"{args.config}:{per[dom]['kernel']}")
        traffic = ent
    except (OSError, ValueError, KeyError):
        traffic = None
    step_flops = 3 * (fv + ff + fb)
    step_s = ms / args.steps * 1e-3
    roof = {"bound": "fp64", "kernel": per[dom]["kernel"],
            "bound_note": "fp64 workload (north_star: achieved FP64 throughput against the B200 "
                          "FP64 peak); DFMA and DMMA share the FP64 datapath, so neither 'hbm' "
                          "(compulsory traffic far below 1 TB/s) nor the bf16 tensor peak "
                          "bounds it",
            "achieved": per[dom]["algorithmic_tflops"], "peak": peak,
            "unit": "TFLOP/s", "frac": per[dom]["algorithmic_tflops"] / peak,
            "executed_achieved": per[dom]["executed_tflops"],
            "executed_frac": per[dom]["executed_frac"],
            "frac_note": "frac uses the reference's operation sequence (SURVEY 8(d)); the kernels "
                         "reach the same result with fewer flops (modal face space, exact "
                         "stiffness), so frac can exceed 1; executed_frac counts the flops the "
                         "kernel actually performs (no tensor-core padding)",
            "traffic": traffic,
            "achieved_note": "algorithmic flops of the kernel class per application (SURVEY "
                             "8(d) per-face / per-element figures x counts) / the summed "
                             "duration of its launches per application (one per colour "
                             "segment), CUDA events on the launching stream",
            "traffic_source": "profiles/ncu_traffic.json (ncu --set full dram bytes per "
                              "application, summed over the kernel's launches)",
            "peak_source": "builder-measured DFMA peak (tdg_fp64_probe, 16 independent FMA "
                           f"chains per thread) on this GPU; nominal {FP64_NOMINAL_TFLOPS} "
                           "TFLOP/s; MEASURED_PEAKS.json has no fp64 figure",
            "per_kernel": per,
            "step_algorithmic_tflops": step_flops / step_s / 1e12,
            "step_frac": step_flops / step_s / 1e12 / peak,
            "step_executed_tflops": 3 * (xv + xf + xb) / step_s / 1e12,
            "executed_note": "executed = the kernels' reformulated sequence without tensor-core "
                             "padding (roofline.executed_split); the frac above uses the "
                             "reference's algorithmic sequence, which is larger",
            "step_hbm_gbs_compulsory": 3 * apply_bytes(d, n_dofs, ne, n_int, n_bnd) / step_s / 1e9,
            "hbm_peak_gbs": pk.get("hbm_gbs")}

    # end to end through the public API: pinned host U -> device, one
    # SSP-RK3 step, result back to host, every step
    e2e = None
    if not args.no_e2e:
        try:
            # the public host-data call: every step copies the state in from
            # pinned host memory and the result back out (undecomposed runs:
            # DiscreteOperator.ssprk3_steps_host; slab runs: copy-in, SSPRK3
            # step with the exchange, copy-out)
            log("e2e: pinning the host state")
            Uh = U.cpu().pin_memory()
            host_api = slab is None
            work = stepper._work if stepper._work is not None else op.new_work()
            if host_api:
                op.ssprk3_steps_host(Uh, 1, dt, U=U, work=work)
            else:
                for _ in range(1):
                    U.copy_(Uh, non_blocking=True)
                    stepper.step(U, dt)
                    Uh.copy_(U, non_blocking=True)
            torch.cuda.synchronize()
            barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            t_enq = time.perf_counter()
            if host_api:
                op.ssprk3_steps_host(Uh, args.steps, dt, U=U, work=work)
            else:
                for _ in range(args.steps):
                    U.copy_(Uh, non_blocking=True)
                    stepper.step(U, dt)
                    Uh.copy_(U, non_blocking=True)
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
                          "copy-in / copy-out of the pinned host state in 8 chunks, overlapping "
                          "the previous step's copy-out and the last stage" if host_api else
                          "copy-in, SSPRK3.step with the halo exchange, copy-out per step"}
            log(f"e2e: {ems / args.steps:.3f} ms/step")
            # the reference's own call shape: one apply_f(numpy) -> numpy per
            # f-evaluation (reference operator.py:286; its stepper composes
            # three per SSP-RK3 step), pageable host memory both ways
            if slab is None:
                Un = Uh.numpy().copy()  # pageable, like a user's numpy state
                op.apply_f(Un)
                torch.cuda.synchronize()
                nrep = 1 if big else 5
                tic = time.perf_counter()
                for _ in range(nrep):
                    Fh = op.apply_f(Un)
                el = (time.perf_counter() - tic) / nrep
                e2e["reference_call_shape"] = {
                    "value": n_dofs / el, "unit": UNIT, "ms_per_apply_f": el * 1e3,
                    "h2d_bytes_per_call": Un.nbytes, "d2h_bytes_per_call": Fh.nbytes,
                    "api": "DiscreteOperator.apply_f(numpy) -> numpy (tdg_apply_host: staged copies through pinned buffers), one f-evaluation per call "
                           "(wall clock, pageable host arrays, result allocated per call)"}
                del Fh, Un
            del Uh
        except (RuntimeError, MemoryError) as err:  # e.g. no room to pin / copy the host state
            # single-GPU runs only reach this on a host-memory shortage: the device line
            # above is still valid, so report it and say why e2e is missing
            log(f"e2e leg failed: {err!r}")
            if dist_on:
                raise
            e2e = {"unavailable": repr(err)[:300]}
            torch.cuda.synchronize()

    # the reference's default integrator on the same state:
    # one SDIRK3 + JFNK step at dt 0.01 (C2) with the reference's Newton /
    # GMRES settings; DoF-updates counted per actual f evaluation
    implicit = None
    if world == 1 and slab is None and not args.no_implicit and cfg.dim == 2 and cfg.order == 2:
        from paper_1403_1157_b200.timeint import integrate
        nk = {"rtol": 1e-8, "atol": 1e-12, "maxiter": 25, "gmres_rtol": 1e-4,
              "gmres_restart": 30, "gmres_maxiter": 200}
        Ui = U.clone()
        args.dt = 0.01 if args.dt is None else args.dt
        integrate(op, Ui, 0.0, 1.0, args.dt, order=3, n_steps=1, newton_kwargs=nk)  # warm-up
        torch.cuda.synchronize()
        ia, ib = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ia.record()
        res = integrate(op, Ui, 0.0, 1.0, args.dt, order=3, n_steps=1, newton_kwargs=nk)
        ib.record()
        ib.synchronize()
        ims = ia.elapsed_time(ib)
        implicit = {"value": n_dofs * res.f_evaluations / (ims * 1e-3), "unit": UNIT,
                    "integrator": "SDIRK3 + JFNK (reference defaults: Newton 1e-8/1e-12/25, "
                                  "GMRES(30) 1e-4/200), dt 0.01, 1 step after 1 warm-up step",
                    "ms_per_step": ims, "f_evaluations": res.f_evaluations,
                    "newton_iterations": res.newton_iterations,
                    "gmres_iterations": res.gmres_iterations}
        del Ui

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        log("cpu baseline")
        val, el, scells, _, cores, cpu_model = cpu_reference(args.config, args.scheme, 1, 0,
                                                             dt=dt, repeats=3, cells=cells)
        where = (f"the full {args.config} mesh" if tuple(scells) == tuple(cfg.cells) else
                 "a " + "x".join(map(str, scells)) + f"-cell x-slab of the {args.config} mesh "
                 "(same cells, order, physics; bounded CPU sample)")
        cpu = {"value": val, "unit": UNIT, "cores": cores, "kind": "port",
               "cpu_model": cpu_model,
               "sample": f"1 SSP-RK3 step (3 apply_f) of {where}, numpy oracle port, "
                         f"{cores} worker threads (physical cores), BLAS pinned to 1 thread, "
                         f"best of 3: {el:.1f} s"}

    launches = int(sum(v["launches_per_application"] for v in per.values()) * 3 * args.steps)
    if rank == 0:
        par = "1 GPU" if world == 1 else (
            f"x-slabs x{world}, NCCL ghost-row exchange per stage overlapped with the owned-row "
            f"faces, " + ("strong scaling (the fixed config split)" if args.scaling == "strong"
                          else "weak scaling (one config-sized slab per GPU)"))
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Gaussian bumps, L2-projected)",
            "config": {"workload": cfg.description + f", {args.scheme}, SSP-RK3 "
                       "steps (3 fused f-evals + stage updates each)",
                       "n_elements": int(np.prod(cfg.cells)) * (2 if d == 2 else 6),
                       "n_dofs": total_dofs, "interior_faces_rank0": n_int,
                       "boundary_faces_rank0": n_bnd, "colour_segments": t.n_seg,
                       "dt": dt, "rho": rho, "rho_source": rho_src,
                       "l2": ("inputs larger than L2 (state vectors of "
                              f"{n_dofs * 8 / 1e9:.1f} GB), no flush") if big else
                             "flushed between timed steps (256 MiB write outside the timed "
                             "events)",
                       "parallelism": par},
            "roofline": roof, "clocks": clocks, "gpu_launches": launches,
            "full_size_checks": checks,
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
    """The reference's default integrator: SDIRK3 + JFNK (dt 0.01, Newton
    1e-8/1e-12/25, GMRES 1e-4/30/200; reference config.py:74-83).
    DoF-updates counted per actual f evaluation.  N > 1:
    slabs, ghost exchange inside every G(V) and the Krylov scalars
    all-reduced over NCCL (timeint.SlabReductions)."""
    import torch
    from paper_1403_1157_b200.operator import DiscreteOperator
    from paper_1403_1157_b200.timeint import integrate
    local = local % max(torch.cuda.device_count(), 1)  # testing: ranks may share a GPU
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist_on = _init_dist(args, world, dev)
    cells = tuple(int(c) for c in args.cells.split("x")) if args.cells else None
    cfg, space, model, scheme, U, slab = build_problem(args.config, args.scheme, rank, world,
                                                       args.scaling, args.force_slab, dev,
                                                       cells=cells)
    op = DiscreteOperator(space, model, scheme, device=dev,
                          n_owned=None if slab is None else slab.n_owned,
                          global_ids=None if slab is None else slab.global_ids)
    halo = None
    if slab is not None:
        from paper_1403_1157_b200.decomp import HaloExchange
        halo = HaloExchange(slab, dev)
    if dist_on:
        torch.distributed.barrier()
    nk = {"rtol": 1e-8, "atol": 1e-12, "maxiter": 25, "gmres_rtol": 1e-4,
          "gmres_restart": 30, "gmres_maxiter": 200}
    if args.dt is None:
        if args.config == "c3":
            from paper_1403_1157_b200.configs import rho_constant
            h = float(space.mesh.diameters.min())
            args.dt = 500.0 / (0.4358665215 * rho_constant(cfg.dim, cfg.order) * 1e-2 / h ** 2)
        else:
            args.dt = 0.01
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
                "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
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
