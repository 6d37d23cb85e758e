"""Benchmark: HBPC(q, k_max) / DGSEM time steps on B200 (arXiv 2109.04804).

One bench "step" is one HBPC time step (Alg. 1) of a BASELINE
config -- every row of SURVEY 8(a): residual, FD JVP, BJ_ext build + apply,
Arnoldi, Newton updates, stage combinations (C5 adds the NS lifting, a14).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3|C4|C5]
                    [--scaling weak|strong] [--impl ours|reference]

* default: C3 (2D Euler isentropic vortex, 128x128 elements, N=7, GLL, LLF,
  HBPC(8,4), BJ_ext, FD JVP, Newton/GMRES rtol 1e-10) on 1 GPU.
* --gpus N without torchrun re-launches itself under torch.distributed.run
  with N ranks (one process per GPU, NCCL); under torchrun WORLD_SIZE must
  equal --gpus.
* --scaling strong: one fixed global mesh element-partitioned px x py
  (1x1, 2x1, 2x2, 4x2); the default for C4 and C5 (parallel
  efficiency is strong scaling on C4).  --scaling weak: one copy of the
  config's mesh per GPU (a (nx px) x (ny py) periodic tiling); the default
  for C3.  `value` is the units all ranks processed / device time (max over
  ranks): strong = global steps/s; weak = config-tile steps/s (N x global).
* `value` is timed with the library's per-kernel profiling OFF; the kernel
  table comes from a separate profiled pass (--profile-steps).  `e2e` replays
  the same K steps from the same state through hbpdc_step_host (host buffer,
  H2D + step + D2H per step).
* --impl reference times the CPU oracle (oracle/, test infrastructure) on a
  bounded sample of the same workload (one predictor stage solve on a small
  periodic window of the config's mesh, same h, N, dt, tolerances), scaled to
  steps/s; ms_per_step is the wall time of one sample.
"""
import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "HBPDC steps/s"
UNIT = "steps/s"
FP64_PEAK_TFLOPS = 37.0     # measured DMMA peak on this B200 pool (scripts/dmma_peak.cu)
PARTS = {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (4, 2)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


IC_CASE = {"T3": "TGV3"}          # input recipe of a bench config (inputs.ic_primitive)


def get_config(name):
    from paper_2109_04804_b200 import configs
    return configs.CONFIGS[name] if name in configs.CONFIGS else configs.EXTRA[name]


def workload_name(cfg, args):
    eqn = {"euler": "3D Euler" if cfg.dim == 3 else "2D Euler",
           "navier_stokes": "2D Navier-Stokes (BR1, Re 1000, Pr 0.72)",
           "advection": "2D advection"}[cfg.equation]
    ic = {"C3": "isentropic vortex (beta=5, mean (1,1)) + seeded U[-1e-6,1e-6) noise",
          "C4": "density wave rho=1+0.2 sin(2 pi (x+y)), u=v=p=1",
          "C5": "TGV-type vortex, Mach 0.1",
          "T3": "Taylor-Green data (P:1088-1091, reading R35, inviscid), acoustic element CFL 1"}[cfg.name]
    mesh = f"{cfg.nx}x{cfg.ny}x{cfg.nz}" if cfg.dim == 3 else f"{cfg.nx}x{cfg.ny}"
    return (f"{cfg.name}: {eqn} {ic}, {mesh} elements, N={cfg.N} {args.nodes.upper()}, "
            f"{args.flux.upper()}, HBPC({cfg.q},{cfg.kmax}), {(args.precond or cfg.precond).upper()}, "
            f"FD JVP, GMRES rtol {cfg.gmres_rtol:g} / Newton {cfg.newton_rtol:g}, restart {cfg.restart}")


# --------------------------------------------------------------------------------
# CPU oracle sample (cpu_baseline and --impl reference)

def stage_solves_per_step(q, kmax):
    s = {4: 2, 6: 3, 8: 4}[q]            # stages of HBPC(q, .) (App. A)
    return (s - 1) * (kmax + 1)


def oracle_sample(cfg_name):
    """First predictor stage solve (with its BJ_ext build) of the config's first
    step on a 4x4-element periodic window of its mesh centred in the domain
    (same h, N, equation, dt, tolerances).  Returns (seconds, cpu_seconds,
    description, scale) with steps/s of the full workload ~= 1 / (seconds * scale),
    scale = stage solves per step x (elements / 16)."""
    import numpy as np  # noqa: F401
    from oracle import basis, dgsem, implicit, physics
    from paper_2109_04804_b200 import configs, inputs
    cfg = get_config(cfg_name)
    ic = IC_CASE.get(cfg_name, cfg_name)
    hx = (cfg.bounds[1] - cfg.bounds[0]) / cfg.nx
    hy = (cfg.bounds[3] - cfg.bounds[2]) / cfg.ny
    cx, cy = 0.5 * (cfg.bounds[0] + cfg.bounds[1]), 0.5 * (cfg.bounds[2] + cfg.bounds[3])
    nw = 4 if cfg.dim == 2 else 2
    eq = physics.Equation(cfg.equation, mu=cfg.mu, dim=cfg.dim)
    if cfg.dim == 3:
        cz = 0.5 * (cfg.bounds[4] + cfg.bounds[5])
        hz = (cfg.bounds[5] - cfg.bounds[4]) / cfg.nz
        me = dgsem.Mesh(3, nw, nw, cx - nw * hx / 2, cx + nw * hx / 2, cy - nw * hy / 2, cy + nw * hy / 2,
                        nz=nw, zmin=cz - nw * hz / 2, zmax=cz + nw * hz / 2)
    else:
        me = dgsem.Mesh(2, nw, nw, cx - nw * hx / 2, cx + nw * hx / 2, cy - nw * hy / 2, cy + nw * hy / 2)
    d = dgsem.Disc(basis.build_basis(cfg.N, "gll"), me, eq)
    W0 = inputs.initial_state(ic, d.node_coords(), noise=cfg.noise)
    if cfg.dt > 0:
        dt = cfg.dt
    else:
        if cfg.dim == 3:
            fm = dgsem.Mesh(3, cfg.nx, cfg.ny, *cfg.bounds[:4], nz=cfg.nz, zmin=cfg.bounds[4], zmax=cfg.bounds[5])
        else:
            fm = dgsem.Mesh(2, cfg.nx, cfg.ny, *cfg.bounds)
        full = dgsem.Disc(d.basis, fm, eq)
        dt = configs.cfl_dt(cfg, inputs.initial_state(ic, full.node_coords()))
    c = {4: 1.0, 6: 0.5, 8: 1.0 / 3.0}[cfg.q]          # first stage spacing of App. A
    a1, a2 = c / 2, c * c / 6
    t0, c0 = time.perf_counter(), time.process_time()
    opts = implicit.NewtonOpts(rtol=cfg.newton_rtol, gmres_rtol=cfg.gmres_rtol, restart=cfg.restart)
    R1 = dgsem.rhs1(d, W0)
    _, R2 = dgsem.rhs12(d, W0, R1)
    b = W0 + a1 * dt * R1 + a2 * dt * dt / 2 * R2
    pc = implicit.BJExt(d, W0, a1, a2, dt)
    implicit.newton_solve(d, a1, a2, dt, b, W0, opts, pc)
    sec, cpu = time.perf_counter() - t0, time.process_time() - c0
    k = stage_solves_per_step(cfg.q, cfg.kmax)
    nwin = nw ** cfg.dim
    scale = k * cfg.n_elem / nwin
    desc = (f"oracle (numpy, fp64): first predictor stage solve (BJ_ext build + Newton-GMRES) of {cfg_name} step 1 "
            f"on a {'x'.join([str(nw)] * cfg.dim)}-element periodic window of {cfg_name}'s mesh (same h, N={cfg.N}, "
            f"dt, tolerances), timed end to end; steps/s = 1/(t x {k} stage solves x {cfg.n_elem // nwin} element ratio)")
    return sec, cpu, desc, scale


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = get_config(args.config)
    times, cpus = [], []
    desc, scale = "", 1.0
    for s in range(args.warmup + args.steps):
        sec, cpu, desc, scale = oracle_sample(args.config)
        if s >= args.warmup:
            times.append(sec)
            cpus.append(cpu)
    t = sum(times) / len(times)
    cores = round(sum(cpus) / sum(times), 2)
    val = 1.0 / (t * scale)
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
            "ms_per_step_note": "wall time of one sample step (value = 1 / (sample seconds x scale))",
            "value_scale": scale, "higher_is_better": True, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(cfg, args), "sample": desc},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc,
                             "cores_note": "process CPU time / wall time of the samples",
                             "host_cpus": os.cpu_count()},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------
# clocks sampler

class Clocks:
    def __init__(self, device):
        self.samples = []
        self.device = device
        self._stop = threading.Event()
        self._th = None

    def start(self):
        self._th = threading.Thread(target=self._run, daemon=True)
        self._th.start()

    def _run(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            hdl = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(hdl, pynvml.NVML_CLOCK_SM)
            while not self._stop.is_set():
                mhz = pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_SM)
                reasons = pynvml.nvmlDeviceGetCurrentClocksEventReasons(hdl)
                util = pynvml.nvmlDeviceGetUtilizationRates(hdl).gpu
                self.samples.append((mhz, reasons, util))
                time.sleep(0.2)
        except Exception as e:  # pragma: no cover
            self.error = str(e)

    def stop(self):
        self._stop.set()
        if self._th:
            self._th.join(timeout=2)
        names = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
                 0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle"}
        loaded = [s for s in self.samples if s[2] > 10] or self.samples
        mhz = sorted(s[0] for s in loaded)
        reasons = set()
        for s in loaded:
            for bit, nm in names.items():
                if s[1] & bit and nm != "gpu_idle":
                    reasons.add(nm)
        return {"sm_mhz": mhz[len(mhz) // 2] if mhz else None,
                "sm_max_mhz": getattr(self, "max_mhz", None), "reasons": sorted(reasons),
                "samples": len(self.samples)}


# --------------------------------------------------------------------------------
# our arm

def local_initial_state(case, cfg, ctx, weak, rank):
    """The rank's block of the config's initial state (layout L).  Strong
    scaling: the global field's block, with the C3 noise drawn once for the
    whole global mesh in global layout order (same numbers as on 1 GPU).
    Weak scaling: this rank's copy of the config tile, noise stream rank."""
    import numpy as np
    from paper_2109_04804_b200 import inputs
    coords = ctx.node_coords()
    if weak:
        coords = inputs.tile_coords(coords, cfg.bounds)
        W = inputs.initial_state(case, coords, noise=cfg.noise, stream=rank)
        Wc = inputs.initial_state(case, coords)
        return W, Wc
    Wc = inputs.initial_state(case, coords)
    W = Wc
    if cfg.noise:
        rng = np.random.default_rng(inputs.MASTER_SEED + inputs.CASE_INDEX[case])
        full = rng.uniform(-cfg.noise, cfg.noise, size=cfg.n).reshape(cfg.ny, cfg.nx, cfg.m)
        blk = full[ctx.ey0:ctx.ey0 + ctx.ny_local, ctx.ex0:ctx.ex0 + ctx.nx_local].reshape(-1)
        W = Wc + blk
    return W, Wc


def global_dt(cfg, Wc_local, use_dist):
    """Element-CFL dt (reading R14) of the global discrete IC (before noise): the
    rule is a max over nodes, so each rank evaluates its block and the ranks take
    the max wave-speed sum (max all-reduce); identical on every rank."""
    import torch
    import torch.distributed as dist
    from paper_2109_04804_b200 import configs
    dt = configs.cfl_dt(cfg, Wc_local)
    if use_dist:
        t = torch.tensor([1.0 / dt], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = 1.0 / float(t.item())
    return dt


def memory_plan(cfg, world, weak, batch, restart, sstep):
    """Device bytes per rank of the library's resident arrays (DESIGN.md 5 / 8): BJ_ext blocks S
    (plus the stored K_i for Navier-Stokes), the Krylov bases (restart + 1 vectors of 2n per
    concurrently solved stage system; a restart above 64 is counted as 64: the basis grows on
    demand and the configs' solves stay below), the Newton workspaces, the stage store (3 arrays
    per stage, two sweeps) and the Gauss-Jordan chunk (<= 1 GiB)."""
    n_el = cfg.n_elem if weak else cfg.n_elem // world
    m = cfg.m
    n = n_el * m
    stages = {4: 2, 6: 3, 8: 4}[cfg.q]
    systems = (stages - 1) if batch and cfg.kmax > 0 else 1
    s_bytes = n_el * m * m * 8 * (2 if cfg.equation == "navier_stokes" else 1)
    krylov = systems * (restart + 1) * 2 * n * 8        # grown on demand up to restart + 1 vectors
    work = systems * (6 * 2 * n + n + 2 * n) * 8
    store = 2 * stages * 3 * n * 8
    total = s_bytes + krylov + work + store + min(1 << 30, m * m * 8 * n_el)
    return {"S_GB": round(s_bytes / 1e9, 1), "krylov_GB": round(krylov / 1e9, 1),
            "workspace_GB": round(work / 1e9, 1), "stage_store_GB": round(store / 1e9, 1),
            "total_GB": round(total / 1e9, 1), "lockstep_systems": systems}


def relaunch_under_torchrun(args):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2109_04804_b200 import configs, hbpdc, inputs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench: WORLD_SIZE={world} but --gpus {args.gpus}")
    if torch.cuda.device_count() < world:
        raise SystemExit(f"bench: --gpus {world} but only {torch.cuda.device_count()} CUDA devices")
    torch.cuda.set_device(local)
    # one dedicated stream for torch and the library (no legacy-default-stream syncs)
    torch.cuda.set_stream(torch.cuda.Stream(device=local))
    use_dist = world > 1 or ("MASTER_ADDR" in os.environ and "RANK" in os.environ)
    if use_dist:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    case = args.config
    cfg = get_config(case)
    if cfg.dim == 3 and world > 1:
        raise SystemExit("bench: the 3D configuration runs on one GPU")
    scaling = args.scaling or ("weak" if case == "C3" else "strong")
    weak = scaling == "weak"
    px, py = PARTS.get(world, (world, 1))
    kw = {}
    if world > 1 or args.self_halo:
        nid = [hbpdc.nccl_unique_id() if rank == 0 else None]
        if use_dist:
            dist.broadcast_object_list(nid, src=0)
        kw = dict(rank=rank, nranks=world, px=px, py=py, comm="nccl", nccl_id=nid[0],
                  force_halo=bool(args.self_halo))
        if weak:
            # one copy of the config's mesh per GPU: a (nx px) x (ny py) tiling
            kw.update(nx=cfg.nx * px, ny=cfg.ny * py,
                      bounds=(cfg.bounds[0], cfg.bounds[0] + px * (cfg.bounds[1] - cfg.bounds[0]),
                              cfg.bounds[2], cfg.bounds[2] + py * (cfg.bounds[3] - cfg.bounds[2])))
    if args.precond:
        kw["precond"] = args.precond
    if args.nodes != "gll" or args.flux != "llf":
        kw.update(nodes=args.nodes, flux=args.flux)      # the paper's own discretisation choices (NEXT-3)
    # memory plan: the lock-step corrector workspaces (NEXT-1) need (s-1) Krylov bases;
    # C4 on few GPUs has room for one (137 GB of BJ_ext blocks on 1 GPU)
    batch = args.batch_stages
    if batch is None:
        batch = not (case == "C4" and world < 4)
    plan = memory_plan(cfg, world, weak, batch, cfg.restart if cfg.restart <= 64 else 64, args.gmres_sstep)
    free_b, total_b = torch.cuda.mem_get_info(local)
    plan["device_free_GB"] = round(free_b / 1e9, 1)
    if plan["total_GB"] * 1e9 > free_b:
        raise SystemExit(f"bench: memory plan {plan} exceeds the free device memory")
    ctx = hbpdc.context_for(cfg, device=local, gmres_sstep=args.gmres_sstep, batch_stages=batch, **kw)
    W0, Wc = local_initial_state(IC_CASE.get(case, case), cfg, ctx, weak, rank)
    dt = global_dt(cfg, Wc, use_dist)
    stream = ctx.stream
    dev = f"cuda:{local}"
    W = torch.tensor(W0, dtype=torch.float64, device=dev)
    for _ in range(args.warmup):
        ctx.step(dt, W)
    torch.cuda.synchronize()
    W_start = W.clone()
    W_start_h = W_start.cpu().pin_memory()
    if use_dist:
        dist.barrier()
    torch.cuda.synchronize()

    # ---- timed region: K steps, profiling off -----------------------------------
    clocks = Clocks(local)
    clocks.start()
    l0 = hbpdc.launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    stats = []
    ev0.record(stream)
    for _ in range(args.steps):
        stats.append(ctx.step(dt, W))
    ev1.record(stream)
    torch.cuda.synchronize()
    launches = hbpdc.launch_count() - l0
    ck = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if use_dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    units = world if weak else 1                    # config-tile steps per global step
    value = units * args.steps / (ms_max / 1e3)
    n = ctx.n
    n_global = n * world if weak or world > 1 else n

    # ---- e2e: the same K steps from the same state, through the C-ABI with a host buffer
    e2e = None
    if not args.no_e2e:
        Wh = W_start_h.clone().pin_memory().numpy()
        ctx.reset()                                   # the FSAL cache belongs to the device run
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            ctx.step_host(dt, Wh)
        torch.cuda.synchronize()
        te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if use_dist:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": units * args.steps / float(te.item()), "unit": UNIT,
               "h2d_bytes_per_step": n * 8, "d2h_bytes_per_step": n * 8, "steps": args.steps,
               "note": "same K steps from the same start state as value, hbpdc_step_host per step"}

    # ---- profiled pass (per-kernel CUDA events; not part of value) -----------------
    peak, peak_kind = measured_peaks()
    kernels, dom, step_roof, pstats = {}, None, None, []
    if args.profile_steps > 0:
        ctx.reset()
        Wp = W_start.clone()
        ctx.profile(True)
        ev0.record(stream)
        for _ in range(args.profile_steps):
            pstats.append(ctx.step(dt, Wp))
        ev1.record(stream)
        torch.cuda.synchronize()
        pms = ev0.elapsed_time(ev1)
        prof = {name: ctx.profile_read(i) for name, i in hbpdc.Context.PROFILE_IDS.items()}
        ctx.profile(False)
        for k, (nl, kms, kb) in prof.items():
            kernels[k] = {"launches": nl, "ms": round(kms, 3), "share": round(kms / pms, 4),
                          "GBps": round(kb / (kms / 1e3) / 1e9, 1) if kms > 0 and kb > 0 else None}
        dom = max((kv for kv in prof.items() if kv[0] != "build"), key=lambda kv: kv[1][1])
        # step-level roofline: sum over the step's profiled calls of
        # algorithmic bytes / BW, plus the BJ_ext build flops / FP64 peak, over the time
        builds = sum(s["precond_builds"] for s in pstats)
        m = ctx.m
        build_flops = builds * ctx.n_elem * 4.0 * m ** 3      # K^2 (2 m^3) + Gauss-Jordan inverse (2 m^3)
        ideal_ms = sum(kb for k, (nl, kms, kb) in prof.items() if k != "build") / (peak * 1e9) * 1e3 \
            + build_flops / (FP64_PEAK_TFLOPS * 1e12) * 1e3
        covered = sum(kms for kms in (v[1] for v in prof.values()))
        step_roof = {"ideal_ms": round(ideal_ms, 1), "measured_ms": round(pms, 1),
                     "frac": round(ideal_ms / pms, 4), "profiled_share": round(covered / pms, 4),
                     "model": "sum of (algorithmic bytes / measured HBM BW) over the profiled kernels + "
                              f"builds x elements x 4 m^3 / {FP64_PEAK_TFLOPS} TFLOP/s (K^2 + inverse), "
                              "over the profiled steps' device time",
                     "steps": args.profile_steps}

    # ---- kernel micro-timings on the current state (C-ABI calls) ----------------------
    g = torch.Generator(device="cpu").manual_seed(inputs.MASTER_SEED + 200)
    sig = ctx.rhs(W)
    dW = torch.randn(n, generator=g, dtype=torch.float64).to(dev)
    dS = torch.randn(n, generator=g, dtype=torch.float64).to(dev)
    o1, o2 = ctx.empty(), ctx.empty()
    b = W.clone()

    def timeit(fn, reps=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(reps):
            fn()
        ev1.record(stream)
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1) / reps

    jms = timeit(lambda: ctx.jvp(1.0, 1.0, dt, W, sig, dW, dS, mode="fd", out1=o1, out2=o2))
    rms = timeit(lambda: ctx.residual(0.5, 1.0 / 6, dt, b, W, sig, G1=o1, G2=o2))
    # bytes per W-DOF: JVP reads W, sigma, dW, dsigma, writes 2 blocks (48; NS +48 for the
    # lifted gradients); residual reads W, sigma, b, writes 2 blocks (40)
    jb = 48 + (48 if cfg.equation == "navier_stokes" else 0)
    micro = {"jvp_fd": {"dof_applies_per_s": n_global / (jms / 1e3) if not weak else n / (jms / 1e3),
                        "ms": jms, "bytes_per_dof": jb,
                        "GBps_alg": round(jb * n / (jms / 1e3) / 1e9, 1),
                        "frac_hbm": round(jb * n / (jms / 1e3) / 1e9 / peak, 4)},
             "residual": {"ms": rms, "bytes_per_dof": 40 + (48 if cfg.equation == "navier_stokes" else 0),
                          "GBps_alg": round((40 + (48 if cfg.equation == "navier_stokes" else 0)) * n / (rms / 1e3) / 1e9, 1)}}
    micro["residual"]["frac_hbm"] = round(micro["residual"]["GBps_alg"] / peak, 4)
    fp64p = os.path.join(ROOT, "profiles", "ncu_fp64.json")
    if os.path.exists(fp64p):
        f = json.load(open(fp64p)).get(case, {})
        for k in ("jvp_fd", "residual"):
            if k in f:
                micro[k]["fp64_pipe_frac_ncu"] = f[k]

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sec, cpus, desc, scale = oracle_sample(case)
        cpu = {"value": 1.0 / (sec * scale), "unit": UNIT, "cores": round(cpus / sec, 2), "kind": "oracle",
               "sample": desc, "sample_seconds": round(sec, 2),
               "cores_note": "process CPU time / wall time of the sample", "host_cpus": os.cpu_count()}

    roof = None
    if dom is not None:
        dname, (dn, dms, dbytes) = dom
        achieved = dbytes / (dms / 1e3) / 1e9 if dms > 0 else 0.0
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp) and dn:
            ratio = json.load(open(tp)).get(dname)
            if isinstance(ratio, (int, float)):
                traffic = round(dbytes / dn * ratio)
        roof = {"bound": "hbm", "kernel": dname, "achieved": round(achieved, 1), "peak": peak,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
                "traffic": traffic, "launches": dn}

    if rank == 0:
        it = {k: sum(s[k] for s in stats) for k in ("stage_solves", "newton_its", "gmres_its",
                                                      "precond_builds", "jvp_calls", "precond_applies",
                                                      "precond_k_reused")}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(cfg, args), "config": case,
                       "arnoldi": ("DCGS2" if args.gmres_sstep <= 1 else f"s-step s={args.gmres_sstep} (block CGS2)"),
                       "precond": args.precond or cfg.precond, "nodes": args.nodes, "flux": args.flux,
                       "lockstep_correctors": bool(batch),
                       "memory_plan": plan,
                       "dt": dt, "n_dof_per_gpu": n, "n_dof": n_global,
                       "parallelism": (f"{scaling} scaling: element partition {px}x{py} of a "
                                       f"{cfg.nx * (px if weak else 1)}x{cfg.ny * (py if weak else 1)} mesh, "
                                       "NCCL halos + all-reduces") if world > 1 else
                                      ("1 GPU, NCCL self-halo" if args.self_halo else "1 GPU"),
                       "value_unit": ("config-tile steps/s (one copy of the config mesh per GPU)" if weak and world > 1
                                      else "global time steps/s"),
                       "l2": "working set > L2 (BJ_ext blocks + Krylov basis, GBs): no flush needed"},
            "global_steps_per_s": args.steps / (ms_max / 1e3),
            "dof_steps_per_s": n_global * args.steps / (ms_max / 1e3),
            "roofline": roof,
            "step_roofline": step_roof,
            "kernels": kernels,
            "micro": micro,
            "solver": it,
            "clocks": ck,
            "e2e": e2e,
            "gpu_launches": launches,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if use_dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3", choices=["C3", "C4", "C5", "T3"],
                    help="BASELINE config (C3 default, C4, C5) or T3: the paper's 3D case, inviscid (NEXT-4)")
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"],
                    help="N > 1: weak (a config tile per GPU; C3 default) or strong (one mesh; C4/C5 default)")
    ap.add_argument("--profile-steps", type=int, default=1,
                    help="steps of the separate profiled pass (per-kernel table, step roofline); 0 = none")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--batch-stages", type=int, default=None, choices=[0, 1],
                    help="lock-step corrector stages (default: on, except C4 below 4 GPUs: memory)")
    ap.add_argument("--precond", default=None, choices=["bjext", "bjext_h", "none"],
                    help="override the config's preconditioner (default: BJ_ext)")
    ap.add_argument("--gmres-sstep", type=int, default=8,
                    help="Arnoldi schedule: 1 = DCGS2, 2/4/8 = s-step blocks")
    ap.add_argument("--nodes", default="gll", choices=["gll", "gl"],
                    help="DGSEM nodes (configs: GLL; gl = the paper's Gauss-Legendre, NEXT-3)")
    ap.add_argument("--flux", default="llf", choices=["llf", "glf"],
                    help="numerical flux (configs: LLF; glf = the paper's global LF, NEXT-3)")
    ap.add_argument("--self-halo", action="store_true",
                    help="test hook: route the periodic wrap through the NCCL transport (N = 1)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args))
    run_ours(args)


if __name__ == "__main__":
    main()
