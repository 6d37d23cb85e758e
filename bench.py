"""Benchmark: HBPC(q, k_max) / DGSEM time steps on B200 (arXiv 2109.04804).

One bench "step" is one HBPC(8,4) time step (Alg. 1) of config C3
(2D Euler isentropic vortex, 128x128 elements, N=7, GLL, LLF, BJ_ext, FD JVP,
Newton-GMRES rtol 1e-10) -- every row of SURVEY 8(a): residual, FD JVP,
BJ_ext build + apply, Arnoldi, Newton updates, stage combinations.
Prints ONE JSON line (rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the CPU oracle (oracle/, test infrastructure) on a
bounded sample of the same workload, scaled to steps/s.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "HBPDC steps/s"
UNIT = "steps/s"
CONFIG = "C3"


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


# --------------------------------------------------------------------------------
# CPU oracle sample (cpu_baseline and --impl reference)

def oracle_sample():
    """First predictor stage solve (with its BJ_ext build) of C3's first step on
    a 4x4-element periodic window of C3's mesh centred on the vortex (same h,
    N=7, dt, tolerances).  Returns (seconds, description, scale): steps/s of
    the full workload ~= 1 / (seconds * scale), scale = 15 stage solves per
    HBPC(8,4) step x (16384 / 16) elements."""
    import numpy as np
    from oracle import basis, dgsem, implicit, physics
    from paper_2109_04804_b200 import configs, inputs
    cfg = configs.CONFIGS[CONFIG]
    h = (cfg.bounds[1] - cfg.bounds[0]) / cfg.nx
    nw = 4
    half = nw * h / 2
    d = dgsem.Disc(basis.build_basis(cfg.N, "gll"), dgsem.Mesh(2, nw, nw, -half, half, -half, half),
                   physics.Equation("euler"))
    W0 = inputs.initial_state(CONFIG, d.node_coords(), noise=cfg.noise)
    # dt of the full config: element CFL 1 on the full discrete IC (reading R15)
    full = dgsem.Disc(d.basis, dgsem.Mesh(2, cfg.nx, cfg.ny, *cfg.bounds), d.eq)
    dt = configs.cfl_dt(cfg, inputs.initial_state(CONFIG, full.node_coords()))
    c = 1.0 / 3.0
    a1, a2 = c / 2, c * c / 6
    t0 = time.perf_counter()
    opts = implicit.NewtonOpts(rtol=cfg.newton_rtol, gmres_rtol=cfg.gmres_rtol)
    R1 = dgsem.rhs1(d, W0)
    _, R2 = dgsem.rhs12(d, W0, R1)
    b = W0 + a1 * dt * R1 + a2 * dt * dt / 2 * R2
    pc = implicit.BJExt(d, W0, a1, a2, dt)
    implicit.newton_solve(d, a1, a2, dt, b, W0, opts, pc)
    sec = time.perf_counter() - t0
    scale = 15 * (cfg.nx * cfg.ny) / (nw * nw)
    desc = ("oracle: first predictor stage solve (BJ_ext build + Newton-GMRES) of C3 step 1 on a 4x4-element "
            "periodic window of C3's mesh (same h, N=7, dt, tolerances); steps/s = 1/(t x 15 stage solves x "
            "1024 element ratio)")
    return sec, desc, scale


def cpu_cores():
    try:
        from threadpoolctl import threadpool_info
        n = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        n = 1
    return n


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    times = []
    desc, scale = "", 1.0
    for s in range(args.warmup + args.steps):
        sec, desc, scale = oracle_sample()
        if s >= args.warmup:
            times.append(sec)
    t = sum(times) / len(times)
    val = 1.0 / (t * scale)
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * scale * 1e3,
            "higher_is_better": True, "dtype": "f64", "data": "synthetic",
            "config": {"workload": CONFIG + " (sampled)", "sample": desc},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cpu_cores(), "kind": "oracle",
                             "sample": desc},
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

def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2109_04804_b200 import configs, hbpdc, inputs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    # one dedicated stream for torch and the library (no legacy-default-stream syncs)
    torch.cuda.set_stream(torch.cuda.Stream(device=local))
    # torchrun sets MASTER_ADDR/RANK even for one process: the distributed
    # plumbing then runs at N = 1 too (with --self-halo it is fully exercised)
    use_dist = world > 1 or ("MASTER_ADDR" in os.environ and "RANK" in os.environ)
    if use_dist:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = configs.CONFIGS[CONFIG]
    # N > 1: ONE global problem, C3's 128x128-element tile repeated on a px x py
    # rank grid (a (128 px) x (128 py) mesh of the periodic vortex field, same h,
    # N, dt and tolerances), element-partitioned with one 128x128 block per GPU:
    # face-trace halos and Krylov/norm all-reduces over NCCL.
    # Per-GPU work is C3's: weak scaling.  DESIGN.md "Multi-GPU".
    px, py = {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (4, 2)}.get(world, (world, 1))
    kw = {}
    if world > 1 or args.self_halo:
        nid = [hbpdc.nccl_unique_id() if rank == 0 else None]
        if use_dist:
            dist.broadcast_object_list(nid, src=0)
        kw = dict(nx=cfg.nx * px, ny=cfg.ny * py,
                  bounds=(cfg.bounds[0], cfg.bounds[0] + px * (cfg.bounds[1] - cfg.bounds[0]),
                          cfg.bounds[2], cfg.bounds[2] + py * (cfg.bounds[3] - cfg.bounds[2])),
                  rank=rank, nranks=world, px=px, py=py, comm="nccl", nccl_id=nid[0],
                  force_halo=bool(args.self_halo))
    if args.precond:
        kw["precond"] = args.precond
    if args.nodes != "gll" or args.flux != "llf":
        kw.update(nodes=args.nodes, flux=args.flux)      # the paper's own discretisation choices (NEXT-3)
    ctx = hbpdc.context_for(cfg, device=local, gmres_sstep=args.gmres_sstep, **kw)
    coords = inputs.tile_coords(ctx.node_coords(), cfg.bounds)
    W0 = inputs.initial_state(CONFIG, coords, noise=cfg.noise, stream=rank)
    dt = configs.cfl_dt(cfg, inputs.initial_state(CONFIG, coords))
    stream = ctx.stream
    W = torch.tensor(W0, dtype=torch.float64, device=f"cuda:{local}")
    for _ in range(args.warmup):
        ctx.step(dt, W)
    torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    clocks = Clocks(local)
    clocks.start()
    ctx.profile(True)
    l0 = hbpdc.launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    stats = []
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(args.steps):
        stats.append(ctx.step(dt, W))
    ev1.record(stream)
    torch.cuda.synchronize()
    launches = hbpdc.launch_count() - l0
    ms = ev0.elapsed_time(ev1)
    prof = {name: ctx.profile_read(i) for name, i in hbpdc.Context.PROFILE_IDS.items()}
    ctx.profile(False)
    ck = clocks.stop()
    t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{local}")
    if use_dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * args.steps / (ms_max / 1e3)

    # dominant kernel + roofline (algorithmic bytes / CUDA-event time)
    peak, peak_kind = measured_peaks()
    dom = max(prof.items(), key=lambda kv: kv[1][1])
    dname, (dn, dms, dbytes) = dom
    achieved = dbytes / (dms / 1e3) / 1e9 if dms > 0 else 0.0
    kernels = {k: {"launches": v[0], "ms": round(v[1], 3), "share": round(v[1] / ms, 4),
                   "GBps": round(v[2] / (v[1] / 1e3) / 1e9, 1) if v[1] > 0 else None}
               for k, v in prof.items()}
    # DRAM traffic per launch: average algorithmic bytes x the DRAM/algorithmic
    # ratio measured by ncu for this kernel (profiles/ncu_traffic.json)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp) and dn:
        ratio = json.load(open(tp)).get(dname)
        if isinstance(ratio, (int, float)):
            traffic = round(dbytes / dn * ratio)

    # matrix-free FD JVP throughput on the C3 state (second headline of the metric)
    n = ctx.n
    g = torch.Generator(device="cpu").manual_seed(inputs.MASTER_SEED + 200)
    sig = ctx.rhs(W)
    dW = torch.randn(n, generator=g, dtype=torch.float64).to(W.device)
    dS = torch.randn(n, generator=g, dtype=torch.float64).to(W.device)
    o1, o2 = ctx.empty(), ctx.empty()
    for _ in range(3):
        ctx.jvp(1.0, 1.0, dt, W, sig, dW, dS, mode="fd", out1=o1, out2=o2)
    reps = 20
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(reps):
        ctx.jvp(1.0, 1.0, dt, W, sig, dW, dS, mode="fd", out1=o1, out2=o2)
    ev1.record(stream)
    torch.cuda.synchronize()
    jms = ev0.elapsed_time(ev1) / reps
    jvp_rate = n / (jms / 1e3)
    jvp_gbps = 48.0 * n / (jms / 1e3) / 1e9

    # end to end through the C-ABI with HOST buffers (H2D + step + D2H per step)
    e2e = None
    if not args.no_e2e:
        Wh = torch.tensor(W0, dtype=torch.float64).pin_memory()
        ctx.reset()
        ctx.step_host(dt, Wh.numpy())                 # warm
        torch.cuda.synchronize()
        if use_dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            ctx.step_host(dt, Wh.numpy())
        te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=f"cuda:{local}")
        if use_dist:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": world * args.e2e_steps / float(te.item()), "unit": UNIT,
               "h2d_bytes_per_step": n * 8, "d2h_bytes_per_step": n * 8, "steps": args.e2e_steps}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sec, desc, scale = oracle_sample()
        cpu = {"value": 1.0 / (sec * scale), "unit": UNIT, "cores": cpu_cores(), "kind": "oracle",
               "sample": desc, "sample_seconds": round(sec, 2)}

    if rank == 0:
        it = {k: sum(s[k] for s in stats) for k in ("stage_solves", "newton_its", "gmres_its",
                                                      "precond_builds", "jvp_calls", "precond_applies")}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C3: 2D Euler isentropic vortex (beta=5, mean (1,1)) + seeded U[-1e-6,1e-6) "
                                   f"noise, [-5,5]^2 periodic, 128x128 elements, N=7 {args.nodes.upper()}, "
                                   f"{args.flux.upper()}, HBPC(8,4), "
                                   "BJ_ext, FD JVP, Newton/GMRES rtol 1e-10, restart 700",
                       "arnoldi": ("DCGS2" if args.gmres_sstep <= 1 else f"s-step s={args.gmres_sstep} (block CGS2)"),
                       "precond": args.precond or cfg.precond,
                       "nodes": args.nodes, "flux": args.flux,
                       "dt": dt, "n_dof_per_gpu": n, "n_dof": n * world,
                       "parallelism": (f"element partition {px}x{py} of a {cfg.nx * px}x{cfg.ny * py} mesh "
                                       "(C3 tile per GPU), NCCL halos + all-reduces") if world > 1 else
                                      ("1 GPU, NCCL self-halo" if args.self_halo else "1 GPU"),
                       "l2": "working set > L2 (BJ_ext blocks 8.6 GB, Krylov basis up to 47 GB)"},
            "roofline": {"bound": "hbm", "kernel": dname, "achieved": round(achieved, 1), "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": traffic, "launches": dn},
            "kernels": kernels,
            "jvp": {"dof_applies_per_s": jvp_rate, "ms": jms, "GBps_alg": round(jvp_gbps, 1),
                    "frac": round(jvp_gbps / peak, 4), "bytes_per_dof": 48},
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
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--precond", default=None, choices=["bjext", "bjext_h", "none"],
                    help="override the config's preconditioner (default: C3's BJ_ext)")
    ap.add_argument("--gmres-sstep", type=int, default=8,
                    help="Arnoldi schedule: 1 = DCGS2, 2/4/8 = s-step blocks")
    ap.add_argument("--nodes", default="gll", choices=["gll", "gl"],
                    help="DGSEM nodes (C3: GLL; gl = the paper's Gauss-Legendre, NEXT-3)")
    ap.add_argument("--flux", default="llf", choices=["llf", "glf"],
                    help="numerical flux (C3: LLF; glf = the paper's global LF, NEXT-3)")
    ap.add_argument("--self-halo", action="store_true",
                    help="test hook: route the periodic wrap through the NCCL transport (N = 1)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
