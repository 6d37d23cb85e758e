"""Operator micro-timings on a full-size config (CUDA events, median of reps):
FD / EXACT JVP, residual, BJ_ext build, BJ_ext apply.

    python scripts/op_times.py [C3|C4|C5] [reps] [gl]   -> one JSON line (gl: GL nodes + the paper's GLF flux)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2109_04804_b200 import configs, hbpdc, inputs  # noqa: E402


def timed(fn, reps, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    case = sys.argv[1] if len(sys.argv) > 1 else "C3"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    cfg = configs.CONFIGS[case]
    gl = len(sys.argv) > 3 and sys.argv[3] == "gl"
    extra = dict(nodes="gl", flux="glf") if gl else {}
    ctx = hbpdc.context_for(cfg, restart=16, batch_stages=False, **extra)
    coords = ctx.node_coords()
    W0 = inputs.perturbed_state(inputs.initial_state(case, coords, noise=cfg.noise), inputs.MASTER_SEED + 900)
    dt = configs.cfl_dt(cfg, inputs.initial_state(case, coords))
    n = ctx.n
    W = torch.tensor(W0, dtype=torch.float64, device="cuda")
    sig = ctx.rhs(W)
    g = torch.Generator().manual_seed(7)
    dW = torch.randn(n, generator=g, dtype=torch.float64).cuda()
    dS = torch.randn(n, generator=g, dtype=torch.float64).cuda()
    o1, o2 = ctx.empty(), ctx.empty()
    b = W.clone()
    res = {"config": case, "n": n, "nodes": "gl" if gl else "gll", "gl_traces": os.environ.get("HBPDC_GL_TRACES", "1")}
    res["jvp_fd_us"] = 1e3 * timed(lambda: ctx.jvp(0.5, 1 / 6, dt, W, sig, dW, dS, mode="fd", out1=o1, out2=o2), reps)
    res["jvp_exact_us"] = 1e3 * timed(lambda: ctx.jvp(0.5, 1 / 6, dt, W, sig, dW, dS, mode="exact", out1=o1, out2=o2), reps)
    res["residual_us"] = 1e3 * timed(lambda: ctx.residual(0.5, 1 / 6, dt, b, W, sig, G1=o1, G2=o2), reps)
    res["r1_us"] = 1e3 * timed(lambda: ctx.rhs(W, out=o1), reps)
    res["precond_build_ms"] = timed(lambda: ctx.precond_build(0.5, 1 / 6, dt, W), 3, warm=1)
    res["precond_apply_us"] = 1e3 * timed(lambda: ctx.precond_apply(dW, dS, o1, o2), reps)
    jb = 48 + (48 if cfg.equation == "navier_stokes" else 0)
    peak = 6533.5
    res["jvp_fd_frac_hbm"] = jb * n / (res["jvp_fd_us"] * 1e-6) / 1e9 / peak
    res["residual_frac_hbm"] = 40 * n / (res["residual_us"] * 1e-6) / 1e9 / peak
    print(json.dumps(res), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
