"""Launch the C3 operator kernels a few times (for ncu captures / timing):
FD JVP, exact JVP, residual, K-apply, on the C3 perturbed state.

    python scripts/jvp_only.py [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2109_04804_b200 import configs, hbpdc, inputs  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    cfg = configs.CONFIGS["C3"]
    ctx = hbpdc.context_for(cfg, restart=30)
    coords = ctx.node_coords()
    W0 = inputs.perturbed_state(inputs.initial_state("C3", coords, noise=cfg.noise), inputs.MASTER_SEED + 900)
    dt = configs.cfl_dt(cfg, inputs.initial_state("C3", coords))
    n = ctx.n
    W = torch.tensor(W0, dtype=torch.float64, device="cuda")
    sig = ctx.rhs(W)
    g = torch.Generator().manual_seed(7)
    dW = torch.randn(n, generator=g, dtype=torch.float64).cuda()
    dS = torch.randn(n, generator=g, dtype=torch.float64).cuda()
    o1, o2 = ctx.empty(), ctx.empty()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    res = {}
    for mode in ("fd", "exact"):
        for _ in range(2):
            ctx.jvp(1.0, 1.0, dt, W, sig, dW, dS, mode=mode, out1=o1, out2=o2)
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(reps):
            ctx.jvp(1.0, 1.0, dt, W, sig, dW, dS, mode=mode, out1=o1, out2=o2)
        ev1.record()
        torch.cuda.synchronize()
        res["jvp_" + mode] = ev0.elapsed_time(ev1) / reps
    b = W.clone()
    ev0.record()
    for _ in range(reps):
        ctx.residual(1.0, 1.0, dt, b, W, sig, G1=o1, G2=o2)
    ev1.record()
    torch.cuda.synchronize()
    res["residual"] = ev0.elapsed_time(ev1) / reps
    ctx.precond_build(1.0, 1.0, dt, W)
    for _ in range(2):
        ctx.precond_apply(dW, dS, o1, o2)
    torch.cuda.synchronize()
    ev0.record()
    for _ in range(reps):
        ctx.precond_apply(dW, dS, o1, o2)
    ev1.record()
    torch.cuda.synchronize()
    res["precond_apply"] = ev0.elapsed_time(ev1) / reps
    alg = {"jvp_fd": 48, "jvp_exact": 48, "residual": 40}
    for k, ms in res.items():
        gbs = alg[k] * n / (ms * 1e-3) / 1e9 if k in alg else None
        print(f"{k:14s} {ms * 1e3:9.1f} us" + (f"  {gbs:7.0f} GB/s alg" if gbs else ""))
    ctx.close()


if __name__ == "__main__":
    main()
