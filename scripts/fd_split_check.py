"""Bitwise check of the two-threads-per-node FD JVP (fdsplit.cuh) against the one-thread
op_kernel: run once per HBPDC_FD_SPLIT setting, save the outputs, compare.

    HBPDC_FD_SPLIT=0 python scripts/fd_split_check.py save /tmp/a.npz
    HBPDC_FD_SPLIT=1 python scripts/fd_split_check.py save /tmp/b.npz
    python scripts/fd_split_check.py cmp /tmp/a.npz /tmp/b.npz
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def save(path):
    import torch
    from paper_2109_04804_b200 import configs, hbpdc, inputs
    out = {}
    for case, nx in (("C3", 128), ("C3", 5)):
        cfg = configs.scaled(configs.CONFIGS[case], nx=nx, ny=nx)
        ctx = hbpdc.context_for(cfg, restart=16, batch_stages=False)
        coords = ctx.node_coords()
        W0 = inputs.perturbed_state(inputs.initial_state(case, coords, noise=cfg.noise), inputs.MASTER_SEED + 901)
        dt = configs.cfl_dt(cfg, inputs.initial_state(case, coords))
        W = torch.tensor(W0, dtype=torch.float64, device="cuda")
        sig = ctx.rhs(W)
        g = torch.Generator().manual_seed(11)
        dW = torch.randn(ctx.n, generator=g, dtype=torch.float64).cuda()
        dS = torch.randn(ctx.n, generator=g, dtype=torch.float64).cuda()
        o1, o2 = ctx.empty(), ctx.empty()
        for tag, eps in (("eps", None), ("zero", [0.0, 0.0])):
            ctx.jvp(0.5, 1 / 6, dt, W, sig, dW, dS, mode="fd", out1=o1, out2=o2, eps_override=eps)
            torch.cuda.synchronize()
            out[f"{case}_{nx}_{tag}_1"] = o1.cpu().numpy().copy()
            out[f"{case}_{nx}_{tag}_2"] = o2.cpu().numpy().copy()
        ctx.close()
    np.savez(path, **out)


def cmp(a, b):
    A, B = np.load(a), np.load(b)
    bad = 0
    for k in A.files:
        same = np.array_equal(A[k].view(np.uint64), B[k].view(np.uint64))
        rel = float(np.linalg.norm(A[k] - B[k]) / max(np.linalg.norm(A[k]), 1e-300))
        print(f"{k}: bitwise {same}, rel {rel:.3e}")
        bad += not same
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    if sys.argv[1] == "save":
        save(sys.argv[2])
    else:
        cmp(sys.argv[2], sys.argv[3])
