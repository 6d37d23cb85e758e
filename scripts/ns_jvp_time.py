"""C5 (Navier-Stokes, BR1) operator timings: FD / EXACT JVP and R1 on the full C5 mesh.

    HBPDC_LIB=... python scripts/ns_jvp_time.py [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2109_04804_b200 import configs, hbpdc, inputs  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    cfg = configs.CONFIGS["C5"]
    ctx = hbpdc.context_for(cfg, restart=30)
    coords = ctx.node_coords()
    W = torch.tensor(inputs.perturbed_state(inputs.initial_state("C5", coords, noise=cfg.noise), 901),
                     dtype=torch.float64, device="cuda")
    sig = ctx.rhs(W)
    g = torch.Generator().manual_seed(7)
    dW = torch.randn(ctx.n, generator=g, dtype=torch.float64).cuda()
    dS = torch.randn(ctx.n, generator=g, dtype=torch.float64).cuda()
    o1, o2 = ctx.empty(), ctx.empty()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for mode in ("fd", "exact"):
        for _ in range(2):
            ctx.jvp(0.5, 0.2, 1e-3, W, sig, dW, dS, mode=mode, out1=o1, out2=o2)
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(reps):
            ctx.jvp(0.5, 0.2, 1e-3, W, sig, dW, dS, mode=mode, out1=o1, out2=o2)
        ev1.record()
        torch.cuda.synchronize()
        print(f"C5 jvp_{mode:6s} {ev0.elapsed_time(ev1) / reps * 1e3:9.1f} us (incl. lifting)")
    ctx.close()


if __name__ == "__main__":
    main()
