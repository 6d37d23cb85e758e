"""NEXT-3: temporal convergence study on the GPU path (the paper's EOC setups,
P:694-817: fig:LinAdv_convtest_*, fig:Euler_convtest_*), qualitative.

HBPC(q, k_max) for q = 4, 6, 8 with k_max = q - 4 (reading R16) and with
k_max = 0 (predictor only: order 4), run to T = 0.8 on 32^2
elements, N = 7 (spatial error far below the temporal one) with halved time
steps; the L2 error against the exact solution gives the experimental order
EOC = log2(e(dt) / e(dt/2)), expected min(4 + k_max, q).

  * linear advection, a = (0.3, 0.3), [-1, 1]^2: w = sin(pi (x - 0.3 t)) sin(pi (y - 0.3 t));
  * Euler density wave (an exact solution): rho = 1 + 0.3 sin(pi (x + y - 0.6 t)),
    v = (0.3, 0.3), p = 1, on [-1, 1]^2 (reading: sin(pi x) of the vector
    argument as the sum of its components).
Tolerances as the paper's convergence runs: GMRES 1e-5, Newton 1e-12.

    python scripts/eoc_study.py > profiles/<round>/eoc_study.md
    python scripts/eoc_study.py --nodes gl --flux glf > profiles/<round>/eoc_study_gl.md
      (the paper's own discretisation: Gauss-Legendre nodes P:176, global LF flux P:197-201)
"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2109_04804_b200 import hbpdc, inputs  # noqa: E402

T_END = 0.8
A = 0.3


def exact(kind, X, Y, t):
    if kind == "advection":
        return [np.sin(np.pi * (X - A * t)) * np.sin(np.pi * (Y - A * t))]
    rho = 1.0 + 0.3 * np.sin(np.pi * (X + Y - 2 * A * t))
    p = np.ones_like(rho)
    return [rho, rho * A, rho * A, p / 0.4 + 0.5 * rho * 2 * A * A]


def l2_error(kind, ctx, W, t):
    X, Y = ctx.node_coords()
    ref = inputs.layout(exact(kind, X, Y, t), 2)
    return float(np.linalg.norm(W - ref) / np.linalg.norm(ref))


NODES, FLUX = "gll", "llf"


def run(kind, q, kmax, nsteps, N=7, ne=32):
    ctx = hbpdc.Context(dim=2, equation=kind, N=N, nx=ne, ny=ne, bounds=(-1.0, 1.0, -1.0, 1.0),
                        a=(A, A), q=q, kmax=kmax, newton_rtol=1e-12, gmres_rtol=1e-5, restart=700,
                        max_krylov=7000, precond="bjext", gmres_sstep=1, nodes=NODES, flux=FLUX)
    X, Y = ctx.node_coords()
    W = torch.tensor(inputs.layout(exact(kind, X, Y, 0.0), 2), dtype=torch.float64, device="cuda")
    dt = T_END / nsteps
    for _ in range(nsteps):
        ctx.step(dt, W)
    torch.cuda.synchronize()
    err = l2_error(kind, ctx, W.cpu().numpy(), T_END)
    ctx.close()
    return err


def main():
    global NODES, FLUX
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--nodes", default="gll", choices=["gll", "gl"])
    ap.add_argument("--flux", default="llf", choices=["llf", "glf"])
    args = ap.parse_args()
    NODES, FLUX = args.nodes, args.flux
    print("# NEXT-3: temporal EOC of HBPC(q, k_max) on the GPU (`scripts/eoc_study.py`)\n")
    print(f"T = {T_END}, 32^2 elements, N = 7 ({NODES.upper()} nodes, {FLUX.upper()} flux), BJ_ext, GMRES 1e-5 / "
          "Newton 1e-12; relative L2 error at the nodes vs the exact solution; EOC = log2 of successive "
          "error ratios.\n")
    schemes = [(4, 0), (6, 2), (6, 0), (8, 4), (8, 0)]
    steps = {4: [4, 8, 16, 32], 6: [2, 4, 8, 16], 8: [2, 4, 8]}
    for kind in ("advection", "euler"):
        print(f"## {kind}\n")
        print("| scheme | expected order | steps: error (EOC) |")
        print("|---|---|---|")
        for q, kmax in schemes:
            errs = []
            cells = []
            for ns in steps[q]:
                e = run(kind, q, kmax, ns)
                eoc = "" if not errs else f" ({math.log2(errs[-1] / e):.2f})"
                errs.append(e)
                cells.append(f"{ns}: {e:.2e}{eoc}")
            print(f"| HBPC({q},{kmax}) | {min(4 + kmax, q)} | " + ", ".join(cells) + " |")
            sys.stdout.flush()
        print()


if __name__ == "__main__":
    main()
