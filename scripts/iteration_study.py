"""NEXT-2: qualitative reproduction of the paper's linear-solver iteration
studies (fig:LinAdv_CondConv, fig:Euler_Hessian, fig:Euler_eps)
on the GPU path: GMRES iterations needed for one time step of the HBPC(4,0)
predictor (one implicit stage solve) as a function of the time
step, for the preconditioners BJ_ext, BJ^H_ext and none.

Setups after P:349-351 and P:386-402 (readings in DESIGN.md):
  * linear advection, a = (0.3, 0.3), [-1, 1]^2, 16^2 elements, N = 5,
    w0 = sin(pi x) sin(pi y);
  * Euler (gamma 1.4), same mesh, rho = 1 + 0.3 sin(pi (x + y)), v = (0.3, 0.3),
    p = 1; LLF flux (reading R3) at eps = 1, and the paper's own setting of
    fig:Euler_eps: global LF flux Lambda = diag(1/eps,1,1,1/eps) at
    reference Mach numbers eps = 1, 0.1, 0.01.
Tolerances as the paper's studies: GMRES 1e-3, Newton 1e-8;
restart 700, at most 7000 iterations per Newton step.

    python scripts/iteration_study.py > profiles/<round>/iteration_study.md
"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2109_04804_b200 import hbpdc, inputs  # noqa: E402


def initial(kind, X, Y, mach=1.0):
    """Conserved variables at the nodes (arrays shaped like X: (ny, nx, p, p));
    Euler energy E = p/(gamma-1) + eps^2/2 rho |v|^2."""
    if kind == "advection":
        return [np.sin(np.pi * X) * np.sin(np.pi * Y)]
    rho = 1.0 + 0.3 * np.sin(np.pi * (X + Y))
    u = v = 0.3
    p = np.ones_like(rho)
    E = p / 0.4 + 0.5 * mach * mach * rho * (u * u + v * v)
    return [rho, rho * u, rho * v, E]


def gmres_iterations(kind, precond, dt, N=5, ne=16, mach=1.0, flux="llf"):
    schur = precond.startswith("schur")
    pc = {"schur_bj": "bjext_h", "schur": "none"}.get(precond, precond)
    ctx = hbpdc.Context(dim=2, equation=kind, N=N, nx=ne, ny=ne, bounds=(-1.0, 1.0, -1.0, 1.0),
                        a=(0.3, 0.3), q=4, kmax=0, newton_rtol=1e-8, gmres_rtol=1e-3, restart=700,
                        max_krylov=7000, precond=pc, mach=mach, flux=flux, schur=schur)
    X, Y = ctx.node_coords()
    W = torch.tensor(inputs.layout(initial(kind, X, Y, mach), 2), dtype=torch.float64, device="cuda")
    try:
        st = ctx.step(dt, W)
        return st["gmres_its"], st["newton_its"]
    except RuntimeError as e:                         # no convergence within 7000 iterations
        return None, str(e).split("\n")[0][:60]
    finally:
        ctx.close()


def slope(dts, its):
    pts = [(math.log(d), math.log(i)) for d, i in zip(dts, its) if i]
    if len(pts) < 2:
        return float("nan")
    x, y = np.array(pts).T
    return float(np.polyfit(x, y, 1)[0])


def main():
    dts = [10 ** e for e in np.linspace(-3.0, -0.5, 6)]
    print("# NEXT-2: GMRES iterations for one HBPC(4,0) step vs dt (GPU, `scripts/iteration_study.py`)\n")
    print("GMRES rtol 1e-3, Newton rtol 1e-8 (P:358), restart 700; 16^2 elements, N = 5, [-1, 1]^2.\n")
    cases = [("advection", 1.0, "llf"), ("euler", 1.0, "llf"),
             ("euler", 1.0, "glf"), ("euler", 0.1, "glf"), ("euler", 0.01, "glf")]
    for kind, mach, flux in cases:
        title = kind if kind == "advection" else f"euler, reference Mach eps = {mach}, flux {flux.upper()}"
        print(f"## {title}\n")
        names = ("BJ_ext", "BJ^H_ext", "none", "Schur + BJ", "Schur, none")
        print("| dt | " + " | ".join(names) + " |")
        print("|---" * (len(names) + 1) + "|")
        res = {pc: [] for pc in ("bjext", "bjext_h", "none", "schur_bj", "schur")}
        for dt in dts:
            row = []
            for pc in res:
                its, nw = gmres_iterations(kind, pc, dt, mach=mach, flux=flux)
                res[pc].append(its)
                row.append(f"{its} ({nw} Newton)" if its is not None else f"no conv.: {nw}")
            print(f"| {dt:.3e} | " + " | ".join(row) + " |")
        print("\nlog-log slope of iterations vs dt: " +
              ", ".join(f"{pc} {slope(dts, res[pc]):.2f}" for pc in res) + "\n")
        sys.stdout.flush()


if __name__ == "__main__":
    main()
