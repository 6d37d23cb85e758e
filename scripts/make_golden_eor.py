"""Write the oracle end-of-run references for the bench-path GPU parity tests
(tests/test_gpu_benchpath.py) into tests/golden/eor_<case>.npz.

Calls only oracle/ (and the seeded input module paper_2109_04804_b200.inputs /
configs, which hold no arithmetic of the method).  The numpy oracle needs
minutes per HBPC(8,4) step at N = 7, too long to re-run inside every GPU test
session, so the end states are stored; the GPU side recomputes nothing from
them except the comparison.  Re-run after any change to the oracle's arithmetic:

    python scripts/make_golden_eor.py [case ...]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import basis, dgsem, hbpc, implicit, physics          # noqa: E402
from paper_2109_04804_b200 import configs, inputs                  # noqa: E402


def case_setup(name):
    """(Disc, q, kmax, W0, dt, steps, NewtonOpts, description) of a golden case."""
    if name == "c3_window_n7":
        # C3's own discretisation and step on a 4x4-element periodic window of its
        # mesh centred on the vortex: same h, N = 7, dt (CFL 1 on the full C3 IC),
        # HBPC(8,4), GMRES/Newton 1e-10, BJ_ext, FD JVP -- the bench's per-element regime
        cfg = configs.CONFIGS["C3"]
        h = (cfg.bounds[1] - cfg.bounds[0]) / cfg.nx
        half = 4 * h / 2
        d = dgsem.Disc(basis.build_basis(7, "gll"), dgsem.Mesh(2, 4, 4, -half, half, -half, half),
                       physics.Equation("euler"))
        W0 = inputs.initial_state("C3", d.node_coords(), noise=cfg.noise)
        full = dgsem.Disc(d.basis, dgsem.Mesh(2, cfg.nx, cfg.ny, *cfg.bounds), d.eq)
        dt = configs.cfl_dt(cfg, inputs.initial_state("C3", full.node_coords()))
        opts = implicit.NewtonOpts(rtol=cfg.newton_rtol, gmres_rtol=cfg.gmres_rtol)
        return d, 8, 4, W0, dt, 1, opts, "C3 window 4x4 el., N=7 GLL, LLF, HBPC(8,4), 1 step, rtol 1e-10"
    if name == "c5_ns_n5":
        # C5 physics (NS, BR1, Re 1000, Pr 0.72, Mach 0.1 TGV-type IC) on 6x6 elements
        # of [0, 2pi]^2 (colouring period 3), N = 5, HBPC(6,2), CFL-1 dt, GMRES 1e-6
        cfg = configs.scaled(configs.CONFIGS["C5"], nx=6, ny=6)
        eq = physics.Equation("navier_stokes", mu=cfg.mu)
        d = dgsem.Disc(basis.build_basis(5, "gll"), dgsem.Mesh(2, 6, 6, *cfg.bounds), eq)
        W0 = inputs.initial_state("C5", d.node_coords())
        dt = configs.cfl_dt(cfg, W0)
        opts = implicit.NewtonOpts(rtol=cfg.newton_rtol, gmres_rtol=cfg.gmres_rtol)
        return d, 6, 2, W0, dt, 2, opts, "C5 physics 6x6 el., N=5 GLL, BR1, HBPC(6,2), 2 steps, GMRES 1e-6"
    if name == "c4_dw_n7_r16":
        # C4 physics (density wave) on 4x4 elements of [0, 1]^2, N = 7, HBPC(8,4),
        # GMRES(16) restarts (C4's setting, reading R11), GMRES 1e-6, Newton 1e-10
        cfg = configs.scaled(configs.CONFIGS["C4"], nx=4, ny=4)
        d = dgsem.Disc(basis.build_basis(7, "gll"), dgsem.Mesh(2, 4, 4, *cfg.bounds), physics.Equation("euler"))
        W0 = inputs.initial_state("C4", d.node_coords())
        dt = configs.cfl_dt(cfg, W0)
        opts = implicit.NewtonOpts(rtol=cfg.newton_rtol, gmres_rtol=cfg.gmres_rtol, restart=cfg.restart)
        return d, 8, 4, W0, dt, 2, opts, "C4 physics 4x4 el., N=7 GLL, HBPC(8,4), restart 16, 2 steps"
    raise KeyError(name)


CASES = ["c3_window_n7", "c5_ns_n5", "c4_dw_n7_r16"]


def main(names):
    for name in names:
        d, q, kmax, W0, dt, steps, opts, desc = case_setup(name)
        H = hbpc.HBPC(d, q, kmax, opts)
        st = dict(stage_solves=0, newton_its=0, gmres_its=0, precond_builds=0)
        W = W0.copy()
        t0 = time.time()
        for _ in range(steps):
            W = H.step(W, dt, st)
        sec = time.time() - t0
        out = os.path.join(ROOT, "tests", "golden", f"eor_{name}.npz")
        np.savez_compressed(out, W=W, dt=dt, steps=steps, desc=desc,
                            stats=np.array([st["stage_solves"], st["newton_its"], st["gmres_its"],
                                            st["precond_builds"]]), seconds=sec)
        print(f"{name}: {desc}; dt {dt:.6g}; {st}; {sec:.1f} s -> {out}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or CASES)
