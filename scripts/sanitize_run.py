"""A small run that exercises the mbarrier / bulk-copy kernels (DMMA GEMV with 2 and 6
right-hand sides, s = 8 TMA block Gram-Schmidt incl. the fused update + re-projection,
the Gauss-Jordan build, the staged FD JVP) for compute-sanitizer racecheck / synccheck /
memcheck:  compute-sanitizer --tool racecheck python scripts/sanitize_run.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2109_04804_b200 import configs, hbpdc, inputs  # noqa: E402

cfg = configs.CONFIGS["C3"]
h = (cfg.bounds[1] - cfg.bounds[0]) / cfg.nx
half = 2 * h
ctx = hbpdc.Context(dim=2, equation="euler", N=7, nx=4, ny=4, bounds=(-half, half, -half, half), q=8, kmax=4,
                    newton_rtol=1e-10, gmres_rtol=1e-10, restart=64, gmres_sstep=8, batch_stages=True)
X, Y = ctx.node_coords()
W = torch.tensor(inputs.initial_state("C3", (X, Y), noise=cfg.noise), dtype=torch.float64, device="cuda")
st = ctx.step(0.0144875, W)
torch.cuda.synchronize()
print("step ok", st)
ctx.close()
