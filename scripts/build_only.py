"""One BJ_ext build on a full-size config (for ncu launch lists): python scripts/build_only.py C3"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2109_04804_b200 import configs, hbpdc, inputs  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "C3"
cfg = configs.CONFIGS[case]
ctx = hbpdc.context_for(cfg, restart=16, batch_stages=False)
coords = ctx.node_coords()
W = torch.tensor(inputs.initial_state(case, coords, noise=cfg.noise), dtype=torch.float64, device="cuda")
dt = configs.cfl_dt(cfg, inputs.initial_state(case, coords))
ctx.precond_build(0.5, 1 / 6, dt, W)
torch.cuda.synchronize()
ctx.close()
