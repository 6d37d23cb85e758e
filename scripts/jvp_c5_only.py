"""Three C5 FD JVPs (for an ncu launch list of the NS operator pipeline)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2109_04804_b200 import configs, hbpdc, inputs  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "C5"
cfg = configs.CONFIGS[case]
ctx = hbpdc.context_for(cfg, restart=16, batch_stages=False)
coords = ctx.node_coords()
W = torch.tensor(inputs.perturbed_state(inputs.initial_state(case, coords, noise=cfg.noise), 901),
                 dtype=torch.float64, device="cuda")
sig = ctx.rhs(W)
g = torch.Generator().manual_seed(7)
dW = torch.randn(ctx.n, generator=g, dtype=torch.float64).cuda()
dS = torch.randn(ctx.n, generator=g, dtype=torch.float64).cuda()
o1, o2 = ctx.empty(), ctx.empty()
for _ in range(3):
    ctx.jvp(0.5, 0.2, 1e-3, W, sig, dW, dS, mode="fd", out1=o1, out2=o2)
torch.cuda.synchronize()
ctx.close()
