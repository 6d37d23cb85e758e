"""BR2 N = 3 (4x4) BJ_ext blocks on the GPU vs the oracle (GJ panel width A/B via HBPDC_GJ_NB)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from gpu_common import ns_ic, to_gpu, to_np, SEED  # noqa: E402
from test_gpu_br2 import _pair  # noqa: E402
from oracle import implicit  # noqa: E402

d, ctx = _pair(3, 4, 4, 2.0, q=4, kmax=0, gmres_rtol=1e-10, newton_rtol=1e-10)
W0 = ns_ic(d, SEED + 100, rel_noise=1e-3)
dt = 0.01
a1, a2 = 0.5, 1.0 / 6.0
pc = implicit.BJExt(d, W0, a1, a2, dt)
ctx.precond_build(a1, a2, dt, to_gpu(W0))
S, _ = ctx.precond_export()
S = to_np(S).reshape(pc.S.shape)
cond = max(np.linalg.cond(M) for M in pc.M)
print("GJ_NB", os.environ.get("HBPDC_GJ_NB", "32"), "m", d.m, "max cond(M)", f"{cond:.3e}",
      "rel S err", f"{np.linalg.norm(S - pc.S) / np.linalg.norm(pc.S):.3e}",
      "max |S|", f"{np.abs(pc.S).max():.3e}")
