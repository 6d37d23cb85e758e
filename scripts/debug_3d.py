"""Which direction of the 3D operator disagrees with the oracle: advection R1 on fields that vary
in x only, y only, z only (and mixed), per node position class (interior / face / edge / corner)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from gpu_common import to_gpu, to_np  # noqa: E402
from test_gpu_3d import pair3  # noqa: E402
from oracle import dgsem  # noqa: E402

for n in [(3, 3, 3), (3, 2, 4)]:
    for N in (1, 2):
        d, ctx = pair3("advection", N, n, a=(1.0, 0.0, 0.0))
        X, Y, Z = d.node_coords()
        for name, f in [("x", np.sin(X)), ("y", np.sin(Y)), ("z", np.sin(Z)), ("xyz", np.sin(X + 2 * Y + 3 * Z))]:
            for a in [(1.0, 0.0, 0.0), (0.0, 1.0, 0.0), (0.0, 0.0, 1.0)]:
                d, ctx = pair3("advection", N, n, a=a)
                W = np.ascontiguousarray(f).reshape(-1)
                g = to_np(ctx.rhs(to_gpu(W)))
                o = dgsem.rhs1(d, W)
                err = np.abs(g - o).reshape(n[2], n[1], n[0], N + 1, N + 1, N + 1)
                print(f"mesh {n} N={N} field {name:3s} a={a}: max err {err.max():.2e} "
                      f"(|o| {np.abs(o).max():.2e}); worst node (ez,ey,ex,k,j,i) {np.unravel_index(err.argmax(), err.shape)}")
                ctx.close()
