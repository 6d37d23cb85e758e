"""Host-side logic of bench.py (no GPU): stage-solve counts, the per-rank memory plan, and the
strong-scaling initial state (each rank's block of the global field, C3's noise drawn once in
global layout order so that every partition sees the same numbers as one GPU)."""
import numpy as np
import pytest

import bench
from oracle import basis, dgsem, physics
from paper_2109_04804_b200 import configs, inputs


def test_stage_solves_per_step():
    # (s - 1)(k_max + 1) with s = 2, 3, 4 stages for q = 4, 6, 8 (App. A)
    assert bench.stage_solves_per_step(8, 4) == 15
    assert bench.stage_solves_per_step(6, 2) == 6
    assert bench.stage_solves_per_step(4, 0) == 1


def test_memory_plan_c4():
    cfg = configs.CONFIGS["C4"]
    p1 = bench.memory_plan(cfg, 1, False, False, 16, 8)
    assert p1["S_GB"] == pytest.approx(137.4, abs=0.1)           # 512^2 x 256^2 x 8 B
    assert p1["total_GB"] < 190.0                                  # one B200: 191.5 GB
    p8 = bench.memory_plan(cfg, 8, False, True, 16, 8)
    assert p8["S_GB"] == pytest.approx(17.2, abs=0.1)


class _FakeCtx:
    """A rank's block as the library reports it (offsets, extents, node coordinates)."""

    def __init__(self, d_global, px, py, rank):
        me = d_global.mesh
        self.nx_local, self.ny_local = me.nx // px, me.ny // py
        self.ex0, self.ey0 = (rank % px) * self.nx_local, (rank // px) * self.ny_local
        X, Y = d_global.node_coords()
        sl = (slice(self.ey0, self.ey0 + self.ny_local), slice(self.ex0, self.ex0 + self.nx_local))
        self._c = (np.ascontiguousarray(X[sl]), np.ascontiguousarray(Y[sl]))

    def node_coords(self):
        return self._c


@pytest.mark.parametrize("px,py", [(2, 1), (2, 2), (4, 2)])
def test_strong_scaling_blocks_tile_the_global_state(px, py):
    """C3 at a reduced mesh (8x8, N = 3): the union of the ranks' blocks is the one-GPU state
    bit for bit, noise included."""
    cfg = configs.scaled(configs.CONFIGS["C3"], N=3, nx=8, ny=8)
    d = dgsem.Disc(basis.build_basis(3, "gll"), dgsem.Mesh(2, 8, 8, *cfg.bounds), physics.Equation("euler"))
    W_global = inputs.initial_state("C3", d.node_coords(), noise=cfg.noise)
    G = W_global.reshape(cfg.ny, cfg.nx, cfg.m)
    for r in range(px * py):
        ctx = _FakeCtx(d, px, py, r)
        W, _ = bench.local_initial_state("C3", cfg, ctx, False, r)
        blk = G[ctx.ey0:ctx.ey0 + ctx.ny_local, ctx.ex0:ctx.ex0 + ctx.nx_local].reshape(-1)
        assert np.array_equal(W, blk)
