"""The five BASELINE.json configurations, restated as concrete problems.

Readings (DESIGN.md / SURVEY 8(c2)): GLL nodes (#1), LLF flux (#3),
k_max = q - 4 (#16), tolerances (#17), eps = 1 (#18), BR1 (#19),
dt from the element CFL rule (#14, #15):
    dt = CFL / max_nodes sum_d (|v_d| + c) / h_d   (c = 0 for advection)
evaluated once, in fp64, on the discrete initial state (before noise).
"""
from dataclasses import dataclass, field, replace
import math

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    dim: int
    equation: str              # advection | euler | navier_stokes
    N: int
    nx: int
    ny: int
    bounds: tuple              # (xmin, xmax, ymin, ymax)
    q: int
    kmax: int
    steps: int
    cfl: float
    a: tuple = (1.0, 1.0)
    gamma: float = 1.4
    mu: float = 0.0
    prandtl: float = 0.72
    noise: float = 0.0
    gmres_rtol: float = 1e-6
    newton_rtol: float = 1e-10
    newton_atol_dw: float = 1e-12
    restart: int = 700
    max_krylov: int = 7000
    precond: str = "bjext"
    nz: int = 1                # 3D (NEXT-4): elements in z; bounds then has 6 entries
    dt: float = 0.0            # > 0: a fixed time step (the paper's 3D case) instead of the CFL rule

    @property
    def nv(self):
        return 1 if self.equation == "advection" else (5 if self.dim == 3 else 4)

    @property
    def p(self):
        return self.N + 1

    @property
    def n_elem(self):
        return self.nx * (self.ny if self.dim >= 2 else 1) * (self.nz if self.dim == 3 else 1)

    @property
    def m(self):
        return self.nv * self.p ** self.dim

    @property
    def n(self):
        return self.n_elem * self.m


CONFIGS = {
    "C1": Config("C1", 1, "advection", 3, 16, 1, (0.0, 1.0, 0.0, 1.0), 4, 0, 10, 1.0,
                 a=(1.0, 0.0), gmres_rtol=1e-12),
    "C2": Config("C2", 2, "advection", 5, 64, 64, (0.0, 1.0, 0.0, 1.0), 6, 2, 50, 2.0),
    "C3": Config("C3", 2, "euler", 7, 128, 128, (-5.0, 5.0, -5.0, 5.0), 8, 4, 20, 1.0,
                 noise=1e-6, gmres_rtol=1e-10),
    "C4": Config("C4", 2, "euler", 7, 512, 512, (0.0, 1.0, 0.0, 1.0), 8, 4, 10, 1.0,
                 restart=16),
    "C5": Config("C5", 2, "navier_stokes", 5, 256, 256,
                 (0.0, 2 * math.pi, 0.0, 2 * math.pi), 6, 2, 20, 1.0, mu=1e-3),
}

# NEXT-4 (not a BASELINE config): the paper's 3D Taylor-Green mesh and scheme (32^3
# elements, N = 3, HBPC(4,0) on [0, 2 pi]^3) in this build's inviscid scope (3D Euler, reading R35).
# The paper's dt = 0.25 (element CFL ~ 8) belongs to its viscous Re-800 run; the inviscid system takes
# the configs' acoustic element-CFL-1 step (reading R14).
EXTRA = {
    "T3": Config("T3", 3, "euler", 3, 32, 32, (0.0, 2 * math.pi) * 3, 4, 0, 2, 1.0, nz=32),
}


def scaled(cfg: Config, **kw):
    """A smaller copy of a config (parity tests at oracle-friendly sizes)."""
    return replace(cfg, **kw)


def cfl_dt(cfg: Config, W):
    """Element CFL rule on a layout-L state W (reading #14); a config's fixed dt if it has one."""
    if cfg.dt > 0.0:
        return cfg.dt
    h = [(cfg.bounds[1] - cfg.bounds[0]) / cfg.nx]
    if cfg.dim >= 2:
        h.append((cfg.bounds[3] - cfg.bounds[2]) / cfg.ny)
    if cfg.dim == 3:
        h.append((cfg.bounds[5] - cfg.bounds[4]) / cfg.nz)
    if cfg.equation == "advection":
        s = sum(abs(cfg.a[d]) / h[d] for d in range(cfg.dim))
        return cfg.cfl / s
    nd = cfg.p ** cfg.dim
    Wv = np.asarray(W).reshape(-1, cfg.nv, nd)      # any block of whole elements
    rho, E = Wv[:, 0], Wv[:, -1]
    vel = [Wv[:, 1 + d] / rho for d in range(cfg.nv - 2)]
    p = (cfg.gamma - 1.0) * (E - 0.5 * rho * sum(v * v for v in vel))
    c = np.sqrt(cfg.gamma * p / rho)
    s = sum((np.abs(vel[d]) + c) / h[d] for d in range(len(vel)))
    return cfg.cfl / float(np.max(s))
