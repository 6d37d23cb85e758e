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

    @property
    def nv(self):
        return 1 if self.equation == "advection" else 4

    @property
    def p(self):
        return self.N + 1

    @property
    def n_elem(self):
        return self.nx * (self.ny if self.dim == 2 else 1)

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


def scaled(cfg: Config, **kw):
    """A smaller copy of a config (parity tests at oracle-friendly sizes)."""
    return replace(cfg, **kw)


def cfl_dt(cfg: Config, W):
    """Element CFL rule on a layout-L state W (reading #14)."""
    h = [(cfg.bounds[1] - cfg.bounds[0]) / cfg.nx]
    if cfg.dim == 2:
        h.append((cfg.bounds[3] - cfg.bounds[2]) / cfg.ny)
    if cfg.equation == "advection":
        s = sum(abs(cfg.a[d]) / h[d] for d in range(cfg.dim))
        return cfg.cfl / s
    nd = cfg.p ** cfg.dim
    Wv = np.asarray(W).reshape(-1, cfg.nv, nd)      # any block of whole elements
    rho, mx, my, E = (Wv[:, k] for k in range(4))
    u, v = mx / rho, my / rho
    p = (cfg.gamma - 1.0) * (E - 0.5 * rho * (u * u + v * v))
    c = np.sqrt(cfg.gamma * p / rho)
    s = (np.abs(u) + c) / h[0] + (np.abs(v) + c) / h[1]
    return cfg.cfl / float(np.max(s))
