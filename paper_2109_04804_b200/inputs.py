"""Seeded synthetic inputs shared by the CUDA path and the CPU oracle.

This module holds NO arithmetic of the method (no basis, no operator, no
solver): it evaluates the analytic initial conditions of BASELINE.json's
configs at node coordinates handed in by the caller, adds the seeded noise,
and draws random perturbations for parity tests.  Node coordinates come
from the library (``hbpdc_node_coords``) in the product path and from the
oracle in tests; tests check that the two agree.

Recipes: DESIGN.md section "Inputs".  Seeds: master 2109_04804; config k
(0-based, C1 = 0) noise stream ``default_rng(2109_04804 + k)``; operator
test inputs ``default_rng(2109_04804 + 100*k + test_id)``.
"""
import math

import numpy as np

MASTER_SEED = 2109_04804
GAMMA = 1.4


def conserved(rho, u, v, p, gamma=GAMMA):
    """(rho, rho u, rho v, E) with E = p/(gamma-1) + rho |v|^2 / 2."""
    return (rho, rho * u, rho * v, p / (gamma - 1.0) + 0.5 * rho * (u * u + v * v))


def conserved3(rho, u, v, w, p, gamma=GAMMA):
    """3D: (rho, rho u, rho v, rho w, E), E = p/(gamma-1) + rho |v|^2 / 2."""
    return (rho, rho * u, rho * v, rho * w, p / (gamma - 1.0) + 0.5 * rho * (u * u + v * v + w * w))


def ic_primitive(case, X, Y=None, Z=None, gamma=GAMMA):
    """Analytic initial condition of a config at coordinates X (and Y, Z).
    Returns a tuple of variables (1 for advection, 4 conserved for Euler/NS in
    2D, 5 in 3D).  3D cases (NEXT-4): "TGV3" = the paper's Taylor-Green data
    (P:1088-1091 with eps = 1 and the standard divergence-free first velocity
    component sin x cos y cos z, reading R35) on [0, 2 pi]^3;
    "DW3" = 3D density wave rho = 1 + 0.2 sin(2 pi (x + y + z)), v = (1, 1, 1),
    p = 1 (an exact translating solution) on [0, 1]^3; "ADV3" = sin(2 pi x)
    sin(2 pi y) sin(2 pi z)."""
    if case == "TGV3":
        rho = np.ones_like(X)
        u = np.sin(X) * np.cos(Y) * np.cos(Z)
        v = -np.cos(X) * np.sin(Y) * np.cos(Z)
        p = rho / gamma + rho / 16.0 * (np.cos(2 * X) + np.cos(2 * Y)) * (np.cos(2 * Z) + 2.0)
        return conserved3(rho, u, v, 0.0 * X, p, gamma)
    if case == "DW3":
        rho = 1.0 + 0.2 * np.sin(2 * math.pi * (X + Y + Z))
        one = np.ones_like(X)
        return conserved3(rho, one, one, one, one, gamma)
    if case == "ADV3":
        return (np.sin(2 * math.pi * X) * np.sin(2 * math.pi * Y) * np.sin(2 * math.pi * Z),)
    if case == "C1":                                       # 1D advection
        return (np.sin(2 * math.pi * X),)
    if case == "C2":                                       # 2D advection
        return (np.sin(2 * math.pi * X) * np.sin(2 * math.pi * Y),)
    if case == "C3":                                       # isentropic vortex
        beta = 5.0
        r2 = X * X + Y * Y
        T = 1.0 - (gamma - 1.0) * beta * beta * np.exp(1.0 - r2) / (8.0 * gamma * math.pi ** 2)
        rho = T ** (1.0 / (gamma - 1.0))
        p = rho ** gamma
        f = beta / (2 * math.pi) * np.exp(0.5 * (1.0 - r2))
        return conserved(rho, 1.0 - f * Y, 1.0 + f * X, p, gamma)
    if case == "C4":                                       # density wave
        rho = 1.0 + 0.2 * np.sin(2 * math.pi * (X + Y))
        one = np.ones_like(X)
        return conserved(rho, one, one, one, gamma)
    if case == "C5":                                       # TGV-type, Mach 0.1
        M = 0.1
        rho = np.ones_like(X)
        u = np.sin(X) * np.cos(Y)
        v = -np.cos(X) * np.sin(Y)
        p = 1.0 / (gamma * M * M) + 0.25 * (np.cos(2 * X) + np.cos(2 * Y))
        return conserved(rho, u, v, p, gamma)
    raise ValueError(case)


def layout(vars_, dim):
    """Stack per-variable node arrays into layout L ([elem][var][(k)][j][i]).
    3D inputs have shape (nz, ny, nx, p, p, p); 2D (ny, nx, p, p) [j, i]; 1D (nx, p)."""
    ax = dim
    return np.ascontiguousarray(np.stack(vars_, axis=ax)).reshape(-1)


CASE_INDEX = {"C1": 0, "C2": 1, "C3": 2, "C4": 3, "C5": 4, "TGV3": 5, "DW3": 6, "ADV3": 7}


def initial_state(case, coords, noise=None, gamma=GAMMA, stream=0):
    """Nodal interpolation of the IC in layout L, plus the seeded
    uniform noise of amplitude `noise` on every conserved variable (C3:
    1e-6), drawn in layout order from default_rng(MASTER_SEED + k).
    stream > 0 (the rank of a tiled multi-GPU bench block) draws from
    default_rng(MASTER_SEED + k + 1000 * stream) instead."""
    dim = len(coords)
    W = layout(ic_primitive(case, *coords, gamma=gamma), dim)
    if noise:
        rng = np.random.default_rng(MASTER_SEED + CASE_INDEX[case] + 1000 * stream)
        W = W + rng.uniform(-noise, noise, size=W.shape)
    return W


def tile_coords(coords, bounds):
    """Map node coordinates of a mesh made of repeated copies of a config's
    periodic domain back into the copy at [xmin, xmax) x [ymin, ymax): each
    element is shifted by whole periods according to its centre, so every
    tile sees exactly the config's own nodes (the multi-GPU bench repeats
    C3's tile).  Identity on the config's own mesh."""
    out = []
    for d, c in enumerate(coords):
        c = np.asarray(c)
        lo, hi = bounds[2 * d], bounds[2 * d + 1]
        ctr = c.mean(axis=tuple(range(c.ndim - (len(coords)), c.ndim)), keepdims=True)
        tile = np.floor((ctr - lo) / (hi - lo))
        out.append(c - tile * (hi - lo))
    return tuple(out)


def perturbed_state(W_ic, seed, rel=1e-2):
    """W = IC + U[-rel, rel) |IC| in layout order (parity inputs)."""
    rng = np.random.default_rng(seed)
    return W_ic + rng.uniform(-rel, rel, size=W_ic.shape) * np.abs(W_ic)


def random_field(n, seed, scale=1.0, unit_norm=False):
    """N(0, 1) * scale, optionally normalised to unit 2-norm (Krylov-like)."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(n) * scale
    if unit_norm:
        x = x / np.linalg.norm(x)
    return x
