"""Closed-form evaluation of HBPC(q, k_max) for LINEAR semi-discretisations
w' = K w (advection), used as pins and as the full-size C1/C2 end-of-run
reference.

TEST INFRASTRUCTURE (see oracle/__init__.py).

For a linear flux R1(w) = K w and R2(w, sigma) = R1(sigma) (the time
derivative of K w along w_t = sigma), so R2(w) := R2(w, R1(w)) = K^2 w.
Every stage equation of Alg. 1 (eq:Newton_Residual, with
G = W - a1 dt R1(W) + (a2 dt^2/2) R2(W) - b, reading R4) is then the LINEAR
system (I - a1 dt K + (a2 dt^2/2) K^2) W = b, solved here exactly (dense LU)
instead of by Newton-GMRES:

  predictor (eq:predictor): a1 = dc/2, a2 = dc^2/6 (dc = c_l - c_{l-1}),
      b = w_{l-1} + a1 dt K w_{l-1} + (a2 dt^2/2) K^2 w_{l-1};
  corrector (eq:corrector, with I_l, reading R5): a1 = a2 = 1,
      b = w^n - dt K w^k_l + (dt^2/2) K^2 w^k_l
          + dt sum_j B1_lj K w^k_j + dt^2 sum_j B2_lj K^2 w^k_j;
  update w^{n+1} = w^{k_max}_s.

On a uniform periodic Cartesian mesh K is block-circulant over the element
grid (every element couples to itself and its face neighbours with the same
blocks), so a 2D DFT over the element indices diagonalises it into nx*ny
independent m x m symbols K^(kx, ky) = sum_off B_off exp(2 pi i (kx dx/nx +
ky dy/ny)); Alg. 1 is applied to each Fourier coefficient (SURVEY 8(c3) T2 iii).
The blocks B_off are read off the oracle's own R^(1) (dgsem.rhs1) on a 3 x 3
element mesh with the same element size.
"""
import numpy as np

from . import dgsem
from .tableau import tableau


def hbpc_linear_stepper(K, q, kmax, dt):
    """w -> one HBPC(q, kmax) step of w' = K w with exact stage solves.
    K: (..., m, m) (real or complex, batched); the returned function maps
    w: (..., m) to w^{n+1}.  The two stage matrices are inverted once."""
    c, B1, B2 = tableau(q)
    s = len(c)
    m = K.shape[-1]
    I = np.broadcast_to(np.eye(m), K.shape)
    K2 = K @ K
    mv = lambda A, x: np.einsum("...ij,...j->...i", A, x)          # noqa: E731
    R1 = lambda x: mv(K, x)                                        # noqa: E731
    R2 = lambda x: mv(K2, x)                                       # noqa: E731
    solves = {}

    def solve(a1, a2, b):
        key = (round(a1, 12), round(a2, 12))
        if key not in solves:
            solves[key] = np.linalg.inv(I - a1 * dt * K + (a2 * dt * dt / 2.0) * K2)
        return mv(solves[key], b)

    def step(w):
        wl = [w] + [None] * (s - 1)
        for l in range(1, s):
            dc = c[l] - c[l - 1]
            a1, a2 = dc / 2.0, dc * dc / 6.0
            b = wl[l - 1] + a1 * dt * R1(wl[l - 1]) + (a2 * dt * dt / 2.0) * R2(wl[l - 1])
            wl[l] = solve(a1, a2, b)
        for _ in range(kmax):
            r1 = [R1(x) for x in wl]
            r2 = [R2(x) for x in wl]
            new = [w] + [None] * (s - 1)
            for l in range(1, s):
                I_l = (dt * sum(B1[l, j] * r1[j] for j in range(s))
                       + dt * dt * sum(B2[l, j] * r2[j] for j in range(s)))
                b = w - dt * r1[l] + (dt * dt / 2.0) * r2[l] + I_l
                new[l] = solve(1.0, 1.0, b)
            wl = new
        return wl[s - 1]

    return step


def hbpc_linear_step(K, q, kmax, dt, w):
    """One HBPC(q, kmax) step of w' = K w with exact stage solves."""
    return hbpc_linear_stepper(K, q, kmax, dt)(w)


def element_blocks(disc):
    """Coupling blocks B_off = dR1_e / dW_{e+off} of a linear periodic
    discretisation, off in {(0,0), (+-1,0), (0,+-1)} (2D) or {0, +-1} (1D),
    read off dgsem.rhs1 applied to unit vectors on a 3 (x 3) element mesh."""
    me, m = disc.mesh, disc.m
    if me.dim == 1:
        d3 = dgsem.Disc(disc.basis, dgsem.Mesh(1, 3, 1, 0.0, 3 * me.dx), disc.eq)
        offs = [(-1, 0), (0, 0), (1, 0)]
        centre = 1
        idx = lambda ox, oy: 1 + ox                                # noqa: E731
    else:
        d3 = dgsem.Disc(disc.basis, dgsem.Mesh(2, 3, 3, 0.0, 3 * me.dx, 0.0, 3 * me.dy), disc.eq)
        offs = [(0, 0), (-1, 0), (1, 0), (0, -1), (0, 1)]
        centre = 4
        idx = lambda ox, oy: (1 + oy) * 3 + (1 + ox)               # noqa: E731
    blocks = {}
    for off in offs:
        B = np.zeros((m, m))
        for col in range(m):
            e = np.zeros(d3.n)
            e[idx(*off) * m + col] = 1.0
            B[:, col] = dgsem.rhs1(d3, e)[centre * m:(centre + 1) * m]
        blocks[off] = B
    return blocks


def run_fourier(disc, q, kmax, dt, W0, steps):
    """`steps` HBPC(q, kmax) steps of the linear periodic problem, evaluated
    per Fourier mode of the element grid.  W0 in layout L; returns layout L."""
    me, m = disc.mesh, disc.m
    nx, ny = me.nx, (me.ny if me.dim == 2 else 1)
    blocks = element_blocks(disc)
    kx = np.arange(nx)[None, :]
    ky = np.arange(ny)[:, None]
    Khat = np.zeros((ny, nx, m, m), complex)
    for (ox, oy), B in blocks.items():
        ph = np.exp(2j * np.pi * (kx * ox / nx + ky * oy / ny))
        Khat += ph[:, :, None, None] * B
    What = np.fft.fft2(np.asarray(W0, float).reshape(ny, nx, m), axes=(0, 1))
    step = hbpc_linear_stepper(Khat, q, kmax, dt)
    for _ in range(steps):
        What = step(What)
    return np.real(np.fft.ifft2(What, axes=(0, 1))).reshape(-1)
