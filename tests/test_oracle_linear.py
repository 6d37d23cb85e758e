"""Pins for oracle.linear (HBPC of w' = K w with exact stage solves, and its
per-Fourier-mode evaluation on periodic meshes).  CPU only."""
import numpy as np
import pytest
import scipy.linalg as sla

from oracle import basis, dgsem, hbpc, implicit, linear, physics
from paper_2109_04804_b200 import configs, inputs


def dense_K(d):
    return np.stack([dgsem.rhs1(d, e) for e in np.eye(d.n)], axis=1)


def adv(dim, N, nx, ny=1, a=(1.0, 0.7)):
    eq = physics.Equation("advection", a=a)
    return dgsem.Disc(basis.build_basis(N, "gll"), dgsem.Mesh(dim, nx, ny, 0.0, 1.0, 0.0, 1.0), eq)


@pytest.mark.parametrize("kmax", [0, 3])
def test_q4_step_is_pade(kmax):
    """HBPC(4, k) on w' = K w is the (2,2)-Pade approximant of exp(dt K)
    (P:110 with c = (0, 1); the correctors leave it unchanged)."""
    d = adv(1, 3, 6, a=(1.0, 0.0))
    K = dense_K(d)
    dt = 0.07
    I = np.eye(d.n)
    P = np.linalg.solve(I - dt * K / 2 + dt * dt * K @ K / 12, I + dt * K / 2 + dt * dt * K @ K / 12)
    w = np.random.default_rng(1).standard_normal(d.n)
    assert np.linalg.norm(linear.hbpc_linear_step(K, 4, kmax, dt, w) - P @ w) <= 1e-13 * np.linalg.norm(P @ w)


@pytest.mark.parametrize("q,kmax,order", [(6, 2, 6), (8, 4, 8), (8, 1, 5)])
def test_time_order_against_expm(q, kmax, order):
    """EOC min(4 + k_max, q) against exp(T K) w0."""
    d = adv(1, 7, 6, a=(1.0, 0.0))
    K = dense_K(d)
    W0 = inputs.initial_state("C1", d.node_coords())
    T = 0.5
    ref = sla.expm(T * K) @ W0
    errs = []
    for nst in (4, 8):
        dt = T / nst
        w = W0.copy()
        for _ in range(nst):
            w = linear.hbpc_linear_step(K, q, kmax, dt, w)
        errs.append(np.linalg.norm(w - ref))
    eoc = np.log2(errs[0] / errs[1])
    assert abs(eoc - order) <= 0.5, (eoc, errs)


def test_exact_stage_solves_equal_newton_gmres_oracle():
    """The linear-algebra Alg. 1 and the general oracle (Newton-GMRES with
    BJ_ext at tight tolerances) give the same step on a 2D advection mesh."""
    d = adv(2, 3, 3, 4)
    K = dense_K(d)
    W0 = inputs.initial_state("C2", d.node_coords())
    dt = 0.05
    H = hbpc.HBPC(d, 6, 2, implicit.NewtonOpts(rtol=1e-13, gmres_rtol=1e-13))
    w_newton = H.step(W0, dt)
    w_lin = linear.hbpc_linear_step(K, 6, 2, dt, W0)
    assert np.linalg.norm(w_newton - w_lin) <= 1e-11 * np.linalg.norm(w_lin)


@pytest.mark.parametrize("dim,nx,ny", [(2, 4, 3), (2, 5, 5), (1, 7, 1)])
def test_fourier_equals_dense(dim, nx, ny):
    """Block-circulant diagonalisation: per-mode evaluation == dense K."""
    d = adv(dim, 2, nx, ny)
    K = dense_K(d)
    rng = np.random.default_rng(3)
    W0 = rng.standard_normal(d.n)
    dt, steps = 0.04, 3
    w = W0.copy()
    for _ in range(steps):
        w = linear.hbpc_linear_step(K, 8, 4, dt, w)
    wf = linear.run_fourier(d, 8, 4, dt, W0, steps)
    assert np.linalg.norm(wf - w) <= 1e-12 * np.linalg.norm(w)


def test_c2_fourier_run_is_bounded_and_translates():
    """Sanity at the full C2 configuration (64 x 64, N = 5, HBPC(6,2), 50
    steps): the discrete solution stays close to the exact translated field
    (T = 0.78125; spatial + temporal error of a well-resolved sine)."""
    cfg = configs.CONFIGS["C2"]
    d = adv(2, cfg.N, cfg.nx, cfg.ny, a=cfg.a)
    X, Y = d.node_coords()
    W0 = inputs.initial_state("C2", (X, Y))
    dt = configs.cfl_dt(cfg, W0)
    W = linear.run_fourier(d, cfg.q, cfg.kmax, dt, W0, cfg.steps)
    T = dt * cfg.steps
    exact = inputs.initial_state("C2", (X - cfg.a[0] * T, Y - cfg.a[1] * T))
    assert np.abs(W - exact).max() <= 1e-5
