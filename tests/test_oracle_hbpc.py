"""Pins for oracle.hbpc (Alg. 1) against closed forms.  CPU only."""
import numpy as np
import pytest
import scipy.linalg as sla

from oracle import basis, dgsem, hbpc, implicit, physics
from paper_2109_04804_b200 import configs, inputs


def adv1d(N, nx, a=1.0):
    eq = physics.Equation("advection", a=(a, 0.0))
    return dgsem.Disc(basis.build_basis(N, "gll"), dgsem.Mesh(1, nx, 1, 0.0, 1.0), eq)


def dense_K(d):
    """Dense matrix of the (linear) advection R1, built column by column."""
    return np.stack([dgsem.rhs1(d, e) for e in np.eye(d.n)], axis=1)


@pytest.mark.parametrize("kmax", [0, 2])
def test_c1_whole_run_is_pade(kmax):
    """For w' = K w, one HBPC(4, k) step is exactly the (2,2)-Pade
    approximant (I - dtK/2 + dt^2K^2/12)^-1 (I + dtK/2 + dt^2K^2/12), read
    off eq:predictor with c = (0, 1); correction sweeps do not change
    it.  The C1 run (10 steps) is that matrix^10 w0."""
    cfg = configs.CONFIGS["C1"]
    d = adv1d(cfg.N, cfg.nx)
    W0 = inputs.initial_state("C1", d.node_coords())
    dt = configs.cfl_dt(cfg, W0)
    assert dt == 0.0625
    K = dense_K(d)
    I = np.eye(d.n)
    R = np.linalg.solve(I - dt * K / 2 + dt * dt * K @ K / 12, I + dt * K / 2 + dt * dt * K @ K / 12)
    ref = np.linalg.matrix_power(R, cfg.steps) @ W0
    opts = implicit.NewtonOpts(rtol=cfg.newton_rtol, gmres_rtol=cfg.gmres_rtol)
    H = hbpc.HBPC(d, 4, kmax, opts)
    W = W0.copy()
    for _ in range(cfg.steps):
        W = H.step(W, dt)
    assert np.linalg.norm(W - ref) <= 1e-11 * np.linalg.norm(ref)


def test_zero_velocity_is_identity():
    """a = 0: R1 = 0, the state is unchanged."""
    d = adv1d(3, 4, a=0.0)
    W0 = np.random.default_rng(0).standard_normal(d.n)
    H = hbpc.HBPC(d, 8, 4, implicit.NewtonOpts(precond="none"))
    W = H.step(W0, 0.3)
    np.testing.assert_array_equal(W, W0)


@pytest.mark.parametrize("q,kmax,order", [(4, 0, 4), (6, 0, 4), (6, 1, 5), (6, 2, 6), (8, 2, 6), (8, 4, 8)])
def test_time_order(q, kmax, order):
    """EOC against the exact semi-discrete solution expm(T K) w0 (isolates
    the time error): min(4 + k_max, q)."""
    d = adv1d(7, 6)
    K = dense_K(d)
    W0 = inputs.initial_state("C1", d.node_coords())
    T = 0.5
    ref = sla.expm(T * K) @ W0
    nst = (4, 8) if order < 8 else (8, 16)
    errs = []
    for n_steps in nst:
        H = hbpc.HBPC(d, q, kmax, implicit.NewtonOpts(rtol=1e-13, gmres_rtol=1e-13, precond="none"))
        W = W0.copy()
        for _ in range(n_steps):
            W = H.step(W, T / n_steps)
        errs.append(np.linalg.norm(W - ref))
    eoc = np.log2(errs[0] / errs[1])
    assert abs(eoc - order) < 0.4, (errs, eoc)


def test_kmax_invariance_q4():
    """HBPC(4, k): k = 0 and k = 2 agree within 10x the Newton tolerance
     -- Euler, nonlinear."""
    eq = physics.Equation("euler")
    d = dgsem.Disc(basis.build_basis(2, "gll"), dgsem.Mesh(2, 2, 2), eq)
    rng = np.random.default_rng(1)
    W0 = np.zeros(d.field_shape())
    for v, x in enumerate([1.0, 0.5, 0.3, 2.5]):
        W0[:, :, v] = x
    W0 = W0.reshape(-1) * (1 + 0.02 * rng.uniform(-1, 1, d.n))
    out = []
    for k in (0, 2):
        H = hbpc.HBPC(d, 4, k, implicit.NewtonOpts(rtol=1e-12, gmres_rtol=1e-12))
        out.append(H.step(W0, 0.05))
    assert np.linalg.norm(out[0] - out[1]) <= 10 * 1e-12 * np.linalg.norm(out[0]) * 100


def test_fsal_and_stage1():
    """FSAL: the cached R1/R2 for the next step are those of the returned
    state (bit identity)."""
    d = adv1d(3, 4)
    W0 = inputs.initial_state("C1", d.node_coords())
    H = hbpc.HBPC(d, 6, 2, implicit.NewtonOpts(precond="none", gmres_rtol=1e-12))
    W1 = H.step(W0, 0.05)
    r1 = dgsem.rhs1(d, W1)
    np.testing.assert_array_equal(H.cache[0], r1)


def test_navier_stokes_run_converges_to_rk4():
    """The Navier-Stokes end of run, pinned to something other than HBPC itself:
    HBPC(4,0) steps of the BR1 semi-discretisation (whose R1 is pinned in
    test_oracle_dgsem.py) converge at order 4 to an independent
    classical RK4 solution of the same ODE W' = R1(W) with 200 steps (its own
    error ~1e-12, far below the HBPC errors).  A wrong NS R2 = dR1/dt (e.g. a
    dropped lifting-derivative term) would reduce the order to 2."""
    eq = physics.Equation("navier_stokes", mu=0.05)
    d = dgsem.Disc(basis.build_basis(2, "gll"), dgsem.Mesh(2, 3, 3, 0.0, 2 * np.pi, 0.0, 2 * np.pi), eq)
    X, Y = d.node_coords()
    W0 = inputs.perturbed_state(inputs.initial_state("C5", (X, Y)), 7, 1e-2)
    T = 0.04

    def rk4(W, n):
        h = T / n
        for _ in range(n):
            k1 = dgsem.rhs1(d, W)
            k2 = dgsem.rhs1(d, W + h / 2 * k1)
            k3 = dgsem.rhs1(d, W + h / 2 * k2)
            k4 = dgsem.rhs1(d, W + h * k3)
            W = W + h / 6 * (k1 + 2 * k2 + 2 * k3 + k4)
        return W

    ref = rk4(W0, 200)
    errs = []
    for n_steps in (1, 2):
        H = hbpc.HBPC(d, 4, 0, implicit.NewtonOpts(rtol=1e-12, gmres_rtol=1e-10, jvp_mode="exact"))
        W = W0.copy()
        for _ in range(n_steps):
            W = H.step(W, T / n_steps)
        errs.append(np.linalg.norm(W - ref) / np.linalg.norm(ref))
    eoc = np.log2(errs[0] / errs[1])
    assert errs[1] < 1e-5 and abs(eoc - 4) < 0.4, (errs, eoc)
