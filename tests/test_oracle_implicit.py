"""Pins for oracle.implicit: residual, JVPs, BJ_ext, GMRES, Newton
(S:406-476).  CPU only."""
import json
import math
import os

import numpy as np
import pytest

from oracle import basis, dgsem, implicit, physics

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def make(kind, N, nx, ny, **kw):
    eq = physics.Equation(kind, **kw)
    return dgsem.Disc(basis.build_basis(N, "gll"), dgsem.Mesh(2, nx, ny), eq)


def euler_state(d, seed, amp=0.05):
    rng = np.random.default_rng(seed)
    W = np.zeros(d.field_shape())
    for v, x in enumerate([1.0, 0.3, -0.2, 2.5]):
        W[:, :, v] = x
    return W.reshape(-1) * (1 + amp * rng.uniform(-1, 1, d.n))


def assembled_jacobian(d, a1, a2, dt, b, W, sig, h=1e-6):
    """Brute force: central differences of the residual G(X) column by column."""
    n = d.n
    J = np.zeros((2 * n, 2 * n))
    X = np.concatenate([W, sig])
    for c in range(2 * n):
        e = np.zeros(2 * n)
        e[c] = h * max(1.0, abs(X[c]))
        Gp = np.concatenate(implicit.residual(d, a1, a2, dt, b, *np.split(X + e, 2)))
        Gm = np.concatenate(implicit.residual(d, a1, a2, dt, b, *np.split(X - e, 2)))
        J[:, c] = (Gp - Gm) / (2 * e[c])
    return J


def test_residual_identities():
    """sigma = R1(W) -> G2 = 0 exactly; dt = 0, b = W -> G = 0."""
    d = make("euler", 2, 3, 3)
    W = euler_state(d, 0)
    sig = dgsem.rhs1(d, W)
    G1, G2 = implicit.residual(d, 0.5, 1 / 6, 0.01, W, W, sig)
    assert np.all(G2 == 0.0)
    G1, G2 = implicit.residual(d, 0.5, 1 / 6, 0.0, W, W, sig)
    assert np.all(G1 == 0.0)


def test_exact_jvp_equals_assembled_jacobian():
    """Tiny mesh (3x3 elements, N=2, Euler, 2n = 648): the EXACT JVP equals
    the brute-force assembled Jacobian of G times dX; the block structure of
    eq:nonlinear_eqsys and the identity dR2/dsigma = dR1/dW hold."""
    d = make("euler", 2, 3, 3)
    n = d.n
    W = euler_state(d, 1)
    rng = np.random.default_rng(2)
    sig = dgsem.rhs1(d, W) + 0.1 * rng.standard_normal(n)
    b = W + 0.01 * rng.standard_normal(n)
    a1, a2, dt = 0.5, 1.0 / 6.0, 0.05
    c2 = a2 * dt * dt / 2
    J = assembled_jacobian(d, a1, a2, dt, b, W, sig)
    # block structure
    np.testing.assert_allclose(J[n:, n:], np.eye(n), atol=1e-8)
    K = -J[n:, :n]                                   # dR1/dW
    np.testing.assert_allclose(J[:n, n:], c2 * K, atol=1e-8 * np.abs(K).max())
    for t in range(3):
        dX = rng.standard_normal(2 * n)
        top, bot = implicit.jvp_exact(d, a1, a2, dt, W, sig, dX[:n], dX[n:])
        ref = J @ dX
        assert np.linalg.norm(np.concatenate([top, bot]) - ref) <= 1e-8 * np.linalg.norm(ref)


def test_hessian_zero_for_advection():
    d = make("advection", 2, 3, 3, a=(0.6, 0.9))
    rng = np.random.default_rng(3)
    W, sig, dW, ds = (rng.standard_normal(d.n) for _ in range(4))
    top, bot = implicit.jvp_exact(d, 0.5, 1 / 6, 0.1, W, sig, dW, ds)
    lt, lb = implicit.jvp_linear(d, 0.5, 1 / 6, 0.1, dW, ds)
    np.testing.assert_allclose(top, lt, atol=1e-12)
    np.testing.assert_allclose(bot, lb, atol=1e-12)


def test_fd_jvp_error_model():
    """FD JVP (eq:MatrixFree_nonlinear) agrees with EXACT to O(sqrt(eps))."""
    d = make("euler", 3, 4, 4)
    W = euler_state(d, 4)
    rng = np.random.default_rng(5)
    sig = dgsem.rhs1(d, W)
    dW = rng.standard_normal(d.n); dW /= np.linalg.norm(dW)
    ds = rng.standard_normal(d.n); ds /= np.linalg.norm(ds)
    ex = np.concatenate(implicit.jvp_exact(d, 0.5, 1 / 6, 0.02, W, sig, dW, ds))
    for lit in (False, True):
        fd = np.concatenate(implicit.jvp_fd(d, 0.5, 1 / 6, 0.02, W, sig, dW, ds, sigma_literal=lit))
        assert np.linalg.norm(fd - ex) <= 1e-5 * np.linalg.norm(ex)


def test_fd_jvp_advection_vs_linear():
    """advection FD path and exact linear path agree within 1e-6."""
    d = make("advection", 3, 4, 4, a=(1.0, 1.0))
    rng = np.random.default_rng(6)
    W, sig, dW, ds = (rng.standard_normal(d.n) for _ in range(4))
    fd = np.concatenate(implicit.jvp_fd(d, 1.0, 1.0, 0.01, W, sig, dW, ds))
    li = np.concatenate(implicit.jvp_linear(d, 1.0, 1.0, 0.01, dW, ds))
    assert np.linalg.norm(fd - li) <= 1e-6 * np.linalg.norm(li)


def test_eps_fd_example_and_zero_guard():
    g = GOLD["eps_fd"]
    v = np.zeros(10); v[0] = g["norm"]
    eps = implicit.fd_eps(v, eps_machine=g["eps_machine"])
    assert eps == pytest.approx(g["eps_fd"], rel=g["rel_tol"])
    # with eps_machine = 2^-52 (reading R7): sqrt(2^-52)/2 = 2^-27 exactly
    assert implicit.fd_eps(v) == 2.0 ** -27
    assert implicit.fd_eps(np.zeros(3)) is None
    d = make("euler", 2, 2, 2)
    W = euler_state(d, 7)
    z = np.zeros(d.n)
    top, bot = implicit.jvp_fd(d, 0.5, 1 / 6, 0.1, W, dgsem.rhs1(d, W), z, z)
    assert np.all(top == 0) and np.all(bot == 0)


def test_element_jacobian_brute_force():
    """K_i (coloured dual seeds) equals central differences of R1 restricted
    to element i with the perturbation confined to element i."""
    d = make("euler", 2, 2, 3)
    W = euler_state(d, 8)
    K = implicit.element_jacobians(d, W)
    m = d.m
    h = 1e-6
    for e in (0, 3):
        for c in (0, 5, m - 1):
            x = np.zeros(d.n); x[e * m + c] = h
            col = (dgsem.rhs1(d, W + x) - dgsem.rhs1(d, W - x))[e * m:(e + 1) * m] / (2 * h)
            np.testing.assert_allclose(K[e][:, c], col, rtol=1e-7, atol=1e-6)


def test_element_jacobian_ns_two_hop():
    """NS-BR1: the diagonal block includes the path through the neighbours'
    lifted gradients (coloring period > stencil radius 2)."""
    d = make("navier_stokes", 2, 4, 4, mu=0.05)
    W = euler_state(d, 9)
    K = implicit.element_jacobians(d, W)
    m, h, e = d.m, 1e-6, 5
    for c in (1, 17):
        x = np.zeros(d.n); x[e * m + c] = h
        col = (dgsem.rhs1(d, W + x) - dgsem.rhs1(d, W - x))[e * m:(e + 1) * m] / (2 * h)
        np.testing.assert_allclose(K[e][:, c], col, rtol=1e-7, atol=1e-6)


@pytest.mark.parametrize("kind", ["advection", "euler"])
def test_bjext_identities(kind):
    """P P^-1 = I per element; commutation A B = B A (P:311,
    S:490); the literal D,E,F,G apply equals the S+K form."""
    d = make(kind, 2, 2, 2, a=(1.0, 0.5))
    W = euler_state(d, 10) if kind == "euler" else np.random.default_rng(0).standard_normal(d.n)
    pc = implicit.BJExt(d, W, 0.5, 1 / 6, 0.3)
    m = d.m
    I = np.eye(m)
    for e in range(d.mesh.n_elem):
        P = np.block([[pc.A[e], pc.B[e]], [pc.C[e], I]])
        Pi = np.block([[pc.D[e], pc.E[e]], [pc.F[e], pc.G[e]]])
        assert np.abs(P @ Pi - np.eye(2 * m)).max() < 1e-10
        assert np.abs(pc.A[e] @ pc.B[e] - pc.B[e] @ pc.A[e]).max() < 1e-11 * max(1, np.abs(pc.B[e]).max() * np.abs(pc.A[e]).max())
    rng = np.random.default_rng(11)
    x, y = rng.standard_normal(d.n), rng.standard_normal(d.n)
    t1, b1 = pc.apply(x, y)
    t2, b2 = pc.apply_sk(x, y)
    assert np.abs(t1 - t2).max() < 1e-11 * np.abs(t1).max()
    assert np.abs(b1 - b2).max() < 1e-11 * np.abs(b1).max()


def test_bjext_dt_zero():
    """dt = 0 -> P^-1 = [[I, 0], [K, I]]."""
    d = make("euler", 2, 2, 2)
    W = euler_state(d, 12)
    pc = implicit.BJExt(d, W, 1.0, 1.0, 0.0)
    rng = np.random.default_rng(13)
    x, y = rng.standard_normal(d.n), rng.standard_normal(d.n)
    t, b = pc.apply(x, y)
    np.testing.assert_allclose(t, x, atol=1e-14)
    Kx = (pc.K @ x.reshape(-1, d.m, 1)).reshape(-1)
    np.testing.assert_allclose(b, Kx + y, atol=1e-12)


def test_element_hessian_brute_force():
    """H_i (hyper-dual seeds) equals central differences of R2(., sigma)
    restricted to element i with the W perturbation confined to element i."""
    d = make("euler", 2, 3, 3)
    W = euler_state(d, 20)
    sig = dgsem.rhs1(d, W) * (1 + 0.1 * np.random.default_rng(21).standard_normal(d.n))
    H = implicit.element_hessian_blocks(d, W, sig)
    m, h = d.m, 1e-6
    for e in (0, 4):
        for c in (0, 7, m - 1):
            x = np.zeros(d.n); x[e * m + c] = h
            col = (dgsem.rhs2(d, W + x, sig) - dgsem.rhs2(d, W - x, sig))[e * m:(e + 1) * m] / (2 * h)
            np.testing.assert_allclose(H[e][:, c], col, rtol=1e-6, atol=1e-5 * np.abs(col).max())


def test_bjext_h_identities():
    """BJ^H_ext: P P^-1 = I per element with A^H = I - a1 dt K + c2 H;
    the literal D,E,F,G apply equals the S+K form u = S(x - c2 K y), (u, y + K u)."""
    d = make("euler", 2, 3, 3)
    W = euler_state(d, 22)
    pc = implicit.BJExtH(d, W, dgsem.rhs1(d, W), 0.5, 1 / 6, 0.3)
    assert np.abs(pc.H).max() > 0.0                      # the Hessian term is present for Euler
    m = d.m
    I = np.eye(m)
    for e in range(d.mesh.n_elem):
        P = np.block([[pc.A[e], pc.B[e]], [pc.C[e], I]])
        Pi = np.block([[pc.D[e], pc.E[e]], [pc.F[e], pc.G[e]]])
        assert np.abs(P @ Pi - np.eye(2 * m)).max() < 1e-10
    rng = np.random.default_rng(23)
    x, y = rng.standard_normal(d.n), rng.standard_normal(d.n)
    t1, b1 = pc.apply(x, y)
    t2, b2 = pc.apply_sk(x, y)
    assert np.abs(t1 - t2).max() < 1e-11 * np.abs(t1).max()
    assert np.abs(b1 - b2).max() < 1e-11 * np.abs(b1).max()


def test_bjext_h_reduces_to_bjext():
    """Linear flux: R2(W, sigma) = R1(sigma) does not depend on W, so H = 0 and
    BJ^H_ext == BJ_ext; dt = 0 gives [[I, 0], [K, I]] for both."""
    d = make("advection", 2, 3, 3, a=(1.0, 0.5))
    W = np.random.default_rng(24).standard_normal(d.n)
    ph = implicit.BJExtH(d, W, dgsem.rhs1(d, W), 0.5, 1 / 6, 0.3)
    pb = implicit.BJExt(d, W, 0.5, 1 / 6, 0.3)
    assert np.abs(ph.H).max() == 0.0
    rng = np.random.default_rng(25)
    x, y = rng.standard_normal(d.n), rng.standard_normal(d.n)
    for u, v in zip(ph.apply(x, y), pb.apply(x, y)):
        assert np.abs(u - v).max() < 1e-12 * np.abs(v).max()
    de = make("euler", 2, 2, 2)
    We = euler_state(de, 26)
    p0 = implicit.BJExtH(de, We, dgsem.rhs1(de, We), 1.0, 1.0, 0.0)
    xe, ye = rng.standard_normal(de.n), rng.standard_normal(de.n)
    t, b = p0.apply(xe, ye)
    np.testing.assert_allclose(t, xe, atol=1e-14)
    np.testing.assert_allclose(b, (p0.K @ xe.reshape(-1, de.m, 1)).reshape(-1) + ye, atol=1e-12)


def test_newton_bjext_h():
    """A stage solve preconditioned with BJ^H_ext converges to the BJ_ext
    solution (same tolerances); the Hessian-including block is at least as good
    an approximation of J ('only a small influence on the iterations')."""
    d = make("euler", 2, 3, 3)
    W0 = euler_state(d, 27)
    dt = 0.02
    b = W0 + 0.5 * dt * dgsem.rhs1(d, W0)
    res = {}
    for kind in ("bjext", "bjext_h"):
        opts = implicit.NewtonOpts(rtol=1e-10, gmres_rtol=1e-10, precond=kind, precond_policy="per_newton")
        st = dict(stage_solves=0, newton_its=0, gmres_its=0, precond_builds=0)
        Wk, _ = implicit.newton_solve(d, 0.5, 1 / 6, dt, b, W0, opts, None, st)
        res[kind] = (Wk, st["gmres_its"])
    assert np.abs(res["bjext"][0] - res["bjext_h"][0]).max() < 1e-9
    assert res["bjext_h"][1] <= res["bjext"][1] + 2


def test_advection_blocks_identical():
    d = make("advection", 3, 4, 4, a=(1.0, 1.0))
    K = implicit.element_jacobians(d, np.zeros(d.n))
    assert np.abs(K - K[0][None]).max() == 0.0


def test_gmres_dense():
    """Identity -> 1 iteration; 20x20 well-conditioned vs LU;
    restart = 2 on a 5x5 system converges; right preconditioning
    returns the same solution."""
    rng = np.random.default_rng(14)
    b = rng.standard_normal(20)
    x, its, ok = implicit.gmres(lambda v: v, b, rtol=1e-12)
    assert its == 1 and ok and np.allclose(x, b)
    A = np.eye(20) * 4 + rng.standard_normal((20, 20))
    x, its, ok = implicit.gmres(lambda v: A @ v, b, rtol=1e-12, restart=30)
    assert ok and np.linalg.norm(x - np.linalg.solve(A, b)) <= 1e-8 * np.linalg.norm(x)
    Minv = np.linalg.inv(np.diag(np.diag(A)))
    x2, its2, ok2 = implicit.gmres(lambda v: A @ v, b, lambda v: Minv @ v, rtol=1e-12, restart=30)
    assert ok2 and np.linalg.norm(x2 - x) <= 1e-8 * np.linalg.norm(x)
    A5 = np.eye(5) * 3 + rng.standard_normal((5, 5))
    b5 = rng.standard_normal(5)
    x5, its5, ok5 = implicit.gmres(lambda v: A5 @ v, b5, rtol=1e-10, restart=2, max_total=500)
    _, its_full, _ = implicit.gmres(lambda v: A5 @ v, b5, rtol=1e-10, restart=5)
    assert ok5 and its5 >= its_full
    assert np.linalg.norm(A5 @ x5 - b5) <= 1e-9 * np.linalg.norm(b5)


def test_newton_linear_one_iteration():
    """Advection: one Newton step when GMRES rtol <= Newton rtol."""
    d = make("advection", 3, 4, 4, a=(1.0, 1.0))
    rng = np.random.default_rng(15)
    Wg = rng.standard_normal(d.n)
    b = rng.standard_normal(d.n)
    stats = dict(newton_its=0, gmres_its=0, precond_builds=0)
    opts = implicit.NewtonOpts(rtol=1e-10, gmres_rtol=1e-11, precond="none")
    W, sig = implicit.newton_solve(d, 0.5, 1 / 6, 0.05, b, Wg, opts, None, stats)
    assert stats["newton_its"] == 1
    G1, G2 = implicit.residual(d, 0.5, 1 / 6, 0.05, b, W, sig)
    assert math.sqrt(G1 @ G1 + G2 @ G2) <= 1e-10 * np.linalg.norm(b) * 100


def test_newton_euler_quadratic():
    """Euler stage solve with BJ_ext converges, and ||G|| drops superlinearly."""
    d = make("euler", 2, 3, 3)
    W0 = euler_state(d, 16, amp=0.02)
    dt = 0.05
    a1, a2 = 0.5, 1 / 6
    b = W0 + a1 * dt * dgsem.rhs1(d, W0)
    pc = implicit.BJExt(d, W0, a1, a2, dt)
    stats = dict(newton_its=0, gmres_its=0, precond_builds=0)
    opts = implicit.NewtonOpts(rtol=1e-12, gmres_rtol=1e-12)
    W, sig = implicit.newton_solve(d, a1, a2, dt, b, W0, opts, pc, stats)
    G1, G2 = implicit.residual(d, a1, a2, dt, b, W, sig)
    assert math.sqrt(G1 @ G1 + G2 @ G2) < 1e-11 * np.linalg.norm(b)
    assert stats["newton_its"] <= 4
    # sigma-consistency
    assert np.linalg.norm(sig - dgsem.rhs1(d, W)) <= 1e-10 * np.linalg.norm(sig)


def test_schur_operator_is_the_schur_complement():
    """eq:nonlinear_eqsys_Schur: J = [[A, B], [C, I]] with B = c2 K, C = -K, so the
    Schur complement A - B C = I - a1 dt K + c2 dR2/dW + c2 K^2 is applied by the
    top block of J (v, K v) (EXACT products, K v = R2(W, v)); checked against the
    blocks of the brute-force assembled Jacobian of G (3x3 Euler, N = 2)."""
    d = make("euler", 2, 3, 3)
    n = d.n
    W = euler_state(d, 40)
    sig = dgsem.rhs1(d, W) * (1 + 1e-2 * np.random.default_rng(41).standard_normal(n))
    a1, a2, dt = 0.5, 1 / 6, 0.05
    b = W.copy()
    J = assembled_jacobian(d, a1, a2, dt, b, W, sig)
    A, B, C = J[:n, :n], J[:n, n:], J[n:, :n]
    np.testing.assert_allclose(J[n:, n:], np.eye(n), atol=1e-6)
    JS = A - B @ C
    v = np.random.default_rng(42).standard_normal(n)
    Kv = dgsem.rhs2(d, W, v)
    top, _ = implicit.jvp_exact(d, a1, a2, dt, W, sig, v, Kv)
    np.testing.assert_allclose(top, JS @ v, rtol=1e-6, atol=1e-6 * np.abs(top).max())


@pytest.mark.parametrize("precond", ["bjext_h", "none"])
def test_newton_schur_equals_extended(precond):
    """The Schur-complement Newton iteration solves the same stage
    equation: same W and sigma as the extended system to the Newton tolerance."""
    d = make("euler", 2, 3, 3)
    W0 = euler_state(d, 43)
    dt = 0.02
    b = W0 + 0.5 * dt * dgsem.rhs1(d, W0)
    out = []
    for schur in (False, True):
        opts = implicit.NewtonOpts(rtol=1e-10, gmres_rtol=1e-10, precond=precond, precond_policy="per_newton",
                                   schur=schur)
        W, sig = implicit.newton_solve(d, 0.5, 1 / 6, dt, b, W0, opts)
        out.append((W, sig))
    assert np.abs(out[0][0] - out[1][0]).max() < 1e-9
    assert np.abs(out[0][1] - out[1][1]).max() < 1e-8 * np.abs(out[0][1]).max()
