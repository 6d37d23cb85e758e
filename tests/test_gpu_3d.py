"""NEXT-4: 3D hexahedral elements on the GPU (advection and Euler, GLL,
one rank) vs the CPU oracle's 3D operators (tests/test_oracle_3d.py pins
them).  Same tolerances as 2D: operators / JVPs <= 1e-11, BJ_ext <= 1e-11
max(1, cond/1e4), end of run <= 1e-8."""
import numpy as np
import pytest

from oracle import basis, dgsem, hbpc, implicit, physics
from paper_2109_04804_b200 import inputs
from gpu_common import rel, to_gpu, to_np, SEED

pytestmark = pytest.mark.gpu

TWO_PI = 2 * np.pi


def pair3(kind, N, n, bounds=(0.0, TWO_PI), a=(1.0, -0.6, 0.4), q=4, kmax=0, **kw):
    from paper_2109_04804_b200 import hbpdc
    eq = physics.Equation(kind, dim=3, a=tuple(a), numflux=kw.get("flux", "llf"))
    me = dgsem.Mesh(3, n[0], n[1], bounds[0], bounds[1], bounds[0], bounds[1], nz=n[2], zmin=bounds[0],
                    zmax=bounds[1])
    d = dgsem.Disc(basis.build_basis(N, "gll"), me, eq)
    ctx = hbpdc.Context(dim=3, equation=kind, N=N, nx=n[0], ny=n[1], nz=n[2],
                        bounds=(bounds[0], bounds[1]) * 3, a=a, q=q, kmax=kmax, **kw)
    return d, ctx


def state(d, kind, seed, amp=1e-2):
    X, Y, Z = d.node_coords()
    W = inputs.initial_state("TGV3" if kind == "euler" else "ADV3", (X, Y, Z))
    return inputs.perturbed_state(W, seed, amp) if kind == "euler" else W + inputs.random_field(d.n, seed, amp)


CASES = [("euler", 2, (3, 2, 2)), ("euler", 2, (2, 3, 3)), ("euler", 3, (3, 2, 3)),
         ("advection", 2, (3, 3, 2)), ("advection", 3, (2, 2, 3))]


@pytest.mark.parametrize("case", CASES)
def test_node_coords_3d(case):
    d, ctx = pair3(*case)
    for a, b in zip(ctx.node_coords(), d.node_coords()):
        np.testing.assert_allclose(a, b, rtol=0, atol=1e-13)


@pytest.mark.parametrize("case", CASES)
def test_operators_3d(case):
    """R1, R2, residual, EXACT JVP, FD JVP (same eps) and the LINEAR JVP (advection)."""
    kind = case[0]
    d, ctx = pair3(*case)
    W = state(d, kind, SEED + 301)
    sig = dgsem.rhs1(d, W) * (1 + 1e-2 * inputs.random_field(d.n, SEED + 302))
    assert rel(to_np(ctx.rhs(to_gpu(W))), dgsem.rhs1(d, W)) <= 1e-11
    assert rel(to_np(ctx.rhs(to_gpu(W), to_gpu(sig))), dgsem.rhs2(d, W, sig)) <= 1e-11
    b = W * (1 + 1e-3 * inputs.random_field(d.n, SEED + 303))
    a1, a2, dt = 0.5, 1 / 6, 0.02
    G1o, G2o = implicit.residual(d, a1, a2, dt, b, W, sig)
    G1g, G2g = ctx.residual(a1, a2, dt, to_gpu(b), to_gpu(W), to_gpu(sig))
    assert rel(np.concatenate([to_np(G1g), to_np(G2g)]), np.concatenate([G1o, G2o])) <= 1e-11
    dW = inputs.random_field(d.n, SEED + 304, unit_norm=True)
    ds = inputs.random_field(d.n, SEED + 305, unit_norm=True)
    to, bo = implicit.jvp_exact(d, a1, a2, dt, W, sig, dW, ds)
    tg, bg = ctx.jvp(a1, a2, dt, to_gpu(W), to_gpu(sig), to_gpu(dW), to_gpu(ds), mode="exact")
    assert rel(np.concatenate([to_np(tg), to_np(bg)]), np.concatenate([to, bo])) <= 1e-11
    if kind == "advection":
        to, bo = implicit.jvp_linear(d, a1, a2, dt, dW, ds)
        tg, bg = ctx.jvp(a1, a2, dt, to_gpu(W), to_gpu(sig), to_gpu(dW), to_gpu(ds), mode="linear")
        assert rel(np.concatenate([to_np(tg), to_np(bg)]), np.concatenate([to, bo])) <= 1e-11
    else:
        eps = 1e-6
        to, bo = implicit.jvp_fd(d, a1, a2, dt, W, sig, dW, ds, eps_override=(eps, None))
        te, be = implicit.jvp_exact(d, a1, a2, dt, W, sig, dW, ds)
        delta = rel(np.concatenate([to, bo]), np.concatenate([te, be]))
        tg, bg = ctx.jvp(a1, a2, dt, to_gpu(W), to_gpu(sig), to_gpu(dW), to_gpu(ds), mode="fd",
                         eps_override=(eps, None))
        assert rel(np.concatenate([to_np(tg), to_np(bg)]), np.concatenate([to, bo])) <= max(1e-11, 4 * delta)


@pytest.mark.parametrize("case", [("euler", 2, (2, 3, 2)), ("euler", 2, (2, 2, 3)), ("euler", 3, (2, 2, 2)),
                                  ("advection", 3, (2, 2, 2))])
def test_bjext_3d(case):
    """BJ_ext in 3D: S_i = (I - a1 dt K_i + c2 K_i^2)^-1 (m up to 5 * 4^3 = 320: the 384-thread
    Gauss-Jordan and the m > 256 GEMV) and P^-1 X vs the oracle."""
    kind = case[0]
    d, ctx = pair3(*case)
    W = state(d, kind, SEED + 311)
    a1, a2, dt = 1.0 / 6.0, 1.0 / 54.0, 0.05
    pc = implicit.BJExt(d, W, a1, a2, dt)
    ctx.precond_build(a1, a2, dt, to_gpu(W))
    cond = max(np.linalg.cond(M) for M in pc.M)
    S, shared = ctx.precond_export()
    So = pc.S[:1] if shared else pc.S
    assert np.linalg.norm(to_np(S).reshape(So.shape) - So) / np.linalg.norm(So) <= 1e-11 * max(1, cond / 1e4)
    x = inputs.random_field(d.n, SEED + 312)
    y = inputs.random_field(d.n, SEED + 313)
    to, bo = pc.apply(x, y)
    tg, bg = ctx.precond_apply(to_gpu(x), to_gpu(y))
    assert rel(np.concatenate([to_np(tg), to_np(bg)]), np.concatenate([to, bo])) <= 1e-11 * max(1, cond / 1e4)


@pytest.mark.parametrize("kind,N,n,q,kmax,sstep", [("euler", 2, (3, 3, 3), 4, 0, 1), ("euler", 3, (3, 3, 3), 4, 0, 8),
                                                  ("euler", 2, (2, 2, 3), 6, 2, 4), ("advection", 3, (2, 2, 2), 6, 2, 1)])
def test_end_of_run_3d(kind, N, n, q, kmax, sstep):
    """The paper's 3D case in its inviscid scope: Taylor-Green initial data (P:1088-1091,
    reading R35) on [0, 2 pi]^3, HBPC(q, k_max), BJ_ext, FD JVP, 2 steps of an acoustic
    element-CFL 1 step; GPU (s-step or DCGS2 Arnoldi) vs the oracle <= 1e-8."""
    d, ctx = pair3(kind, N, n, q=q, kmax=kmax, gmres_rtol=1e-10, newton_rtol=1e-10, gmres_sstep=sstep)
    X, Y, Z = d.node_coords()
    W0 = inputs.initial_state("TGV3" if kind == "euler" else "ADV3", (X, Y, Z))
    h = TWO_PI / max(n)
    dt = 0.5 / (3 * (1.0 + 1.1) / h) if kind == "euler" else 1.0 / (2.0 / h)      # acoustic element CFL 0.5
    H = hbpc.HBPC(d, q, kmax, implicit.NewtonOpts(rtol=1e-10, gmres_rtol=1e-10))
    Wo = W0.copy()
    for _ in range(2):
        Wo = H.step(Wo, dt)
    Wg = to_gpu(W0)
    for _ in range(2):
        ctx.step(dt, Wg)
    assert rel(to_np(Wg), Wo) <= 1e-8
