"""NEXT-3: BR2 lifting for Navier-Stokes (reading R33) -- GPU
(C-ABI) vs the oracle's Equation(lifting="br2").  The volume viscous flux keeps
the global (BR1-type) lifted gradient; each face uses the gradient of its own
local lifting (strong form), scaled by eta_BR2.

Tolerances as test_gpu_parity.py: operators / EXACT JVP <= 1e-11, FD JVP
within max(1e-11, 4 delta_FD), BJ_ext apply <= 1e-11 max(1, cond/1e4), end of
run <= 1e-8."""
import numpy as np
import pytest

from oracle import dgsem, hbpc, implicit
from paper_2109_04804_b200 import inputs
from gpu_common import make_pair, ns_ic, rel, to_gpu, to_np, SEED

pytestmark = pytest.mark.gpu

TWO_PI = 2 * np.pi
BR2_CASES = [
    # (N, nx, ny, eta, nodes)
    (3, 4, 4, 2.0, "gll"),
    (5, 5, 3, 4.0, "gll"),
    (2, 6, 5, 1.0, "gll"),
    (3, 4, 4, 2.0, "gl"),        # the paper's own NS discretisation: GL nodes + BR2
    (4, 3, 5, 1.0, "gl"),
]


def _pair(N, nx, ny, eta, nodes="gll", **kw):
    return make_pair("navier_stokes", N, nx, ny, bounds=(0.0, TWO_PI, 0.0, TWO_PI), a=(1.0, -0.6), mu=0.05,
                     lifting="br2", eta_br2=eta, nodes=nodes, **kw)


@pytest.mark.parametrize("case", BR2_CASES)
def test_br2_operators(case):
    d, ctx = _pair(*case)
    W = ns_ic(d, SEED + 91)
    sig = dgsem.rhs1(d, W) * (1 + 1e-2 * inputs.random_field(d.n, SEED + 92))
    assert rel(to_np(ctx.rhs(to_gpu(W))), dgsem.rhs1(d, W)) <= 1e-11
    assert rel(to_np(ctx.rhs(to_gpu(W), to_gpu(sig))), dgsem.rhs2(d, W, sig)) <= 1e-11
    b = W * (1 + 1e-3 * inputs.random_field(d.n, SEED + 93))
    a1, a2, dt = 0.5, 1 / 6, 0.02
    G1o, G2o = implicit.residual(d, a1, a2, dt, b, W, sig)
    G1g, G2g = ctx.residual(a1, a2, dt, to_gpu(b), to_gpu(W), to_gpu(sig))
    assert rel(np.concatenate([to_np(G1g), to_np(G2g)]), np.concatenate([G1o, G2o])) <= 1e-11
    dW = inputs.random_field(d.n, SEED + 94, unit_norm=True)
    ds = inputs.random_field(d.n, SEED + 95, unit_norm=True)
    to, bo = implicit.jvp_exact(d, a1, a2, dt, W, sig, dW, ds)
    tg, bg = ctx.jvp(a1, a2, dt, to_gpu(W), to_gpu(sig), to_gpu(dW), to_gpu(ds), mode="exact")
    assert rel(np.concatenate([to_np(tg), to_np(bg)]), np.concatenate([to, bo])) <= 1e-11
    eps = implicit.fd_eps(dW)
    fo = np.concatenate(implicit.jvp_fd(d, a1, a2, dt, W, sig, dW, ds, eps_override=(eps, None)))
    delta = rel(fo, np.concatenate([to, bo]))
    tg, bg = ctx.jvp(a1, a2, dt, to_gpu(W), to_gpu(sig), to_gpu(dW), to_gpu(ds), mode="fd",
                     eps_override=(eps, None))
    assert rel(np.concatenate([to_np(tg), to_np(bg)]), fo) <= max(1e-11, 4 * delta)


def test_br2_differs_from_br1():
    """The GPU BR2 operator is not the BR1 one (the jump terms reach the face flux)."""
    d, ctx = _pair(3, 4, 4, 2.0)
    _, ctx1 = make_pair("navier_stokes", 3, 4, 4, bounds=(0.0, TWO_PI, 0.0, TWO_PI), a=(1.0, -0.6), mu=0.05)
    W = to_gpu(ns_ic(d, SEED + 96))
    assert rel(to_np(ctx.rhs(W)), to_np(ctx1.rhs(W))) > 1e-6


@pytest.mark.parametrize("nodes", ["gll", "gl"])
def test_br2_precond(nodes):
    """BJ_ext by the two-hop colouring with BR2 face gradients."""
    d, ctx = _pair(2, 4, 3, 2.0, nodes=nodes)
    W = ns_ic(d, SEED + 97)
    a1, a2, dt = 1.0 / 6.0, 1.0 / 54.0, 0.05
    pc = implicit.BJExt(d, W, a1, a2, dt)
    ctx.precond_build(a1, a2, dt, to_gpu(W))
    cond = max(np.linalg.cond(M) for M in pc.M)
    x = inputs.random_field(d.n, SEED + 98)
    y = inputs.random_field(d.n, SEED + 99)
    to, bo = pc.apply(x, y)
    tg, bg = ctx.precond_apply(to_gpu(x), to_gpu(y))
    assert rel(np.concatenate([to_np(tg), to_np(bg)]), np.concatenate([to, bo])) <= 1e-11 * max(1, cond / 1e4)


@pytest.mark.parametrize("nodes", ["gll", "gl"])
def test_br2_end_of_run(nodes):
    """HBPC(4,0), BJ_ext, 2 steps on 4x4 elements, N = 3: end of run vs the oracle <= 1e-8.
    dt = 0.004: at dt = 0.01 the eta = 2 stage Newton sits at the edge of its basin on this
    coarse mesh (BR2 diverges there on 6x6, N = 2, in the oracle and on the GPU);
    whether it converges then hinges on rounding-level differences of the preconditioner
    (Gauss-Jordan panel width 16 vs 32, r02f/r02g: identical S to 1e-15, opposite outcomes)."""
    d, ctx = _pair(3, 4, 4, 2.0, nodes=nodes, q=4, kmax=0, gmres_rtol=1e-10, newton_rtol=1e-10)
    W0 = ns_ic(d, SEED + 100, rel_noise=1e-3)
    dt = 0.004
    H = hbpc.HBPC(d, 4, 0, implicit.NewtonOpts(rtol=1e-10, gmres_rtol=1e-10))
    Wo = W0.copy()
    st = dict(stage_solves=0, newton_its=0, gmres_its=0, precond_builds=0)
    Wg = to_gpu(W0)
    for _ in range(2):
        Wo = H.step(Wo, dt, st)
        ctx.step(dt, Wg)
    assert rel(to_np(Wg), Wo) <= 1e-8


@pytest.mark.parametrize("px,py,nodes", [(2, 2, "gll"), (2, 1, "gll"), (2, 2, "gl")])
def test_br2_loopback_operators_bitwise(px, py, nodes):
    """BR2 across loopback ranks: the neighbour ranks' face gradients arrive by the
    face-buffer halo and every rank's operator output equals its block of the
    single-rank result bit for bit (GLL; GL: the ghost W traces are interpolated by
    the sender, so to rounding); one HBPC(4,0) step <= 1e-10 vs one rank."""
    import torch
    from paper_2109_04804_b200 import hbpdc
    from test_gpu_partition import _block, _run_threads
    N, nx, ny, eta = 2, 6, 6, 2.0
    d, ctx1 = _pair(N, nx, ny, eta, nodes=nodes)
    W = ns_ic(d, SEED + 101)
    sig = dgsem.rhs1(d, W) * (1 + 1e-2 * inputs.random_field(d.n, SEED + 102))
    dW = inputs.random_field(d.n, SEED + 103, unit_norm=True)
    ds = inputs.random_field(d.n, SEED + 104, unit_norm=True)
    a1, a2, dt = 1 / 6, 1 / 54, 0.02
    eps = implicit.fd_eps(dW)

    def ops(ctx, blk):
        Wg, sg, dWg, dsg = (to_gpu(blk(x)) for x in (W, sig, dW, ds))
        torch.cuda.synchronize()
        out = {"R1": ctx.rhs(Wg), "R2": ctx.rhs(Wg, sg),
               "exact": ctx.jvp(a1, a2, dt, Wg, sg, dWg, dsg, mode="exact"),
               "fd": ctx.jvp(a1, a2, dt, Wg, sg, dWg, dsg, mode="fd", eps_override=(eps, None))}
        ctx.precond_build(a1, a2, dt, Wg)
        out["pc"] = ctx.precond_apply(dWg, dsg)
        torch.cuda.synchronize()
        return {k: (np.concatenate([to_np(x) for x in v]) if isinstance(v, tuple) else to_np(v))
                for k, v in out.items()}

    ref = ops(ctx1, lambda x: x)
    assert rel(ref["R1"], dgsem.rhs1(d, W)) <= 1e-11
    group = hbpdc.LoopbackGroup(px * py)
    ctxs = [hbpdc.Context(dim=2, equation="navier_stokes", N=N, nx=nx, ny=ny, bounds=(0.0, TWO_PI, 0.0, TWO_PI),
                          a=(1.0, -0.6), mu=0.05, lifting="br2", eta_br2=eta, q=4, kmax=0, gmres_rtol=1e-10,
                          newton_rtol=1e-10, rank=r, nranks=px * py, px=px, py=py, comm="loopback",
                          loopback=group, stream=torch.cuda.Stream(), nodes=nodes)
            for r in range(px * py)]
    try:
        def blk_of(c):
            return lambda x: _block(x, 2, nx, ny, d.m, c.ex0, c.ey0, c.nx_local, c.ny_local)
        outs = _run_threads([lambda c=c: ops(c, blk_of(c)) for c in ctxs])
        for c, o in zip(ctxs, outs):
            blk = blk_of(c)
            for key, r in ref.items():
                rb = np.concatenate([blk(r[:d.n]), blk(r[d.n:])]) if r.size == 2 * d.n else blk(r)
                if nodes == "gll":
                    assert np.array_equal(o[key], rb), (key, c.rank, np.abs(o[key] - rb).max())
                else:
                    assert rel(o[key], rb) <= (1e-6 if key == "fd" else 1e-12), (key, c.rank, rel(o[key], rb))
        # one step, partitioned vs single rank
        _, c1 = _pair(N, nx, ny, eta, nodes=nodes, q=4, kmax=0, gmres_rtol=1e-10, newton_rtol=1e-10)
        W0 = ns_ic(d, SEED + 105, rel_noise=1e-3)
        W1 = to_gpu(W0)
        c1.step(0.004, W1)
        W1 = to_np(W1)

        def run(c):
            Wl = to_gpu(blk_of(c)(W0))
            torch.cuda.synchronize()
            c.step(0.004, Wl)
            torch.cuda.synchronize()
            return to_np(Wl)
        outs = _run_threads([lambda c=c: run(c) for c in ctxs])
        for c, Wl in zip(ctxs, outs):
            assert rel(Wl, blk_of(c)(W1)) <= 1e-10, (c.rank, rel(Wl, blk_of(c)(W1)))
    finally:
        for c in ctxs:
            c.close()
        group.close()
