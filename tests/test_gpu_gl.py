"""NEXT-3: Gauss-Legendre nodes (the element has no node on its edge, so
the face trace is the line sum sum_l l_l(+-1) W_l and every node receives the
surface terms weighted by lhat_i(+-1), eq:DGSEM_wt) -- GPU (C-ABI) vs the
oracle's build_basis(N, "gl") discretisation.

Tolerances as test_gpu_parity.py: operators / JVPs <= 1e-11 relative, FD JVP
within max(1e-11, 4 delta_FD), BJ_ext build <= 1e-11 max(1, cond/1e4), end of
run <= 1e-8.  Sizes span several CTAs with a ragged last CTA."""
import numpy as np
import pytest

from oracle import dgsem, hbpc, implicit
from paper_2109_04804_b200 import inputs
from gpu_common import adv_ic, euler_ic, make_pair, ns_ic, rel, to_gpu, to_np, SEED

pytestmark = pytest.mark.gpu

GL_CASES = [
    # (kind, N, nx, ny)
    ("advection", 3, 10, None),
    ("advection", 4, 7, 5),
    ("euler", 3, 5, 4),
    ("euler", 7, 3, 3),
    ("euler", 1, 6, 5),
    ("navier_stokes", 3, 4, 4),
    ("navier_stokes", 5, 3, 5),
]
NS_MU = 0.05      # viscous terms O(1) relative, as test_gpu_parity.py


def _pair(kind, N, nx, ny, **kw):
    a = (1.0, 0.0) if ny is None else (1.0, -0.6)
    if kind == "navier_stokes":
        kw.setdefault("mu", NS_MU)
        kw.setdefault("bounds", (0.0, 2 * np.pi, 0.0, 2 * np.pi))
    return make_pair(kind, N, nx, ny, a=a, nodes="gl", **kw)


def _state(d, kind, seed):
    return {"advection": adv_ic, "euler": euler_ic, "navier_stokes": ns_ic}[kind](d, seed)


@pytest.mark.parametrize("case", GL_CASES)
def test_gl_node_coords(case):
    d, ctx = _pair(*case)
    for a, b in zip(ctx.node_coords(), d.node_coords()):
        np.testing.assert_allclose(a, b, rtol=0, atol=1e-14)


@pytest.mark.parametrize("case", GL_CASES)
def test_gl_operators(case):
    """R1, R2, residual and the JVPs (EXACT for Euler, LINEAR for advection)."""
    kind = case[0]
    d, ctx = _pair(*case)
    W = _state(d, kind, SEED + 61)
    sig = dgsem.rhs1(d, W) * (1 + 1e-2 * inputs.random_field(d.n, SEED + 62))
    assert rel(to_np(ctx.rhs(to_gpu(W))), dgsem.rhs1(d, W)) <= 1e-11
    assert rel(to_np(ctx.rhs(to_gpu(W), to_gpu(sig))), dgsem.rhs2(d, W, sig)) <= 1e-11
    b = W * (1 + 1e-3 * inputs.random_field(d.n, SEED + 63))
    a1, a2, dt = 0.5, 1 / 6, 0.02
    G1o, G2o = implicit.residual(d, a1, a2, dt, b, W, sig)
    G1g, G2g = ctx.residual(a1, a2, dt, to_gpu(b), to_gpu(W), to_gpu(sig))
    assert rel(np.concatenate([to_np(G1g), to_np(G2g)]), np.concatenate([G1o, G2o])) <= 1e-11
    dW = inputs.random_field(d.n, SEED + 64, unit_norm=True)
    ds = inputs.random_field(d.n, SEED + 65, unit_norm=True)
    if kind == "advection":
        z = np.zeros(d.n)
        to, bo = implicit.jvp_linear(d, a1, a2, dt, dW, ds)
        tg, bg = ctx.jvp(a1, a2, dt, to_gpu(z), to_gpu(z), to_gpu(dW), to_gpu(ds), mode="linear")
    else:
        to, bo = implicit.jvp_exact(d, a1, a2, dt, W, sig, dW, ds)
        tg, bg = ctx.jvp(a1, a2, dt, to_gpu(W), to_gpu(sig), to_gpu(dW), to_gpu(ds), mode="exact")
    assert rel(np.concatenate([to_np(tg), to_np(bg)]), np.concatenate([to, bo])) <= 1e-11


@pytest.mark.parametrize("case", [c for c in GL_CASES if c[0] != "advection"])
def test_gl_jvp_fd(case):
    kind = case[0]
    d, ctx = _pair(*case)
    W = _state(d, kind, SEED + 66)
    sig = dgsem.rhs1(d, W) * (1 + 1e-2 * inputs.random_field(d.n, SEED + 67))
    dW = inputs.random_field(d.n, SEED + 68, unit_norm=True)
    ds = inputs.random_field(d.n, SEED + 69, unit_norm=True)
    a1, a2, dt = 1.0, 1.0, 0.01
    eps = implicit.fd_eps(dW)
    fo = np.concatenate(implicit.jvp_fd(d, a1, a2, dt, W, sig, dW, ds, eps_override=(eps, None)))
    ex = np.concatenate(implicit.jvp_exact(d, a1, a2, dt, W, sig, dW, ds))
    delta = rel(fo, ex)
    tg, bg = ctx.jvp(a1, a2, dt, to_gpu(W), to_gpu(sig), to_gpu(dW), to_gpu(ds), mode="fd",
                     eps_override=(eps, None))
    assert rel(np.concatenate([to_np(tg), to_np(bg)]), fo) <= max(1e-11, 4 * delta)


@pytest.mark.parametrize("precond", ["bjext", "bjext_h"])
@pytest.mark.parametrize("case", [("advection", 3, 8, None), ("advection", 2, 6, 4), ("euler", 3, 4, 3),
                                  ("navier_stokes", 2, 4, 3)])
def test_gl_precond(case, precond):
    """BJ_ext / BJ^H_ext on GL nodes: the element blocks see the full line traces
    (Navier-Stokes: K_i and H_i by the two-hop colouring)."""
    kind = case[0]
    d, ctx = _pair(*case, precond=precond)
    W = _state(d, kind, SEED + 70)
    a1, a2, dt = 1.0 / 6.0, 1.0 / 54.0, 0.05
    pc = implicit.make_precond(precond, d, W, a1, a2, dt)
    ctx.precond_build(a1, a2, dt, to_gpu(W))
    cond = max(np.linalg.cond(M) for M in pc.M)
    x = inputs.random_field(d.n, SEED + 71)
    y = inputs.random_field(d.n, SEED + 72)
    to, bo = pc.apply(x, y)
    tg, bg = ctx.precond_apply(to_gpu(x), to_gpu(y))
    assert rel(np.concatenate([to_np(tg), to_np(bg)]), np.concatenate([to, bo])) <= 1e-11 * max(1, cond / 1e4)


def test_gl_free_stream():
    """A uniform Euler state is a steady solution on GL nodes too (the free-stream
    row identity of Dhat, reading R2): |R1| at rounding level."""
    d, ctx = _pair("euler", 5, 4, 3)
    X = d.node_coords()[0]
    W = inputs.layout([np.full_like(X, v) for v in (1.2, 0.3, -0.2, 2.5)], 2)
    r = to_np(ctx.rhs(to_gpu(W)))
    assert np.abs(r).max() <= 1e-12


def _run_oracle(d, q, kmax, W0, dt, steps, **opt):
    H = hbpc.HBPC(d, q, kmax, implicit.NewtonOpts(**opt))
    W = W0.copy()
    st = dict(stage_solves=0, newton_its=0, gmres_its=0, precond_builds=0)
    for _ in range(steps):
        W = H.step(W, dt, st)
    return W


@pytest.mark.parametrize("kind,q,kmax,sstep", [("advection", 6, 2, 1), ("euler", 4, 0, 1), ("euler", 4, 0, 4),
                                               ("navier_stokes", 4, 0, 1)])
def test_gl_end_of_run(kind, q, kmax, sstep):
    """HBPC(q, k_max) with BJ_ext on GL nodes, 2 steps: end of run vs the oracle <= 1e-8."""
    ny = 4
    d, ctx = _pair(kind, 3, 5, ny, q=q, kmax=kmax, gmres_rtol=1e-10, newton_rtol=1e-10, gmres_sstep=sstep)
    W0 = _state(d, kind, SEED + 73)
    dt = 0.02 if kind == "advection" else 0.01
    Wo = _run_oracle(d, q, kmax, W0, dt, 2, rtol=1e-10, gmres_rtol=1e-10)
    Wg = to_gpu(W0)
    for _ in range(2):
        ctx.step(dt, Wg)
    assert rel(to_np(Wg), Wo) <= 1e-8


# ---- element partition (loopback ranks on one GPU; the halo carries interpolated traces) ----
GL_PART_CASES = [
    # kind, N, nx, ny, px, py
    ("euler", 3, 4, 4, 2, 2),
    ("euler", 4, 6, 4, 3, 1),
    ("advection", 3, 4, 6, 1, 2),
    ("advection", 3, 8, None, 2, 1),
    # Navier-Stokes: the lifting's central value needs the neighbours' g(w) traces (gtrace_kernel)
    ("navier_stokes", 2, 6, 6, 2, 2),
    ("navier_stokes", 3, 6, 4, 2, 1),
]


@pytest.mark.parametrize("case", GL_PART_CASES)
def test_gl_loopback_operators(case):
    """Per-rank operators of a partitioned GL problem vs the single-rank result.
    The ghost trace is interpolated by the sender (per field), the local one from
    the loaded jet state, so the two agree to rounding (<= 1e-13) rather than
    bitwise; the FD JVP within its own FD noise (vs the oracle, as test_gl_jvp_fd)."""
    import torch
    from paper_2109_04804_b200 import hbpdc
    from test_gpu_partition import _block, _run_threads
    kind, N, nx, ny, px, py = case
    dim = 1 if ny is None else 2
    d, ctx1 = _pair(kind, N, nx, ny)
    W = _state(d, kind, SEED + 81)
    sig = dgsem.rhs1(d, W) * (1 + 1e-2 * inputs.random_field(d.n, SEED + 82))
    dW = inputs.random_field(d.n, SEED + 83, unit_norm=True)
    ds = inputs.random_field(d.n, SEED + 84, unit_norm=True)
    b = W * (1 + 1e-3 * inputs.random_field(d.n, SEED + 85))
    a1, a2, dt = 1 / 6, 1 / 54, 0.02
    eps = implicit.fd_eps(dW)
    modes = ["linear"] if kind == "advection" else ["exact", "fd"]

    def ops(ctx, blk):
        Wg, sg, dWg, dsg, bg = (to_gpu(blk(x)) for x in (W, sig, dW, ds, b))
        torch.cuda.synchronize()
        out = {"R1": ctx.rhs(Wg), "R2": ctx.rhs(Wg, sg), "G": ctx.residual(a1, a2, dt, bg, Wg, sg)}
        for md in modes:
            out["jvp_" + md] = ctx.jvp(a1, a2, dt, Wg, sg, dWg, dsg, mode=md,
                                       eps_override=(eps, None) if md == "fd" else None)
        ctx.precond_build(a1, a2, dt, Wg)
        out["pc"] = ctx.precond_apply(dWg, dsg)
        torch.cuda.synchronize()
        return {k: (np.concatenate([to_np(x) for x in v]) if isinstance(v, tuple) else to_np(v))
                for k, v in out.items()}

    ref = ops(ctx1, lambda x: x)
    assert rel(ref["R1"], dgsem.rhs1(d, W)) <= 1e-11
    fd_tol = None
    if kind != "advection":
        fo = np.concatenate(implicit.jvp_fd(d, a1, a2, dt, W, sig, dW, ds, eps_override=(eps, None)))
        ex = np.concatenate(implicit.jvp_exact(d, a1, a2, dt, W, sig, dW, ds))
        fd_tol = max(1e-11, 4 * rel(fo, ex))
    group = hbpdc.LoopbackGroup(px * py)
    a = (1.0, 0.0) if dim == 1 else (1.0, -0.6)
    nskw = dict(mu=NS_MU, bounds=(0.0, 2 * np.pi, 0.0, 2 * np.pi)) if kind == "navier_stokes" else {}
    ctxs = [hbpdc.Context(dim=dim, equation=kind, N=N, nx=nx, ny=ny or 1, a=a, rank=r, nranks=px * py, px=px,
                          py=py, comm="loopback", loopback=group, stream=torch.cuda.Stream(), nodes="gl", **nskw)
            for r in range(px * py)]
    try:
        def blk_of(c):
            return lambda x: _block(x, dim, nx, ny or 1, d.m, c.ex0, c.ey0, c.nx_local, c.ny_local)
        outs = _run_threads([lambda c=c: ops(c, blk_of(c)) for c in ctxs])
        for c, o in zip(ctxs, outs):
            blk = blk_of(c)
            for key, r in ref.items():
                rb = np.concatenate([blk(r[:d.n]), blk(r[d.n:])]) if r.size == 2 * d.n else blk(r)
                tol = fd_tol if key == "jvp_fd" else 1e-13
                assert rel(o[key], rb) <= tol, (key, c.rank, rel(o[key], rb))
    finally:
        for c in ctxs:
            c.close()
        group.close()


def test_gl_loopback_hbpc_step():
    """Euler HBPC(4,0) on GL nodes, 2 x 2 loopback ranks: one step vs the oracle <= 1e-8."""
    import torch
    from paper_2109_04804_b200 import hbpdc
    from test_gpu_partition import _block, _run_threads
    N, nx, ny, px, py = 3, 4, 4, 2, 2
    d, _ = _pair("euler", N, nx, ny)
    W0 = _state(d, "euler", SEED + 86)
    dt = 0.01
    Wo = _run_oracle(d, 4, 0, W0, dt, 1, rtol=1e-10, gmres_rtol=1e-10)
    group = hbpdc.LoopbackGroup(px * py)
    ctxs = [hbpdc.Context(dim=2, equation="euler", N=N, nx=nx, ny=ny, a=(1.0, -0.6), q=4, kmax=0,
                          gmres_rtol=1e-10, newton_rtol=1e-10, rank=r, nranks=px * py, px=px, py=py,
                          comm="loopback", loopback=group, stream=torch.cuda.Stream(), nodes="gl")
            for r in range(px * py)]
    try:
        def run(c):
            Wl = to_gpu(_block(W0, 2, nx, ny, d.m, c.ex0, c.ey0, c.nx_local, c.ny_local))
            torch.cuda.synchronize()
            c.step(dt, Wl)
            torch.cuda.synchronize()
            return to_np(Wl)
        outs = _run_threads([lambda c=c: run(c) for c in ctxs])
        for c, Wl in zip(ctxs, outs):
            blk = _block(Wo, 2, nx, ny, d.m, c.ex0, c.ey0, c.nx_local, c.ny_local)
            assert rel(Wl, blk) <= 1e-8, (c.rank, rel(Wl, blk))
    finally:
        for c in ctxs:
            c.close()
        group.close()


def test_gl_nccl_self_halo():
    """GL through the NCCL transport with a forced self halo (1 rank): R1 and one step vs single rank."""
    from paper_2109_04804_b200 import hbpdc
    d, ctx1 = _pair("euler", 3, 4, 4)
    ctxn = hbpdc.Context(dim=2, equation="euler", N=3, nx=4, ny=4, a=(1.0, -0.6), comm="nccl",
                         nccl_id=hbpdc.nccl_unique_id(), force_halo=True, nodes="gl")
    try:
        W = _state(d, "euler", SEED + 87)
        assert rel(to_np(ctxn.rhs(to_gpu(W))), to_np(ctx1.rhs(to_gpu(W)))) <= 1e-13
        W1, Wn = to_gpu(W), to_gpu(W)
        ctx1.step(0.01, W1)
        ctxn.step(0.01, Wn)
        assert rel(to_np(Wn), to_np(W1)) <= 1e-10
    finally:
        ctxn.close()
