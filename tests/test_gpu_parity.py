"""GPU (CUDA, through the C-ABI) vs CPU oracle parity.

Tolerances (north_star): relative L2 <= 1e-11 per operator /
JVP application on seeded perturbed inputs; FD JVP within
max(1e-11, 4 delta_FD) with delta_FD the oracle's own FD-vs-EXACT gap at the
same eps; precond apply with identical S <= 1e-13; S build
<= 1e-11 max(1, cond/1e4); end of run <= 1e-8.
Sizes span several CTAs and a ragged last CTA (element counts not multiples
of the elements-per-CTA)."""
import numpy as np
import pytest

from oracle import dgsem, hbpc, implicit
from paper_2109_04804_b200 import configs, inputs
from gpu_common import adv_ic, euler_ic, make_pair, ns_ic, rel, to_gpu, to_np, SEED

pytestmark = pytest.mark.gpu

OPS_CASES = [
    # (kind, N, nx, ny, bounds)
    ("advection", 3, 16, None, (0.0, 1.0, 0.0, 1.0)),
    ("advection", 5, 9, 7, (0.0, 1.0, 0.0, 1.0)),
    ("euler", 7, 5, 3, (0.0, 1.0, 0.0, 1.0)),
    ("euler", 3, 11, 6, (0.0, 1.0, 0.0, 1.0)),
    ("euler", 2, 4, 4, (0.0, 1.0, 0.0, 1.0)),
    ("navier_stokes", 3, 4, 4, (0.0, 2 * np.pi, 0.0, 2 * np.pi)),
    ("navier_stokes", 5, 5, 3, (0.0, 2 * np.pi, 0.0, 2 * np.pi)),
]

NS_MU = 0.05      # viscosity for NS operator tests: viscous terms O(1) relative (C5 uses 1e-3)


def _state(d, kind, seed):
    if kind == "advection":
        return adv_ic(d, seed)
    if kind == "euler":
        return euler_ic(d, seed)
    return ns_ic(d, seed)


def _pair(kind, N, nx, ny, bounds, **kw):
    a = (1.0, 0.0) if ny is None else (1.0, -0.6)
    if kind == "navier_stokes":
        kw.setdefault("mu", NS_MU)
    return make_pair(kind, N, nx, ny, bounds=bounds, a=a, **kw)


@pytest.mark.parametrize("case", OPS_CASES)
def test_node_coords(case):
    d, ctx = _pair(*case)
    g = ctx.node_coords()
    o = d.node_coords()
    for a, b in zip(g, o):
        np.testing.assert_allclose(a, b, rtol=0, atol=1e-14)


@pytest.mark.parametrize("case", OPS_CASES)
def test_rhs_r1_r2(case):
    kind = case[0]
    d, ctx = _pair(*case)
    W = _state(d, kind, SEED + 1)
    sig = dgsem.rhs1(d, W) * (1 + 1e-2 * inputs.random_field(d.n, SEED + 2))
    R1o = dgsem.rhs1(d, W)
    R2o = dgsem.rhs2(d, W, sig)
    R1g = to_np(ctx.rhs(to_gpu(W)))
    R2g = to_np(ctx.rhs(to_gpu(W), to_gpu(sig)))
    assert rel(R1g, R1o) <= 1e-11
    assert rel(R2g, R2o) <= 1e-11


@pytest.mark.parametrize("case", OPS_CASES)
def test_residual(case):
    kind = case[0]
    d, ctx = _pair(*case)
    W = _state(d, kind, SEED + 3)
    sig = dgsem.rhs1(d, W) * (1 + 1e-2 * inputs.random_field(d.n, SEED + 4))
    b = W * (1 + 1e-3 * inputs.random_field(d.n, SEED + 5))
    a1, a2, dt = 1.0 / 6.0, 1.0 / 54.0, 0.01
    G1o, G2o = implicit.residual(d, a1, a2, dt, b, W, sig)
    G1g, G2g, nrm = ctx.residual(a1, a2, dt, to_gpu(b), to_gpu(W), to_gpu(sig), norm=True)
    o = np.concatenate([G1o, G2o])
    g = np.concatenate([to_np(G1g), to_np(G2g)])
    assert rel(g, o) <= 1e-11
    assert abs(nrm - np.linalg.norm(o)) <= 1e-11 * np.linalg.norm(o)


def test_residual_degenerate():
    """dt = 0, b = W -> G1 = 0 exactly; sigma = R1(W) -> G2 = 0 up to the
    rounding of two R1 evaluations (plain vs dual carrier; FMA contraction
    differs between them)."""
    d, ctx = _pair("euler", 3, 4, 4, (0.0, 1.0, 0.0, 1.0))
    W = euler_ic(d, SEED + 6)
    Wg = to_gpu(W)
    sig = ctx.rhs(Wg)
    G1, G2 = ctx.residual(0.5, 1 / 6, 0.0, Wg, Wg, sig)
    assert np.abs(to_np(G1)).max() == 0.0
    assert np.abs(to_np(G2)).max() <= 1e-13 * np.abs(to_np(sig)).max()


@pytest.mark.parametrize("case", [c for c in OPS_CASES if c[0] != "advection"])
def test_jvp_exact(case):
    kind = case[0]
    d, ctx = _pair(*case)
    W = _state(d, kind, SEED + 7)
    sig = dgsem.rhs1(d, W) * (1 + 1e-2 * inputs.random_field(d.n, SEED + 8))
    dW = inputs.random_field(d.n, SEED + 9, unit_norm=True)
    ds = inputs.random_field(d.n, SEED + 10, unit_norm=True)
    a1, a2, dt = 0.5, 1 / 6, 0.02
    to, bo = implicit.jvp_exact(d, a1, a2, dt, W, sig, dW, ds)
    tg, bg = ctx.jvp(a1, a2, dt, to_gpu(W), to_gpu(sig), to_gpu(dW), to_gpu(ds), mode="exact")
    assert rel(np.concatenate([to_np(tg), to_np(bg)]), np.concatenate([to, bo])) <= 1e-11


@pytest.mark.parametrize("case", [c for c in OPS_CASES if c[0] == "advection"])
def test_jvp_linear(case):
    d, ctx = _pair(*case)
    dW = inputs.random_field(d.n, SEED + 11, unit_norm=True)
    ds = inputs.random_field(d.n, SEED + 12, unit_norm=True)
    z = np.zeros(d.n)
    a1, a2, dt = 1.0, 1.0, 0.05
    to, bo = implicit.jvp_linear(d, a1, a2, dt, dW, ds)
    tg, bg = ctx.jvp(a1, a2, dt, to_gpu(z), to_gpu(z), to_gpu(dW), to_gpu(ds), mode="linear")
    assert rel(np.concatenate([to_np(tg), to_np(bg)]), np.concatenate([to, bo])) <= 1e-11


@pytest.mark.parametrize("case", [c for c in OPS_CASES if c[0] != "advection"])
def test_jvp_fd(case):
    """FD JVP with eps pinned via eps_override."""
    kind = case[0]
    d, ctx = _pair(*case)
    W = _state(d, kind, SEED + 13)
    sig = dgsem.rhs1(d, W) * (1 + 1e-2 * inputs.random_field(d.n, SEED + 14))
    dW = inputs.random_field(d.n, SEED + 15, unit_norm=True)
    ds = inputs.random_field(d.n, SEED + 16, unit_norm=True)
    a1, a2, dt = 1.0, 1.0, 0.01
    eps = implicit.fd_eps(dW)
    fo = np.concatenate(implicit.jvp_fd(d, a1, a2, dt, W, sig, dW, ds, eps_override=(eps, None)))
    ex = np.concatenate(implicit.jvp_exact(d, a1, a2, dt, W, sig, dW, ds))
    delta = rel(fo, ex)
    tg, bg = ctx.jvp(a1, a2, dt, to_gpu(W), to_gpu(sig), to_gpu(dW), to_gpu(ds), mode="fd",
                     eps_override=(eps, None))
    g = np.concatenate([to_np(tg), to_np(bg)])
    assert rel(g, fo) <= max(1e-11, 4 * delta), (rel(g, fo), delta)
    # the library's own eps (device-side norm) gives the same answer within the FD floor
    tg2, bg2 = ctx.jvp(a1, a2, dt, to_gpu(W), to_gpu(sig), to_gpu(dW), to_gpu(ds), mode="fd")
    assert rel(np.concatenate([to_np(tg2), to_np(bg2)]), fo) <= max(1e-11, 4 * delta)
    # zero direction: the quotient is 0
    z = np.zeros(d.n)
    tz, bz = ctx.jvp(a1, a2, dt, to_gpu(W), to_gpu(sig), to_gpu(z), to_gpu(z), mode="fd")
    assert np.abs(to_np(tz)).max() == 0.0 and np.abs(to_np(bz)).max() == 0.0


PC_CASES = [
    ("advection", 3, 8, None, (0.0, 1.0, 0.0, 1.0)),
    ("advection", 2, 6, 4, (0.0, 1.0, 0.0, 1.0)),
    ("euler", 2, 4, 4, (0.0, 1.0, 0.0, 1.0)),
    ("euler", 3, 4, 2, (0.0, 1.0, 0.0, 1.0)),
    ("navier_stokes", 2, 4, 3, (0.0, 2 * np.pi, 0.0, 2 * np.pi)),
    ("navier_stokes", 3, 3, 3, (0.0, 2 * np.pi, 0.0, 2 * np.pi)),
]


@pytest.mark.parametrize("case", PC_CASES)
def test_precond_build_and_apply(case):
    kind = case[0]
    d, ctx = _pair(*case)
    W = _state(d, kind, SEED + 17)
    a1, a2, dt = 1.0 / 6.0, 1.0 / 54.0, 0.05
    pc = implicit.BJExt(d, W, a1, a2, dt)
    ctx.precond_build(a1, a2, dt, to_gpu(W))
    shared = kind == "advection"
    Sg, flag = ctx.precond_export(shared_hint=shared)
    assert flag == shared
    Sg = to_np(Sg).reshape(-1, d.m, d.m)
    So = pc.S[:1] if shared else pc.S
    cond = max(np.linalg.cond(M) for M in pc.M)
    err = np.linalg.norm(Sg - So) / np.linalg.norm(So)
    assert err <= 1e-11 * max(1.0, cond / 1e4), (err, cond)
    x = inputs.random_field(d.n, SEED + 18)
    y = inputs.random_field(d.n, SEED + 19)
    to, bo = pc.apply(x, y)
    tg, bg = ctx.precond_apply(to_gpu(x), to_gpu(y))
    assert rel(np.concatenate([to_np(tg), to_np(bg)]), np.concatenate([to, bo])) <= 1e-11 * max(1, cond / 1e4)
    if kind == "navier_stokes":
        return        # NS applies its stored K_i as well; precond_set installs S only
    # identical S (the oracle's, installed into the library): apply <= 1e-13
    ctx.precond_set(a1, a2, dt, to_gpu(W), to_gpu(So.reshape(-1)), shared)
    tg, bg = ctx.precond_apply(to_gpu(x), to_gpu(y))
    to2, bo2 = pc.apply_sk(x, y)
    assert rel(np.concatenate([to_np(tg), to_np(bg)]), np.concatenate([to2, bo2])) <= 1e-13


def _run_oracle(d, q, kmax, W0, dt, steps, **opt):
    H = hbpc.HBPC(d, q, kmax, implicit.NewtonOpts(**opt))
    W = W0.copy()
    st = dict(stage_solves=0, newton_its=0, gmres_its=0, precond_builds=0)
    for _ in range(steps):
        W = H.step(W, dt, st)
    return W, st


def test_c1_end_of_run():
    """C1 exactly as BASELINE.json states it: 1D advection, N=3, 16 elements,
    HBPC(4,0), CFL 1, 10 steps, GMRES rtol 1e-12."""
    cfg = configs.CONFIGS["C1"]
    d, ctx = make_pair("advection", cfg.N, cfg.nx, None, a=cfg.a, q=cfg.q, kmax=cfg.kmax,
                       gmres_rtol=cfg.gmres_rtol, newton_rtol=cfg.newton_rtol)
    W0 = inputs.initial_state("C1", d.node_coords())
    dt = configs.cfl_dt(cfg, W0)
    Wo, sto = _run_oracle(d, cfg.q, cfg.kmax, W0, dt, cfg.steps, rtol=cfg.newton_rtol,
                          gmres_rtol=cfg.gmres_rtol)
    Wg = to_gpu(W0)
    its = 0
    for _ in range(cfg.steps):
        its += ctx.step(dt, Wg)["gmres_its"]
    assert rel(to_np(Wg), Wo) <= 1e-8


@pytest.mark.parametrize("precond,cfl", [("bjext", 2.0), ("none", 0.25)])
def test_c2_shape_end_of_run(precond, cfl):
    """C2 physics at a reduced mesh (8x8, N=5, HBPC(6,2), 3 steps); CFL 2 with
    BJ_ext as configured, CFL 0.25 without a preconditioner (no-PC is
    only competitive for small steps; at CFL 2 unpreconditioned GMRES(700)
    stalls)."""
    cfg = configs.scaled(configs.CONFIGS["C2"], nx=8, ny=8, steps=3, cfl=cfl)
    d, ctx = make_pair("advection", cfg.N, cfg.nx, cfg.ny, a=cfg.a, q=cfg.q, kmax=cfg.kmax,
                       gmres_rtol=cfg.gmres_rtol, newton_rtol=cfg.newton_rtol, precond=precond)
    W0 = inputs.initial_state("C2", d.node_coords())
    dt = configs.cfl_dt(cfg, W0)
    Wo, _ = _run_oracle(d, cfg.q, cfg.kmax, W0, dt, cfg.steps, rtol=cfg.newton_rtol,
                        gmres_rtol=cfg.gmres_rtol, precond=precond)
    Wg = to_gpu(W0)
    for _ in range(cfg.steps):
        ctx.step(dt, Wg)
    assert rel(to_np(Wg), Wo) <= 1e-8


@pytest.mark.parametrize("q,kmax", [(4, 0), (8, 4)])
def test_euler_end_of_run(q, kmax):
    """C3 physics (isentropic vortex + seeded noise) at a reduced mesh:
    4x4 elements, N=3, BJ_ext, FD JVP, 2 steps."""
    cfg = configs.scaled(configs.CONFIGS["C3"], N=3, nx=4, ny=4, steps=2, q=q, kmax=kmax)
    d, ctx = make_pair("euler", cfg.N, cfg.nx, cfg.ny, bounds=cfg.bounds, q=q, kmax=kmax,
                       gmres_rtol=cfg.gmres_rtol, newton_rtol=cfg.newton_rtol)
    W0 = inputs.initial_state("C3", d.node_coords(), noise=cfg.noise)
    dt = configs.cfl_dt(cfg, inputs.initial_state("C3", d.node_coords()))
    Wo, sto = _run_oracle(d, q, kmax, W0, dt, cfg.steps, rtol=cfg.newton_rtol, gmres_rtol=cfg.gmres_rtol)
    Wg = to_gpu(W0)
    for _ in range(cfg.steps):
        ctx.step(dt, Wg)
    assert rel(to_np(Wg), Wo) <= 1e-8


@pytest.mark.parametrize("precond", ["bjext", "bjext_h"])
def test_c5_shape_end_of_run(precond):
    """C5 physics (2D Navier-Stokes, BR1, TGV-type vortex at Mach 0.1, mu = 1e-3,
    Pr 0.72) at a reduced mesh: 4x4 elements, N=3, HBPC(6,2), BJ_ext or BJ^H_ext
    (NEXT-2: H_i by the two-hop colouring), FD JVP, 2 steps of the CFL-1 step;
    GPU vs oracle <= 1e-8."""
    cfg = configs.scaled(configs.CONFIGS["C5"], N=3, nx=4, ny=4, steps=2)
    d, ctx = make_pair("navier_stokes", cfg.N, cfg.nx, cfg.ny, bounds=cfg.bounds, mu=cfg.mu, q=cfg.q,
                       kmax=cfg.kmax, gmres_rtol=cfg.gmres_rtol, newton_rtol=cfg.newton_rtol, precond=precond)
    W0 = inputs.initial_state("C5", d.node_coords())
    dt = configs.cfl_dt(cfg, W0)
    Wo, sto = _run_oracle(d, cfg.q, cfg.kmax, W0, dt, cfg.steps, rtol=cfg.newton_rtol, gmres_rtol=cfg.gmres_rtol,
                          precond=precond)
    Wg = to_gpu(W0)
    for _ in range(cfg.steps):
        ctx.step(dt, Wg)
    assert rel(to_np(Wg), Wo) <= 1e-8


@pytest.mark.parametrize("q,kmax", [(8, 4), (6, 2)])
def test_batched_correctors_bitwise(q, kmax):
    """NEXT-1: the s-1 corrector stages of a sweep solved in lock step (one
    BJ_ext S pass per Arnoldi step for all of them) give bit-identical steps
    and identical iteration counts to the sequential order."""
    import torch
    cfg = configs.scaled(configs.CONFIGS["C3"], N=3, nx=4, ny=4, q=q, kmax=kmax)
    out = []
    for batch in (True, False):
        d, ctx = make_pair("euler", cfg.N, cfg.nx, cfg.ny, bounds=cfg.bounds, q=q, kmax=kmax,
                           gmres_rtol=cfg.gmres_rtol, newton_rtol=cfg.newton_rtol, batch_stages=batch)
        W0 = inputs.initial_state("C3", d.node_coords(), noise=cfg.noise)
        dt = configs.cfl_dt(cfg, inputs.initial_state("C3", d.node_coords()))
        Wg = to_gpu(W0)
        st = [ctx.step(dt, Wg) for _ in range(2)]
        torch.cuda.synchronize()
        out.append((to_np(Wg), [(s["gmres_its"], s["newton_its"]) for s in st]))
        ctx.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1]


@pytest.mark.parametrize("q,kmax", [(6, 2), (8, 4)])
def test_batched_correctors_bitwise_ns(q, kmax):
    """Navier-Stokes (stored K_i): the lock-step corrector stages share ONE pass over S
    and ONE over K for all systems (2B right-hand sides each); bit-identical to the
    sequential order, identical iteration counts."""
    import torch
    cfg = configs.scaled(configs.CONFIGS["C5"], N=3, nx=6, ny=6, q=q, kmax=kmax)
    out = []
    for batch in (True, False):
        d, ctx = make_pair("navier_stokes", cfg.N, cfg.nx, cfg.ny, bounds=cfg.bounds, q=q, kmax=kmax,
                           mu=cfg.mu, gmres_rtol=cfg.gmres_rtol, newton_rtol=cfg.newton_rtol, batch_stages=batch)
        W0 = inputs.initial_state("C5", d.node_coords())
        dt = configs.cfl_dt(cfg, W0)
        Wg = to_gpu(W0)
        st = [ctx.step(dt, Wg) for _ in range(2)]
        torch.cuda.synchronize()
        out.append((to_np(Wg), [(s["gmres_its"], s["newton_its"]) for s in st]))
        ctx.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1]


@pytest.mark.parametrize("nodes,lifting", [("gll", "br1"), ("gl", "br2")])
def test_ns_k_reuse_bitwise(nodes, lifting, monkeypatch):
    """Navier-Stokes: the second BJ_ext build of a step (the correctors' alpha pair, same W^n)
    reuses the stored K_i of the first and only redoes M_i and its inverse; bit-identical
    steps and iteration counts to rebuilding K_i (HBPDC_NS_KREUSE=0), and the reuse is
    counted in the step stats (one per step for HBPC(6,2): two builds, one colour loop)."""
    import torch
    cfg = configs.scaled(configs.CONFIGS["C5"], N=3, nx=6, ny=6, q=6, kmax=2)
    out = []
    for reuse in ("1", "0"):
        monkeypatch.setenv("HBPDC_NS_KREUSE", reuse)
        d, ctx = make_pair("navier_stokes", cfg.N, cfg.nx, cfg.ny, bounds=cfg.bounds, q=cfg.q, kmax=cfg.kmax,
                           mu=cfg.mu, gmres_rtol=cfg.gmres_rtol, newton_rtol=cfg.newton_rtol, nodes=nodes,
                           lifting=lifting)
        W0 = inputs.initial_state("C5", d.node_coords())
        dt = configs.cfl_dt(cfg, W0)
        Wg = to_gpu(W0)
        st = [ctx.step(dt, Wg) for _ in range(2)]
        torch.cuda.synchronize()
        out.append((to_np(Wg), [(s["gmres_its"], s["newton_its"], s["precond_builds"]) for s in st],
                    [s["precond_k_reused"] for s in st]))
        ctx.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1]
    assert out[0][2] == [1, 1] and out[1][2] == [0, 0], (out[0][2], out[1][2])


@pytest.mark.parametrize("s", [2, 4, 8])
@pytest.mark.parametrize("q,kmax", [(4, 0), (8, 4)])
def test_sstep_gmres_end_of_run(s, q, kmax):
    """s-step (communication-avoiding) Arnoldi: Newton-basis powers + block
    CGS2/CholQR2.  Same GMRES iterates in exact arithmetic: end of run vs the
    oracle <= 1e-8, iteration counts close to the DCGS2 schedule's."""
    import torch
    cfg = configs.scaled(configs.CONFIGS["C3"], N=3, nx=4, ny=4, steps=2, q=q, kmax=kmax)
    d, ctx = make_pair("euler", cfg.N, cfg.nx, cfg.ny, bounds=cfg.bounds, q=q, kmax=kmax,
                       gmres_rtol=cfg.gmres_rtol, newton_rtol=cfg.newton_rtol, gmres_sstep=s)
    d1, ctx1 = make_pair("euler", cfg.N, cfg.nx, cfg.ny, bounds=cfg.bounds, q=q, kmax=kmax,
                         gmres_rtol=cfg.gmres_rtol, newton_rtol=cfg.newton_rtol)
    W0 = inputs.initial_state("C3", d.node_coords(), noise=cfg.noise)
    dt = configs.cfl_dt(cfg, inputs.initial_state("C3", d.node_coords()))
    Wo, _ = _run_oracle(d, q, kmax, W0, dt, cfg.steps, rtol=cfg.newton_rtol, gmres_rtol=cfg.gmres_rtol)
    its = []
    for cx in (ctx, ctx1):
        Wg = to_gpu(W0)
        n = 0
        for _ in range(cfg.steps):
            n += cx.step(dt, Wg)["gmres_its"]
        torch.cuda.synchronize()
        its.append(n)
        assert rel(to_np(Wg), Wo) <= 1e-8
    assert its[0] <= 1.25 * its[1] + 2 * s, its


@pytest.mark.parametrize("tau", ["0", "1e-6"])
@pytest.mark.parametrize("kind", ["euler", "advection"])
def test_sstep_selective_reorth_end_of_run(kind, tau, monkeypatch):
    """s = 8 block CGS with the second update skipped when |C2 Rw^-1| <= tau
    (reading R37, HBPDC_SEL_REORTH; the default 1e-12 runs in every other s = 8 test):
    end of run vs the oracle <= 1e-8 with tau = 0 (every block reorthogonalised) and
    tau = 1e-6 (a loose threshold: the skip branch fires on nearly every block)."""
    import torch
    monkeypatch.setenv("HBPDC_SEL_REORTH", tau)
    if kind == "euler":
        cfg = configs.scaled(configs.CONFIGS["C3"], N=3, nx=4, ny=4, steps=2, q=6, kmax=2)
        d, ctx = make_pair("euler", cfg.N, cfg.nx, cfg.ny, bounds=cfg.bounds, q=cfg.q, kmax=cfg.kmax,
                           gmres_rtol=cfg.gmres_rtol, newton_rtol=cfg.newton_rtol, gmres_sstep=8)
        W0 = inputs.initial_state("C3", d.node_coords(), noise=cfg.noise)
        dt = configs.cfl_dt(cfg, inputs.initial_state("C3", d.node_coords()))
        Wo, _ = _run_oracle(d, cfg.q, cfg.kmax, W0, dt, cfg.steps, rtol=cfg.newton_rtol, gmres_rtol=cfg.gmres_rtol)
    else:
        cfg = configs.scaled(configs.CONFIGS["C2"], nx=8, ny=8, steps=3, cfl=2.0)
        d, ctx = make_pair("advection", cfg.N, cfg.nx, cfg.ny, a=cfg.a, q=cfg.q, kmax=cfg.kmax,
                           gmres_rtol=cfg.gmres_rtol, newton_rtol=cfg.newton_rtol, gmres_sstep=8)
        W0 = inputs.initial_state("C2", d.node_coords())
        dt = configs.cfl_dt(cfg, W0)
        Wo, _ = _run_oracle(d, cfg.q, cfg.kmax, W0, dt, cfg.steps, rtol=cfg.newton_rtol, gmres_rtol=cfg.gmres_rtol)
    Wg = to_gpu(W0)
    for _ in range(cfg.steps):
        ctx.step(dt, Wg)
    torch.cuda.synchronize()
    assert rel(to_np(Wg), Wo) <= 1e-8


@pytest.mark.parametrize("s", [4, 8])
@pytest.mark.parametrize("precond,cfl", [("bjext", 2.0), ("none", 0.25)])
def test_sstep_advection_end_of_run(precond, cfl, s):
    """s = 8 runs the TMA-streamed block kernels on a ragged length (2n = 4608)."""
    cfg = configs.scaled(configs.CONFIGS["C2"], nx=8, ny=8, steps=3, cfl=cfl)
    d, ctx = make_pair("advection", cfg.N, cfg.nx, cfg.ny, a=cfg.a, q=cfg.q, kmax=cfg.kmax,
                       gmres_rtol=cfg.gmres_rtol, newton_rtol=cfg.newton_rtol, precond=precond, gmres_sstep=s)
    W0 = inputs.initial_state("C2", d.node_coords())
    dt = configs.cfl_dt(cfg, W0)
    Wo, _ = _run_oracle(d, cfg.q, cfg.kmax, W0, dt, cfg.steps, rtol=cfg.newton_rtol,
                        gmres_rtol=cfg.gmres_rtol, precond=precond)
    Wg = to_gpu(W0)
    for _ in range(cfg.steps):
        ctx.step(dt, Wg)
    assert rel(to_np(Wg), Wo) <= 1e-8


# ---- NEXT-2: BJ^H_ext (the Hessian block included) -----------------------

@pytest.mark.parametrize("case", PC_CASES)
def test_precond_bjext_h_build_and_apply(case):
    """S^H = (I - a1 dt K + c2 (H + K^2))^-1 per element and the apply
    u = S^H (x - c2 K y), (u, y + K u) vs the oracle's literal D^H,E^H,F^H,G^H
    blocks (built at (W, R1(W)), reading R31)."""
    kind = case[0]
    d, ctx = _pair(*case, precond="bjext_h")
    W = _state(d, kind, SEED + 27)
    a1, a2, dt = 1.0 / 6.0, 1.0 / 54.0, 0.05
    pc = implicit.BJExtH(d, W, dgsem.rhs1(d, W), a1, a2, dt)
    ctx.precond_build(a1, a2, dt, to_gpu(W))
    shared = kind == "advection"
    Sg, flag = ctx.precond_export(shared_hint=shared)
    Sg = to_np(Sg).reshape(-1, d.m, d.m)
    So = pc.S[:1] if shared else pc.S
    cond = max(np.linalg.cond(M) for M in pc.M)
    assert np.linalg.norm(Sg - So) / np.linalg.norm(So) <= 1e-11 * max(1.0, cond / 1e4)
    x = inputs.random_field(d.n, SEED + 28)
    y = inputs.random_field(d.n, SEED + 29)
    to, bo = pc.apply(x, y)
    tg, bg = ctx.precond_apply(to_gpu(x), to_gpu(y))
    assert rel(np.concatenate([to_np(tg), to_np(bg)]), np.concatenate([to, bo])) <= 1e-11 * max(1, cond / 1e4)
    if kind == "navier_stokes":
        return      # precond_set cannot install NS blocks (the stored K_i comes from the build)
    # identical S^H installed: the K pieces alone differ by rounding
    ctx.precond_set(a1, a2, dt, to_gpu(W), to_gpu(So.reshape(-1)), shared)
    tg, bg = ctx.precond_apply(to_gpu(x), to_gpu(y))
    to2, bo2 = pc.apply_sk(x, y)
    assert rel(np.concatenate([to_np(tg), to_np(bg)]), np.concatenate([to2, bo2])) <= 1e-13


@pytest.mark.parametrize("batch", [False, True])
def test_euler_end_of_run_bjext_h(batch):
    """C3 physics at 4x4 elements, N=3, HBPC(8,4) with BJ^H_ext: end of run vs the
    oracle <= 1e-8; lock-step correctors (3 systems, 1-RHS GEMV each) as well."""
    q, kmax = 8, 4
    cfg = configs.scaled(configs.CONFIGS["C3"], N=3, nx=4, ny=4, steps=2, q=q, kmax=kmax)
    d, ctx = make_pair("euler", cfg.N, cfg.nx, cfg.ny, bounds=cfg.bounds, q=q, kmax=kmax,
                       gmres_rtol=cfg.gmres_rtol, newton_rtol=cfg.newton_rtol, precond="bjext_h",
                       batch_stages=batch)
    W0 = inputs.initial_state("C3", d.node_coords(), noise=cfg.noise)
    dt = configs.cfl_dt(cfg, inputs.initial_state("C3", d.node_coords()))
    Wo, sto = _run_oracle(d, q, kmax, W0, dt, cfg.steps, rtol=cfg.newton_rtol, gmres_rtol=cfg.gmres_rtol,
                          precond="bjext_h")
    Wg = to_gpu(W0)
    its = 0
    for _ in range(cfg.steps):
        its += ctx.step(dt, Wg)["gmres_its"]
    assert rel(to_np(Wg), Wo) <= 1e-8
    assert its <= 1.25 * sto["gmres_its"] + 10, (its, sto["gmres_its"])


# ---- NEXT-3 (part): the paper's numerical flux eq:Riemann (global LF, Lambda = I at eps = 1) ----

GLF_CASES = [("advection", 3, 16, None, (0.0, 1.0, 0.0, 1.0)),
             ("advection", 5, 9, 7, (0.0, 1.0, 0.0, 1.0)),
             ("euler", 3, 5, 4, (0.0, 1.0, 0.0, 1.0)),
             ("euler", 7, 3, 3, (0.0, 1.0, 0.0, 1.0)),
             ("navier_stokes", 3, 4, 4, (0.0, 2 * np.pi, 0.0, 2 * np.pi))]


@pytest.mark.parametrize("case", GLF_CASES)
def test_glf_operators(case):
    """R1, R2, residual, EXACT JVP and (advection, Euler) BJ_ext with flux = GLF_PAPER
    (eq:Riemann literally: the full Lambda on the jump) vs the oracle's
    Equation(numflux='glf'), <= 1e-11."""
    kind = case[0]
    d, ctx = _pair(*case, flux="glf")
    W = _state(d, kind, SEED + 41)
    sig = dgsem.rhs1(d, W) * (1 + 1e-2 * inputs.random_field(d.n, SEED + 42))
    assert rel(to_np(ctx.rhs(to_gpu(W))), dgsem.rhs1(d, W)) <= 1e-11
    assert rel(to_np(ctx.rhs(to_gpu(W), to_gpu(sig))), dgsem.rhs2(d, W, sig)) <= 1e-11
    b = W * (1 + 1e-3 * inputs.random_field(d.n, SEED + 43))
    a1, a2, dt = 0.5, 1 / 6, 0.02
    G1o, G2o = implicit.residual(d, a1, a2, dt, b, W, sig)
    G1g, G2g = ctx.residual(a1, a2, dt, to_gpu(b), to_gpu(W), to_gpu(sig))
    assert rel(np.concatenate([to_np(G1g), to_np(G2g)]), np.concatenate([G1o, G2o])) <= 1e-11
    dW = inputs.random_field(d.n, SEED + 44, unit_norm=True)
    ds = inputs.random_field(d.n, SEED + 45, unit_norm=True)
    to, bo = implicit.jvp_exact(d, a1, a2, dt, W, sig, dW, ds)
    tg, bg = ctx.jvp(a1, a2, dt, to_gpu(W), to_gpu(sig), to_gpu(dW), to_gpu(ds), mode="exact")
    assert rel(np.concatenate([to_np(tg), to_np(bg)]), np.concatenate([to, bo])) <= 1e-11
    if kind != "navier_stokes":
        pc = implicit.BJExt(d, W, a1, a2, dt)
        ctx.precond_build(a1, a2, dt, to_gpu(W))
        cond = max(np.linalg.cond(M) for M in pc.M)
        to, bo = pc.apply(dW, ds)
        tg, bg = ctx.precond_apply(to_gpu(dW), to_gpu(ds))
        assert rel(np.concatenate([to_np(tg), to_np(bg)]), np.concatenate([to, bo])) <= 1e-11 * max(1, cond / 1e4)


def test_glf_euler_end_of_run():
    """C3 physics at 4x4 elements, N=3, HBPC(6,2) with the paper's flux: end of run
    vs the oracle <= 1e-8."""
    q, kmax = 6, 2
    cfg = configs.scaled(configs.CONFIGS["C3"], N=3, nx=4, ny=4, steps=2, q=q, kmax=kmax)
    d, ctx = make_pair("euler", cfg.N, cfg.nx, cfg.ny, bounds=cfg.bounds, q=q, kmax=kmax,
                       gmres_rtol=cfg.gmres_rtol, newton_rtol=cfg.newton_rtol, flux="glf")
    W0 = inputs.initial_state("C3", d.node_coords(), noise=cfg.noise)
    dt = configs.cfl_dt(cfg, inputs.initial_state("C3", d.node_coords()))
    Wo, _ = _run_oracle(d, q, kmax, W0, dt, cfg.steps, rtol=cfg.newton_rtol, gmres_rtol=cfg.gmres_rtol)
    Wg = to_gpu(W0)
    for _ in range(cfg.steps):
        ctx.step(dt, Wg)
    assert rel(to_np(Wg), Wo) <= 1e-8


@pytest.mark.parametrize("flux", ["llf", "glf"])
@pytest.mark.parametrize("mach", [0.1, 0.01])
def test_reference_mach_operators(flux, mach):
    """eq:Euler with a reference Mach number eps < 1 (the paper's
    fig:Euler_eps setups): R1, R2, residual and EXACT JVP vs the oracle <= 1e-11."""
    d, ctx = _pair("euler", 3, 5, 4, (0.0, 1.0, 0.0, 1.0), flux=flux, mach=mach)
    W = euler_ic(d, SEED + 51)
    sig = dgsem.rhs1(d, W) * (1 + 1e-2 * inputs.random_field(d.n, SEED + 52))
    assert rel(to_np(ctx.rhs(to_gpu(W))), dgsem.rhs1(d, W)) <= 1e-11
    assert rel(to_np(ctx.rhs(to_gpu(W), to_gpu(sig))), dgsem.rhs2(d, W, sig)) <= 1e-11
    b = W * (1 + 1e-3 * inputs.random_field(d.n, SEED + 53))
    a1, a2, dt = 0.5, 1 / 6, 0.002
    G1o, G2o = implicit.residual(d, a1, a2, dt, b, W, sig)
    G1g, G2g = ctx.residual(a1, a2, dt, to_gpu(b), to_gpu(W), to_gpu(sig))
    assert rel(np.concatenate([to_np(G1g), to_np(G2g)]), np.concatenate([G1o, G2o])) <= 1e-11
    dW = inputs.random_field(d.n, SEED + 54, unit_norm=True)
    ds = inputs.random_field(d.n, SEED + 55, unit_norm=True)
    to, bo = implicit.jvp_exact(d, a1, a2, dt, W, sig, dW, ds)
    tg, bg = ctx.jvp(a1, a2, dt, to_gpu(W), to_gpu(sig), to_gpu(dW), to_gpu(ds), mode="exact")
    assert rel(np.concatenate([to_np(tg), to_np(bg)]), np.concatenate([to, bo])) <= 1e-11


def test_reference_mach_end_of_run():
    """eps = 0.1 with the paper's flux and BJ_ext: 4x4 elements, N = 3, HBPC(4,0),
    2 steps of an acoustic-CFL-1 step, FD JVP (eps_FD with the Mach number):
    end of run vs the oracle <= 1e-8."""
    mach = 0.1
    d, ctx = make_pair("euler", 3, 4, 4, q=4, kmax=0, gmres_rtol=1e-10, newton_rtol=1e-10, flux="glf", mach=mach)
    W0 = euler_ic(d, SEED + 56, rel_noise=1e-3)
    h = 1.0 / 4
    dt = 1.0 * h / 7 ** 2 * mach        # ~acoustic CFL for c/eps ~ 10 c
    Wo, _ = _run_oracle(d, 4, 0, W0, dt, 2, rtol=1e-10, gmres_rtol=1e-10)
    Wg = to_gpu(W0)
    for _ in range(2):
        ctx.step(dt, Wg)
    assert rel(to_np(Wg), Wo) <= 1e-8


# ---- NEXT-2: the Schur-complement formulation --------------------------

@pytest.mark.parametrize("precond,sstep", [("bjext_h", 1), ("bjext_h", 8), ("none", 1)])
def test_schur_end_of_run(precond, sstep):
    """Newton on the Schur complement J_S dw = -G1 + c2 K G2, dsigma = -G2 + K dw
    (J_S applied as the top block of J (v, K v)), element-block Jacobi from the
    BJ^H_ext D block (reading R32) or unpreconditioned: C3 physics at 4x4
    elements, N = 3, HBPC(6,2), 2 steps, end of run vs the oracle <= 1e-8."""
    q, kmax = 6, 2
    cfg = configs.scaled(configs.CONFIGS["C3"], N=3, nx=4, ny=4, steps=2, q=q, kmax=kmax)
    cfl_scale = 1.0 if precond != "none" else 0.25
    d, ctx = make_pair("euler", cfg.N, cfg.nx, cfg.ny, bounds=cfg.bounds, q=q, kmax=kmax,
                       gmres_rtol=cfg.gmres_rtol, newton_rtol=cfg.newton_rtol, precond=precond,
                       schur=True, gmres_sstep=sstep)
    W0 = inputs.initial_state("C3", d.node_coords(), noise=cfg.noise)
    dt = cfl_scale * configs.cfl_dt(cfg, inputs.initial_state("C3", d.node_coords()))
    Wo, sto = _run_oracle(d, q, kmax, W0, dt, cfg.steps, rtol=cfg.newton_rtol, gmres_rtol=cfg.gmres_rtol,
                          precond=precond, schur=True)
    Wg = to_gpu(W0)
    its = 0
    for _ in range(cfg.steps):
        its += ctx.step(dt, Wg)["gmres_its"]
    assert rel(to_np(Wg), Wo) <= 1e-8
    assert its <= 1.25 * sto["gmres_its"] + 2 * sstep + 8, (its, sto["gmres_its"])


@pytest.mark.gpu
@pytest.mark.parametrize("case", [c for c in PC_CASES if c[0] == "navier_stokes"])
def test_ns_onehop_build_matches_colour_lifting(case, monkeypatch):
    """The one-hop NS colour build (ModeKNS: lifting on the colour's elements only, the neighbours'
    face gradients from the build state plus the seed's BR1 central-value term) against the
    colour passes that lift the colour's elements and their neighbours (HBPDC_NS_ONEHOP=0):
    the same K_i, so the same S_i up to rounding."""
    kind = case[0]
    d, ctx = _pair(*case)
    W = to_gpu(_state(d, kind, SEED + 23))
    a1, a2, dt = 1.0 / 6.0, 1.0 / 54.0, 0.05
    monkeypatch.setenv("HBPDC_NS_ONEHOP", "0")
    ctx.precond_build(a1, a2, dt, W)
    S2 = to_np(ctx.precond_export()[0]).copy()
    monkeypatch.setenv("HBPDC_NS_ONEHOP", "1")
    ctx.precond_build(a1, a2, dt, W)
    S1 = to_np(ctx.precond_export()[0])
    assert rel(S1, S2) <= 1e-12, rel(S1, S2)
