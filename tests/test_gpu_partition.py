"""Element partition on the GPU, through the C-ABI.

One B200 is available, so the multi-rank path runs as LOOPBACK ranks: host
threads of this process, one context and stream each, exchanging halos by
device copies and summing norms / Arnoldi dots in rank order (comm.h).  The
pack / ghost-unpack kernels, the ghost addressing of the operator kernels and
every all-reduce site are the ones the NCCL transport uses; the NCCL
transport itself is exercised with a forced self-halo on one rank.

* Operators are element-local given the ghost traces, so every rank's output
  must equal its block of the single-rank result BIT FOR BIT.
* A whole HBPC step differs only in reduction order: <= 1e-10 relative.
* Each is also checked against the CPU oracle (the single-rank path is).
"""
import threading

import numpy as np
import pytest

from oracle import dgsem, hbpc, implicit
from paper_2109_04804_b200 import configs, hbpdc, inputs
from gpu_common import adv_ic, euler_ic, make_pair, ns_ic, rel, to_gpu, to_np, SEED

TWO_PI = 2 * np.pi
NS_MU = 0.05

pytestmark = pytest.mark.gpu


def _block(x, cfg_dim, nx, ny, m, ex0, ey0, nxl, nyl):
    if cfg_dim == 1:
        return np.ascontiguousarray(np.asarray(x).reshape(nx, m)[ex0:ex0 + nxl]).reshape(-1)
    return np.ascontiguousarray(np.asarray(x).reshape(ny, nx, m)[ey0:ey0 + nyl, ex0:ex0 + nxl]).reshape(-1)


def _run_threads(fns):
    """Run one callable per rank concurrently (ctypes releases the GIL); re-raise."""
    res = [None] * len(fns)
    err = [None] * len(fns)

    def go(i):
        try:
            res[i] = fns[i]()
        except BaseException as e:  # noqa: BLE001
            err[i] = e

    th = [threading.Thread(target=go, args=(i,)) for i in range(len(fns))]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for e in err:
        if e is not None:
            raise e
    return res


def _ns_kw(kind):
    return dict(bounds=(0.0, TWO_PI, 0.0, TWO_PI), mu=NS_MU) if kind == "navier_stokes" else {}


def _rank_contexts(kind, N, nx, ny, px, py, group, **kw):
    import torch
    dim = 1 if ny is None else 2
    a = (1.0, 0.0) if dim == 1 else (1.0, -0.6)
    kw.update(_ns_kw(kind))
    out = []
    for r in range(px * py):
        s = torch.cuda.Stream()
        out.append(hbpdc.Context(dim=dim, equation=kind, N=N, nx=nx, ny=ny or 1, a=a, rank=r, nranks=px * py,
                                 px=px, py=py, comm="loopback", loopback=group, stream=s, **kw))
    return out


CASES = [
    # kind, N, nx, ny, px, py
    ("euler", 3, 4, 4, 2, 1),
    ("euler", 3, 4, 6, 1, 2),
    ("euler", 2, 4, 4, 2, 2),
    ("euler", 4, 6, 4, 3, 2),
    ("advection", 3, 4, 4, 2, 2),
    ("advection", 3, 8, None, 2, 1),
    # local blocks >= 3 x 3: the halo / compute overlap path (interior elements while the
    # halo is in flight, then the boundary ring) -- still bitwise equal to one rank
    ("euler", 2, 8, 6, 2, 2),
    ("advection", 3, 9, 8, 3, 2),
    ("euler", 7, 6, 3, 2, 1),
    # Navier-Stokes (BR1): second halo of the lifted gradients; local grids
    # keep a colouring period >= 3 for the two-hop BJ_ext blocks
    ("navier_stokes", 2, 6, 6, 2, 2),
    ("navier_stokes", 3, 8, 4, 2, 1),
]


@pytest.mark.parametrize("case", CASES)
def test_loopback_operators_bitwise(case):
    import torch
    kind, N, nx, ny, px, py = case
    dim = 1 if ny is None else 2
    d, ctx1 = make_pair(kind, N, nx, ny, a=(1.0, 0.0) if dim == 1 else (1.0, -0.6), **_ns_kw(kind))
    W = {"advection": adv_ic, "euler": euler_ic, "navier_stokes": ns_ic}[kind](d, SEED + 31)
    sig = dgsem.rhs1(d, W) * (1 + 1e-2 * inputs.random_field(d.n, SEED + 32))
    dW = inputs.random_field(d.n, SEED + 33, unit_norm=True)
    ds = inputs.random_field(d.n, SEED + 34, unit_norm=True)
    b = W * (1 + 1e-3 * inputs.random_field(d.n, SEED + 35))
    a1, a2, dt = 1 / 6, 1 / 54, 0.02
    eps = implicit.fd_eps(dW)
    modes = ["linear"] if kind == "advection" else ["exact", "fd"]

    def ops(ctx, blk):
        Wg, sg, dWg, dsg, bg = (to_gpu(blk(x)) for x in (W, sig, dW, ds, b))
        torch.cuda.synchronize()                 # inputs ready for the context's stream
        out = {"R1": ctx.rhs(Wg), "R2": ctx.rhs(Wg, sg)}
        G1, G2, nrm = ctx.residual(a1, a2, dt, bg, Wg, sg, norm=True)
        out["G"] = (G1, G2)
        for md in modes:
            out["jvp_" + md] = ctx.jvp(a1, a2, dt, Wg, sg, dWg, dsg, mode=md,
                                       eps_override=(eps, None) if md == "fd" else None)
        ctx.precond_build(a1, a2, dt, Wg)
        out["pc"] = ctx.precond_apply(dWg, dsg)
        torch.cuda.synchronize()                 # the context's stream is done
        res = {k: (np.concatenate([to_np(x) for x in v]) if isinstance(v, tuple) else to_np(v))
               for k, v in out.items()}
        res["Gnorm"] = nrm
        return res

    ref = ops(ctx1, lambda x: x)
    # the single-rank path against the oracle
    assert rel(ref["R1"], dgsem.rhs1(d, W)) <= 1e-11
    group = hbpdc.LoopbackGroup(px * py)
    ctxs = _rank_contexts(kind, N, nx, ny, px, py, group)
    try:
        outs = _run_threads([lambda c=c: ops(c, lambda x, c=c: _block(x, dim, nx, ny or 1, d.m, c.ex0, c.ey0,
                                                                      c.nx_local, c.ny_local))
                             for c in ctxs])
        for c, o in zip(ctxs, outs):
            blk = lambda x: _block(x, dim, nx, ny or 1, d.m, c.ex0, c.ey0, c.nx_local, c.ny_local)  # noqa: E731
            for key in ref:
                if key == "Gnorm":
                    assert abs(o[key] - ref[key]) <= 1e-14 * ref[key]       # global norm, rank-order sum
                    continue
                n = d.n
                r = ref[key]
                rb = np.concatenate([blk(r[:n]), blk(r[n:])]) if r.size == 2 * n else blk(r)
                assert np.array_equal(o[key], rb), (key, c.rank, np.abs(o[key] - rb).max())
    finally:
        for c in ctxs:
            c.close()
        group.close()


@pytest.mark.parametrize("px,py", [(2, 2), (2, 1)])
def test_loopback_hbpc_step(px, py):
    """C3 physics (vortex + noise), 4x4 elements N=3, HBPC(6,2), one step:
    partitioned vs single rank vs the oracle."""
    import torch
    cfg = configs.scaled(configs.CONFIGS["C3"], N=3, nx=4, ny=4, q=6, kmax=2)
    d, ctx1 = make_pair("euler", cfg.N, cfg.nx, cfg.ny, bounds=cfg.bounds, q=cfg.q, kmax=cfg.kmax,
                        gmres_rtol=cfg.gmres_rtol, newton_rtol=cfg.newton_rtol)
    W0 = inputs.initial_state("C3", d.node_coords(), noise=cfg.noise)
    dt = configs.cfl_dt(cfg, inputs.initial_state("C3", d.node_coords()))
    W1 = to_gpu(W0)
    st1 = ctx1.step(dt, W1)
    W1 = to_np(W1)
    Wo = hbpc.HBPC(d, cfg.q, cfg.kmax, implicit.NewtonOpts(rtol=cfg.newton_rtol,
                                                           gmres_rtol=cfg.gmres_rtol)).step(W0, dt)
    assert rel(W1, Wo) <= 1e-8
    group = hbpdc.LoopbackGroup(px * py)
    ctxs = []
    for r in range(px * py):
        ctxs.append(hbpdc.Context(dim=2, equation="euler", N=cfg.N, nx=cfg.nx, ny=cfg.ny, bounds=cfg.bounds,
                                  q=cfg.q, kmax=cfg.kmax, gmres_rtol=cfg.gmres_rtol, newton_rtol=cfg.newton_rtol,
                                  rank=r, nranks=px * py, px=px, py=py, comm="loopback", loopback=group,
                                  stream=torch.cuda.Stream()))
    try:
        def run(c):
            Wl = to_gpu(_block(W0, 2, cfg.nx, cfg.ny, d.m, c.ex0, c.ey0, c.nx_local, c.ny_local))
            torch.cuda.synchronize()
            st = c.step(dt, Wl)
            torch.cuda.synchronize()
            return to_np(Wl), st
        outs = _run_threads([lambda c=c: run(c) for c in ctxs])
        for c, (Wl, st) in zip(ctxs, outs):
            blk = _block(W1, 2, cfg.nx, cfg.ny, d.m, c.ex0, c.ey0, c.nx_local, c.ny_local)
            assert rel(Wl, blk) <= 1e-10, (c.rank, rel(Wl, blk))
            assert st["gmres_its"] == outs[0][1]["gmres_its"]        # identical global decisions
        assert abs(outs[0][1]["gmres_its"] - st1["gmres_its"]) <= max(2, st1["gmres_its"] // 20)
    finally:
        for c in ctxs:
            c.close()
        group.close()


def test_nccl_self_halo():
    """The NCCL transport on one GPU: nranks = 1 with the periodic wrap forced
    through a self halo (ncclSend/ncclRecv to oneself and a 1-rank all-reduce)."""
    import torch
    kind, N, nx, ny = "euler", 3, 4, 4
    d, ctx1 = make_pair(kind, N, nx, ny)
    nid = hbpdc.nccl_unique_id()
    ctxn = hbpdc.Context(dim=2, equation=kind, N=N, nx=nx, ny=ny, comm="nccl", nccl_id=nid, force_halo=True)
    W = euler_ic(d, SEED + 41)
    sig = dgsem.rhs1(d, W) * (1 + 1e-2 * inputs.random_field(d.n, SEED + 42))
    dW = inputs.random_field(d.n, SEED + 43, unit_norm=True)
    ds = inputs.random_field(d.n, SEED + 44, unit_norm=True)
    torch.cuda.synchronize()
    r1 = [to_np(c.rhs(to_gpu(W))) for c in (ctx1, ctxn)]
    assert np.array_equal(r1[0], r1[1])
    j = [np.concatenate([to_np(x) for x in c.jvp(0.5, 1 / 6, 0.02, to_gpu(W), to_gpu(sig), to_gpu(dW),
                                                 to_gpu(ds), mode="exact")]) for c in (ctx1, ctxn)]
    assert np.array_equal(j[0], j[1])
    cfg = configs.scaled(configs.CONFIGS["C3"], N=3, nx=4, ny=4, q=4, kmax=0)
    W0 = inputs.initial_state("C3", d.node_coords(), noise=cfg.noise)
    dt = 0.05
    outs = []
    for c in (ctx1, ctxn):
        Wg = to_gpu(W0)
        c.step(dt, Wg)
        torch.cuda.synchronize()
        outs.append(to_np(Wg))
    assert rel(outs[1], outs[0]) <= 1e-10
    ctxn.close()
