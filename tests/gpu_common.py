"""Shared helpers for the GPU parity tests: build matching oracle / GPU
discretisations and seeded inputs (paper_2109_04804_b200.inputs)."""
import numpy as np

from oracle import basis, dgsem, physics
from paper_2109_04804_b200 import inputs

SEED = inputs.MASTER_SEED


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def make_pair(kind, N, nx, ny=None, bounds=(0.0, 1.0, 0.0, 1.0), a=(1.0, 1.0), mu=0.0, q=4, kmax=0, **ctx_kw):
    """(oracle Disc, GPU Context) for the same problem."""
    from paper_2109_04804_b200 import hbpdc
    dim = 1 if ny is None else 2
    eq = physics.Equation(kind, a=tuple(a), mu=mu, numflux=ctx_kw.get("flux", "llf"), mach=ctx_kw.get("mach", 1.0),
                          lifting=ctx_kw.get("lifting", "br1"), eta_br2=ctx_kw.get("eta_br2", 2.0))
    d = dgsem.Disc(basis.build_basis(N, ctx_kw.get("nodes", "gll")), dgsem.Mesh(dim, nx, ny or 1, *bounds), eq)
    ctx = hbpdc.Context(dim=dim, equation=kind, N=N, nx=nx, ny=ny or 1, bounds=bounds, a=a, mu=mu, q=q,
                        kmax=kmax, **ctx_kw)
    return d, ctx


def euler_ic(d, seed, rel_noise=1e-2):
    """Perturbed smooth Euler state (SURVEY 8(c4) recipe): density wave + noise."""
    X, Y = d.node_coords()
    W = inputs.initial_state("C4", (X / (d.mesh.xmax - d.mesh.xmin), Y / (d.mesh.ymax - d.mesh.ymin)))
    return inputs.perturbed_state(W, seed, rel_noise)


def ns_ic(d, seed, rel_noise=1e-2):
    X, Y = d.node_coords()
    W = inputs.initial_state("C5", (X, Y))
    return inputs.perturbed_state(W, seed, rel_noise)


def adv_ic(d, seed, rel_noise=1e-2):
    if d.mesh.dim == 1:
        W = inputs.initial_state("C1", d.node_coords())
    else:
        W = inputs.initial_state("C2", d.node_coords())
    return W + inputs.random_field(d.n, seed, rel_noise)


def to_gpu(x):
    import torch
    return torch.tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")


def to_np(t):
    return t.detach().cpu().numpy()
