"""Pins for oracle.dgsem: R1, R2, BR1 lifting.  CPU only."""
import json
import math
import os

import numpy as np
import pytest

from oracle import basis, dgsem, physics
from paper_2109_04804_b200 import inputs

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def make(kind, N, nx, ny=None, nodes="gll", bounds=(0.0, 1.0, 0.0, 1.0), **kw):
    eq = physics.Equation(kind, **kw)
    dim = 1 if ny is None else 2
    me = dgsem.Mesh(dim, nx, ny or 1, *bounds)
    return dgsem.Disc(basis.build_basis(N, nodes), me, eq)


def const_state(d, vals):
    W = np.zeros(d.field_shape())
    for v, x in enumerate(vals):
        W[:, :, v] = x
    return W.reshape(-1)


def test_mesh_example():
    g = GOLD["mesh_16"]
    me = dgsem.Mesh(2, 16, 16, -1, 1, -1, 1)
    assert me.dx == g["dx"] and me.dx * me.dy / 4 == g["jgeo"] and me.dy / 2 == g["shat"]


@pytest.mark.parametrize("nodes", ["gl", "gll"])
@pytest.mark.parametrize("kind", ["euler", "navier_stokes"])
def test_free_stream(kind, nodes):
    """R1 and R2 vanish on a constant state (reading R26)."""
    d = make(kind, 4, 3, 4, nodes=nodes, mu=1e-3)
    W = const_state(d, [1.2, 0.3, -0.4, 2.7])
    R1 = dgsem.rhs1(d, W)
    scale = (2 / d.mesh.dx) * 3.0
    assert np.abs(R1).max() < 1e-13 * scale
    sig = const_state(d, [0.1, 0.2, 0.3, 0.4])
    assert np.abs(dgsem.rhs2(d, W, sig)).max() < 1e-13 * scale


def _quad_sums(d, F):
    """sum_e sum_ij w_i w_j J (field)_v per variable."""
    b, me = d.basis, d.mesh
    Ff = F.reshape(d.field_shape())
    ww = np.outer(b.w, b.w)
    return np.array([(Ff[:, :, v] * ww).sum() for v in range(d.nv)]) * me.dx * me.dy / 4, \
        np.array([(np.abs(Ff[:, :, v]) * ww).sum() for v in range(d.nv)]) * me.dx * me.dy / 4


@pytest.mark.parametrize("kind", ["advection", "euler", "navier_stokes"])
def test_discrete_conservation(kind):
    """Quadrature-weighted sums of R1 and R2 vanish per variable on periodic
    meshes (reading R27)."""
    d = make(kind, 3, 4, 3, mu=1e-2, a=(0.7, -0.4))
    rng = np.random.default_rng(3)
    if kind == "advection":
        W = rng.standard_normal(d.n)
    else:
        W = const_state(d, [1.0, 0.2, 0.1, 2.5]) * (1 + 0.1 * rng.uniform(-1, 1, d.n))
    sig = rng.standard_normal(d.n)
    for F in (dgsem.rhs1(d, W), dgsem.rhs2(d, W, sig)):
        s, a = _quad_sums(d, F)
        assert np.all(np.abs(s) <= 1e-12 * a)


def test_advection_spectral_accuracy():
    """On a smooth field R1 converges to -a.grad(w) at rate >= N."""
    errs = []
    for n in (4, 8):
        d = make("advection", 5, n, n, a=(1.0, 1.0))
        X, Y = d.node_coords()
        W = inputs.initial_state("C2", (X, Y))
        exact = inputs.layout((-2 * math.pi * (np.cos(2 * math.pi * X) * np.sin(2 * math.pi * Y)
                                               + np.sin(2 * math.pi * X) * np.cos(2 * math.pi * Y)),), 2)
        errs.append(np.abs(dgsem.rhs1(d, W) - exact).max())
    assert errs[1] < 5e-4 and errs[0] / errs[1] > 2 ** 4.5


def test_advection_linearity_and_r2_equals_r1():
    """Advection: R1 linear; R2(w, s) = R1(s)."""
    d = make("advection", 3, 5, 4, a=(0.3, -1.1))
    rng = np.random.default_rng(4)
    a, b = rng.standard_normal(d.n), rng.standard_normal(d.n)
    lhs = dgsem.rhs1(d, 2.0 * a - 3.0 * b)
    rhs = 2.0 * dgsem.rhs1(d, a) - 3.0 * dgsem.rhs1(d, b)
    assert np.abs(lhs - rhs).max() < 1e-12 * np.abs(rhs).max()
    np.testing.assert_allclose(dgsem.rhs2(d, a, b), dgsem.rhs1(d, b), rtol=0, atol=1e-12)


@pytest.mark.parametrize("nodes", ["gll", "gl"])
def test_upwind_1d_matches_dense_formula(nodes):
    """1D advection, a > 0: assemble R1 element-wise from the textbook weak
    form with exact upwinding,  w_t,i = (2/dx)/w_i [ a sum_l w_l l'_i(x_l) w_l
    - a w(1) l_i(1) + a w_left(1) l_i(-1) ], and compare."""
    d = make("advection", 3, 6, a=(0.8, 0.0), nodes=nodes)
    b = d.basis
    rng = np.random.default_rng(5)
    W = rng.standard_normal(d.n).reshape(6, 1, 4)[:, 0, :]
    out = np.zeros_like(W)
    for e in range(6):
        wl = W[e - 1] @ b.l_plus                 # upwind trace at the left face
        wr = W[e] @ b.l_plus                     # own trace at the right face
        for i in range(4):
            vol = 0.8 * sum(b.w[l] * b.D[l, i] * W[e, l] for l in range(4))
            out[e, i] = (2 / d.mesh.dx) / b.w[i] * (vol - 0.8 * wr * b.l_plus[i] + 0.8 * wl * b.l_minus[i])
    np.testing.assert_allclose(dgsem.rhs1(d, W.reshape(-1)), out.reshape(-1), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("kind", ["euler", "navier_stokes"])
def test_r2_is_time_derivative_of_r1(kind):
    """R2(W, s) = d/dt R1(W + t s) at t = 0, checked against
    central differences of the plain R1."""
    d = make(kind, 3, 3, 4, mu=5e-2)
    rng = np.random.default_rng(6)
    W = const_state(d, [1.0, 0.3, -0.2, 2.5]) * (1 + 0.05 * rng.uniform(-1, 1, d.n))
    s = rng.standard_normal(d.n) * 0.1
    h = 1e-5
    fd = (dgsem.rhs1(d, W + h * s) - dgsem.rhs1(d, W - h * s)) / (2 * h)
    r2 = dgsem.rhs2(d, W, s)
    assert np.linalg.norm(r2 - fd) <= 1e-7 * np.linalg.norm(r2)


def test_lifting_derivative_convergence():
    """BR1 lifted gradient of a smooth velocity field converges to the exact
    gradient, rate >= N."""
    errs = []
    for n in (4, 8):
        d = make("navier_stokes", 4, n, n, bounds=(0, 2 * math.pi, 0, 2 * math.pi), mu=1e-3)
        X, Y = d.node_coords()
        W = inputs.initial_state("C5", (X, Y))
        gx, gy = dgsem.lifting(d, d.to_field(W))
        ux_exact = np.cos(X) * np.cos(Y)
        vy_exact = -np.cos(X) * np.cos(Y)
        errs.append(max(np.abs(gx[0] - ux_exact).max(), np.abs(gy[1] - vy_exact).max()))
    assert errs[1] < 1e-3 and errs[0] / errs[1] > 2 ** 3.5


def test_lifting_constant_is_zero():
    d = make("navier_stokes", 3, 3, 3, mu=1e-3)
    W = const_state(d, [1.0, 0.5, 0.2, 3.0])
    gx, gy = dgsem.lifting(d, d.to_field(W))
    assert max(np.abs(g).max() for g in gx + gy) < 1e-12


# ---- BR2 lifting (reading R33) ------------------------------------
def _br2(N=3, nx=4, ny=3, eta=2.0, nodes="gll"):
    return make("navier_stokes", N, nx, ny, nodes=nodes, bounds=(0, 2 * math.pi, 0, 2 * math.pi), mu=5e-2,
                lifting="br2", eta_br2=eta)


def test_br2_eta1_face_gradients_match_br1_traces():
    """GLL, eta = 1: the local lifting of face f evaluated on f equals the trace of
    the (independently computed, weak-form) BR1 lifted gradient in the normal
    component everywhere, and in the tangential component away from the corner
    nodes (where BR1 also carries the other direction's face term)."""
    d = _br2(eta=1.0)
    rng = np.random.default_rng(11)
    W = const_state(d, [1.0, 0.3, -0.2, 2.5]) * (1 + 0.05 * rng.uniform(-1, 1, d.n))
    Wf = d.to_field(W)
    gx, gy = dgsem.lifting(d, Wf)
    G = [np.stack(gx, axis=2), np.stack(gy, axis=2)]
    ops = dgsem._Ops(d)
    br2 = dgsem.lifting_br2_faces(d, Wf)
    for dd in range(2):
        br1_faces = [ops.faces(G[c], dd) for c in range(2)]        # per component: (own+, nbr+, nbr-, own-)
        for t in range(4):
            for c in range(2):
                a, b = br2[dd][t][c], br1_faces[c][t]
                if c == dd:
                    np.testing.assert_allclose(a, b, rtol=0, atol=1e-11 * np.abs(b).max())
                else:
                    np.testing.assert_allclose(a[..., 1:-1], b[..., 1:-1], rtol=0, atol=1e-11 * np.abs(b).max())
                    assert np.abs(a[..., [0, -1]] - b[..., [0, -1]]).max() > 1e-6   # corners differ


@pytest.mark.parametrize("nodes", ["gll", "gl"])
def test_br2_free_stream_conservation_and_r2(nodes):
    """BR2 (eta = 2): free stream, discrete conservation (the viscous surface flux
    stays single valued), R2 = d/dt R1 by central differences, and eta
    enters R1 (the jump terms reach the viscous face flux)."""
    d = _br2(nodes=nodes)
    assert np.abs(dgsem.rhs1(d, const_state(d, [1.2, 0.3, -0.2, 2.5]))).max() < 1e-13
    rng = np.random.default_rng(12)
    W = const_state(d, [1.0, 0.3, -0.2, 2.5]) * (1 + 0.05 * rng.uniform(-1, 1, d.n))
    R = dgsem.rhs1(d, W)
    wq = np.outer(d.basis.w, d.basis.w).reshape(-1)
    cons = (R.reshape(-1, 4, d.p * d.p) * wq).sum(axis=(0, 2))
    assert np.abs(cons).max() <= 1e-12 * np.abs(R).max()
    s = rng.standard_normal(d.n) * 0.1
    h = 1e-5
    fd = (dgsem.rhs1(d, W + h * s) - dgsem.rhs1(d, W - h * s)) / (2 * h)
    r2 = dgsem.rhs2(d, W, s)
    assert np.linalg.norm(r2 - fd) <= 1e-7 * np.linalg.norm(r2)
    R4 = dgsem.rhs1(_br2(nodes=nodes, eta=4.0), W)
    assert np.linalg.norm(R4 - R) > 1e-6 * np.linalg.norm(R)


def test_br2_face_gradients_converge():
    """BR2 face gradients of a smooth velocity field converge to the exact gradient
    on the faces (the jump terms vanish with the jumps)."""
    errs = []
    for n in (4, 8):
        d = make("navier_stokes", 4, n, n, bounds=(0, 2 * math.pi, 0, 2 * math.pi), mu=1e-3, lifting="br2")
        X, Y = d.node_coords()
        W = inputs.initial_state("C5", (X, Y))
        br2 = dgsem.lifting_br2_faces(d, d.to_field(W))
        ops = dgsem._Ops(d)
        ux = np.cos(X) * np.cos(Y)                     # u = sin x cos y (C5): u_x
        e = 0.0
        for dd in range(2):
            own_p = br2[dd][0][0][:, :, 0]                # x-gradient of u on the + face in direction dd
            e = max(e, np.abs(own_p - ops.trace(ux, dd, +1)).max())
        errs.append(e)
    assert errs[1] < 1e-3 and errs[0] / errs[1] > 2 ** 3.5


def _exact_time_derivative(case, X, Y):
    """w_t of an exactly translating Euler solution with mean flow (1, 1):
    w(x, t) = w0(x - t, y - t), so w_t = -(d/dx + d/dy) w0.  The spatial
    derivatives of the analytic IC are taken by complex step (exact to
    rounding), independent of any flux formula."""
    h = 1e-30
    Wx = inputs.layout(inputs.ic_primitive(case, X + 1j * h, Y), 2).imag / h
    Wy = inputs.layout(inputs.ic_primitive(case, X, Y + 1j * h), 2).imag / h
    return -(Wx + Wy)


@pytest.mark.parametrize("case,N,nxs,bounds,nodes,numflux,min_eoc", [
    # isentropic vortex (C3 family, beta = 5, mean flow (1, 1)) on a domain wide
    # enough that the periodic wrap of its Gaussian tail is below rounding
    ("C3", 4, (16, 32, 64), (-10.0, 10.0, -10.0, 10.0), "gll", "llf", 3.5),
    ("C3", 3, (16, 32, 64), (-10.0, 10.0, -10.0, 10.0), "gl", "glf", 2.5),
    # density wave (C4 family): rho = 1 + 0.2 sin(2 pi (x + y)), u = v = p = 1
    ("C4", 3, (4, 8, 16), (0.0, 1.0, 0.0, 1.0), "gll", "llf", 2.8),
    ("C4", 5, (4, 8, 16), (0.0, 1.0, 0.0, 1.0), "gl", "glf", 4.5),
])
def test_euler_r1_converges_to_exact_translation(case, N, nxs, bounds, nodes, numflux, min_eoc):
    """Spatial-order pin of R^(1) for the Euler equations against exact solutions
    of the PDE (eq:Euler P:388-394, eq:DGSEM_wt P:179-201):
    the nodal truncation error ||R1(I_h w0) - I_h w_t||, with w_t of the exactly
    translating vortex / density wave, decays like h^N.  A wrong flux term
    (e.g. the energy flux v E instead of v (E + p), or a momentum flux without
    p) leaves an O(1) error that does not converge."""
    eq = physics.Equation("euler", numflux=numflux)
    errs = []
    for nx in nxs:
        d = dgsem.Disc(basis.build_basis(N, nodes), dgsem.Mesh(2, nx, nx, *bounds), eq)
        X, Y = d.node_coords()
        W = inputs.layout(inputs.ic_primitive(case, X, Y), 2)
        wt = _exact_time_derivative(case, X, Y)
        R = dgsem.rhs1(d, W)
        errs.append(float(np.sqrt(np.mean((R - wt) ** 2)) / np.sqrt(np.mean(wt ** 2))))
    eoc = [math.log2(a / b) for a, b in zip(errs[:-1], errs[1:])]
    assert eoc[-1] >= min_eoc, (errs, eoc)
    assert errs[-1] < 5e-3, errs
