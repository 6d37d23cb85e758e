"""Pins for the 3D extension of the oracle (NEXT-4: hexahedral elements, the
paper's 3D Taylor-Green case P:1080-1093, inviscid scope).  CPU only.

The 3D operators are pinned to things other than themselves: the pinned 2D
oracle (a z- or x-independent 3D state reduces exactly to a 2D problem),
exact PDE solutions (spatial order of the truncation error), free stream,
discrete conservation, the time-derivative definition of R2, brute-force
Jacobians and the (2,2)-Pade closed form of HBPC(4,0) for advection."""
import math

import numpy as np
import pytest
import scipy.linalg as sla

from oracle import ad, basis, dgsem, hbpc, implicit, physics
from paper_2109_04804_b200 import inputs


def disc3(kind, N, n, bounds=(0.0, 1.0), nodes="gll", **kw):
    eq = physics.Equation(kind, dim=3, **kw) if kind != "advection" else physics.Equation(kind, dim=3, **kw)
    me = dgsem.Mesh(3, n[0], n[1], bounds[0], bounds[1], bounds[0], bounds[1], nz=n[2], zmin=bounds[0], zmax=bounds[1])
    return dgsem.Disc(basis.build_basis(N, nodes), me, eq)


def euler3_state(d, seed, amp=0.05):
    rng = np.random.default_rng(seed)
    W = np.zeros(d.field_shape())
    for v, x in enumerate([1.0, 0.3, -0.2, 0.25, 2.5]):
        W[:, :, :, v] = x
    return W.reshape(-1) * (1 + amp * rng.uniform(-1, 1, d.n))


@pytest.mark.parametrize("nodes", ["gll", "gl"])
def test_free_stream_3d(nodes):
    d = disc3("euler", 3, (3, 2, 4), nodes=nodes)
    W = np.zeros(d.field_shape())
    for v, x in enumerate([1.1, 0.2, -0.3, 0.4, 2.4]):
        W[:, :, :, v] = x
    R = dgsem.rhs1(d, W.reshape(-1))
    assert np.abs(R).max() < 1e-12 * 2 * 4 * 10


def test_discrete_conservation_3d():
    d = disc3("euler", 2, (3, 3, 3))
    W = euler3_state(d, 3)
    R = dgsem.rhs1(d, W).reshape(d.mesh.n_elem, 5, -1)
    w = d.basis.w
    wq = np.einsum("k,j,i->kji", w, w, w).reshape(-1)
    for v in range(5):
        tot = np.sum(R[:, v] * wq)
        assert abs(tot) <= 1e-12 * np.sum(np.abs(R[:, v]) * wq)


@pytest.mark.parametrize("flux", ["llf", "glf"])
def test_z_independent_state_reduces_to_2d(flux):
    """A 3D state independent of z with zero z-momentum is a 2D solution: R1_3D
    on every z-layer equals the pinned 2D R1 of (rho, rho u, rho v, E), and the
    z-momentum component of R1_3D vanishes (eq:DGSEM_wt)."""
    N, n = 3, (3, 4, 2)
    d3 = disc3("euler", N, n, numflux=flux)
    d2 = dgsem.Disc(basis.build_basis(N, "gll"), dgsem.Mesh(2, n[0], n[1], 0.0, 1.0, 0.0, 1.0),
                    physics.Equation("euler", numflux=flux))
    W2 = np.zeros(d2.field_shape())
    rng = np.random.default_rng(5)
    for v, x in enumerate([1.0, 0.3, -0.2, 2.5]):
        W2[:, :, v] = x * (1 + 0.05 * rng.uniform(-1, 1, W2[:, :, v].shape))
    R2 = dgsem.rhs1(d2, W2.reshape(-1)).reshape(d2.field_shape())
    p = N + 1
    W3 = np.zeros(d3.field_shape())          # (nz, ny, nx, 5, k, j, i)
    for v3, v2 in zip((0, 1, 2, 4), (0, 1, 2, 3)):
        W3[:, :, :, v3] = W2[None, :, :, v2, None, :, :]
    R3 = dgsem.rhs1(d3, W3.reshape(-1)).reshape(d3.field_shape())
    sc = np.abs(R2).max()
    for v3, v2 in zip((0, 1, 2, 4), (0, 1, 2, 3)):
        np.testing.assert_allclose(R3[:, :, :, v3], np.broadcast_to(R2[None, :, :, v2, None], R3[:, :, :, v3].shape),
                                   rtol=0, atol=1e-12 * sc)
    assert np.abs(R3[:, :, :, 3]).max() <= 1e-12 * sc


def test_x_independent_state_reduces_to_2d_in_yz():
    """Same in the (y, z) plane: the 2D problem in (x', y') = (y, z) with the
    momenta (rho v, rho w) -- pins the y and z directions of the 3D operator."""
    N, n = 2, (2, 3, 4)
    d3 = disc3("euler", N, n)
    d2 = dgsem.Disc(basis.build_basis(N, "gll"), dgsem.Mesh(2, n[1], n[2], 0.0, 1.0, 0.0, 1.0),
                    physics.Equation("euler"))
    W2 = np.zeros(d2.field_shape())           # (ny2 = nz, nx2 = ny, 4, j2 = k, i2 = j)
    rng = np.random.default_rng(6)
    for v, x in enumerate([1.0, 0.3, -0.2, 2.5]):
        W2[:, :, v] = x * (1 + 0.05 * rng.uniform(-1, 1, W2[:, :, v].shape))
    R2 = dgsem.rhs1(d2, W2.reshape(-1)).reshape(d2.field_shape())
    W3 = np.zeros(d3.field_shape())          # (nz, ny, nx, 5, k, j, i)
    for v3, v2 in zip((0, 2, 3, 4), (0, 1, 2, 3)):
        W3[:, :, :, v3] = W2[:, :, None, v2, :, :, None]
    R3 = dgsem.rhs1(d3, W3.reshape(-1)).reshape(d3.field_shape())
    sc = np.abs(R2).max()
    for v3, v2 in zip((0, 2, 3, 4), (0, 1, 2, 3)):
        np.testing.assert_allclose(R3[:, :, :, v3],
                                   np.broadcast_to(R2[:, :, None, v2, :, :, None], R3[:, :, :, v3].shape),
                                   rtol=0, atol=1e-12 * sc)
    assert np.abs(R3[:, :, :, 1]).max() <= 1e-12 * sc


def _dt_exact(case, X, Y, Z, vel):
    h = 1e-30
    parts = [inputs.layout(inputs.ic_primitive(case, *(c + (1j * h if k == a else 0.0) for k, c in enumerate((X, Y, Z)))), 3).imag / h
             for a in range(3)]
    return -sum(v * p for v, p in zip(vel, parts))


@pytest.mark.parametrize("case,kind,N,ns,min_eoc", [("DW3", "euler", 3, (2, 4, 8), 2.7),
                                                     ("ADV3", "advection", 3, (2, 4, 8), 2.7)])
def test_r1_converges_to_exact_translation_3d(case, kind, N, ns, min_eoc):
    """Spatial order in 3D against exact solutions: the nodal truncation error
    ||R1(I_h w0) - I_h w_t|| of the translating density wave (v = (1,1,1)) and of
    advected sin x sin y sin z (a = (1,1,1)) decays like h^N."""
    errs = []
    for n in ns:
        kw = {"a": (1.0, 1.0, 1.0)} if kind == "advection" else {}
        d = disc3(kind, N, (n, n, n), **kw)
        X, Y, Z = d.node_coords()
        W = inputs.layout(inputs.ic_primitive(case, X, Y, Z), 3)
        wt = _dt_exact(case, X, Y, Z, (1.0, 1.0, 1.0))
        R = dgsem.rhs1(d, W)
        errs.append(float(np.sqrt(np.mean((R - wt) ** 2)) / np.sqrt(np.mean(wt ** 2))))
    eoc = [math.log2(a / b) for a, b in zip(errs[:-1], errs[1:])]
    assert eoc[-1] >= min_eoc, (errs, eoc)


def test_r2_is_time_derivative_3d():
    """R2(W, R1(W)) = d/dt R1(W(t)) along the semi-discrete trajectory."""
    d = disc3("euler", 2, (2, 3, 2))
    W = euler3_state(d, 8)
    R1 = dgsem.rhs1(d, W)
    R2 = dgsem.rhs2(d, W, R1)
    h = 1e-5
    fd = (dgsem.rhs1(d, W + h * R1) - dgsem.rhs1(d, W - h * R1)) / (2 * h)
    np.testing.assert_allclose(R2, fd, rtol=0, atol=1e-7 * np.abs(R2).max())


def test_exact_jvp_equals_assembled_jacobian_3d():
    """3x3x3 elements, N = 1, Euler 3D (2n = 2160): EXACT JVP = brute-force
    assembled Jacobian of G times dX."""
    d = disc3("euler", 1, (3, 3, 3))
    n = d.n
    W = euler3_state(d, 9)
    rng = np.random.default_rng(10)
    sig = dgsem.rhs1(d, W) * (1 + 0.01 * rng.standard_normal(n))
    b = W * (1 + 1e-3 * rng.standard_normal(n))
    a1, a2, dt = 0.5, 1 / 6, 0.02
    dW, ds = rng.standard_normal(n), rng.standard_normal(n)
    # columns of the Jacobian along dX by central differences of G (the brute force)
    h = 1e-6
    X = np.concatenate([W, sig])
    dX = np.concatenate([dW, ds])
    Gp = np.concatenate(implicit.residual(d, a1, a2, dt, b, *np.split(X + h * dX, 2)))
    Gm = np.concatenate(implicit.residual(d, a1, a2, dt, b, *np.split(X - h * dX, 2)))
    fd = (Gp - Gm) / (2 * h)
    t, bo = implicit.jvp_exact(d, a1, a2, dt, W, sig, dW, ds)
    ex = np.concatenate([t, bo])
    assert np.linalg.norm(ex - fd) <= 1e-7 * np.linalg.norm(ex)


def test_hbpc4_step_is_pade_3d_advection():
    """HBPC(4,0) on 3D advection is the (2,2)-Pade map of the dense DGSEM matrix."""
    d = disc3("advection", 1, (2, 2, 3), a=(1.0, 0.5, -0.7))
    K = np.stack([dgsem.rhs1(d, e) for e in np.eye(d.n)], axis=1)
    X, Y, Z = d.node_coords()
    W0 = inputs.layout(inputs.ic_primitive("ADV3", X, Y, Z), 3)
    dt = 0.05
    H = hbpc.HBPC(d, 4, 0, implicit.NewtonOpts(rtol=1e-13, gmres_rtol=1e-13))
    W1 = H.step(W0, dt)
    I = np.eye(d.n)
    P = np.linalg.solve(I - dt * K / 2 + dt * dt * K @ K / 12, (I + dt * K / 2 + dt * dt * K @ K / 12) @ W0)
    np.testing.assert_allclose(W1, P, rtol=0, atol=1e-11 * np.abs(P).max())


def test_element_jacobians_3d_brute_force():
    """K_i by the 3D colouring = brute-force element block of dR1/dW."""
    d = disc3("euler", 1, (3, 3, 3))
    W = euler3_state(d, 11)
    K = implicit.element_jacobians(d, W)
    m = d.m
    e = 13                                     # an interior element of the 3x3x3 mesh
    h = 1e-6
    Kb = np.zeros((m, m))
    for c in range(m):
        dv = np.zeros(d.n)
        dv[e * m + c] = h
        Kb[:, c] = ((dgsem.rhs1(d, W + dv) - dgsem.rhs1(d, W - dv)) / (2 * h))[e * m:(e + 1) * m]
    np.testing.assert_allclose(K[e], Kb, rtol=0, atol=1e-7 * np.abs(Kb).max())
