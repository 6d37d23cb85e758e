"""Pins for oracle.physics and oracle.ad.  CPU only."""
import json
import math
import os

import numpy as np
import pytest

from oracle import ad, physics

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))
EU = physics.Equation("euler")
NS = physics.Equation("navier_stokes", mu=1e-3)


def test_euler_flux_example():
    g = GOLD["euler_flux_eps1"]
    w = tuple(np.array(x) for x in g["w"])
    assert float(physics.pressure(EU, w)) == pytest.approx(g["p"], abs=1e-15)
    np.testing.assert_allclose([float(f) for f in physics.flux(EU, w, 0)], g["Fx"], atol=1e-15)


def test_pressure_example():
    g = GOLD["pressure"]
    # S:140 uses the momentum components as given (rho v = 0.3)
    w = tuple(np.array(x) for x in g["w"])
    assert float(physics.pressure(EU, w)) == pytest.approx(g["p"], abs=1e-12)


def test_advection_flux_and_upwind():
    g = GOLD["advection_flux"]
    eq = physics.Equation("advection", a=tuple(g["a"]))
    assert physics.flux(eq, (np.array(g["w"]),), 0)[0] == pytest.approx(g["Fx"])
    assert physics.flux(eq, (np.array(g["w"]),), 1)[0] == pytest.approx(g["Fy"])
    u = GOLD["llf_upwind"]
    f = physics.llf(eq, (np.array(u["wL"]),), (np.array(u["wR"]),), 0)[0]
    assert float(f) == pytest.approx(u["fstar_llf"], abs=1e-15)
    # the exact upwind flux: a>0 takes the left state
    assert float(f) == pytest.approx(0.3 * u["wL"], abs=1e-15)


def _rand_states(rng, n=50):
    rho = rng.uniform(0.5, 2.0, n)
    u, v = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    p = rng.uniform(0.5, 2.0, n)
    return (rho, rho * u, rho * v, p / 0.4 + 0.5 * rho * (u * u + v * v))


def test_llf_consistency_and_conservation():
    rng = np.random.default_rng(1)
    wL, wR = _rand_states(rng), _rand_states(rng)
    for d in range(2):
        F = physics.flux(EU, wL, d)
        fc = physics.llf(EU, wL, wL, d)
        for a, b in zip(F, fc):
            np.testing.assert_allclose(a, b, rtol=1e-15, atol=1e-15)
        # f*(L, R; +e) and the flux the right element sees with its outward
        # normal are exact negatives (canonical orientation) -- and the flux
        # is symmetric under L<->R swap with normal flip:
        #   f*(wL, wR, n) = -f*(wR, wL, -n): with -n the physical flux and the
        # velocity flip sign, so mirror the states' normal momentum.
        fl = physics.llf(EU, wL, wR, d)
        mir = lambda w: tuple(-x if k == 1 + d else x for k, x in enumerate(w))
        fr = physics.llf(EU, mir(wR), mir(wL), d)
        for k in range(4):
            sgn = 1.0 if k == 1 + d else -1.0
            np.testing.assert_allclose(fl[k], sgn * fr[k], rtol=1e-13, atol=1e-13)


def test_dual_derivatives_match_central_fd():
    """(dF/dw) sigma from the dual part equals central differences of the
    plain flux; the d12 part equals FD of the d1 part."""
    rng = np.random.default_rng(2)
    w, s, t = _rand_states(rng), _rand_states(rng), _rand_states(rng)
    h = 1e-6
    for d in range(2):
        J = physics.llf(EU, tuple(ad.Jet(a, b, c) for a, b, c in zip(w, s, t)),
                        tuple(ad.Jet(a + 0.1, b, c) for a, b, c in zip(w, s, t)), d)
        fp = physics.llf(EU, tuple(a + h * b for a, b in zip(w, s)),
                         tuple(a + 0.1 + h * b for a, b in zip(w, s)), d)
        fm = physics.llf(EU, tuple(a - h * b for a, b in zip(w, s)),
                         tuple(a + 0.1 - h * b for a, b in zip(w, s)), d)
        for k in range(4):
            fd = (fp[k] - fm[k]) / (2 * h)
            np.testing.assert_allclose(J[k].d1, fd, rtol=1e-7, atol=1e-7)
        # mixed second derivative: FD of the e1 part along direction t
        Jp = physics.llf(EU, tuple(ad.Jet(a + h * c, b) for a, b, c in zip(w, s, t)),
                         tuple(ad.Jet(a + 0.1 + h * c, b) for a, b, c in zip(w, s, t)), d)
        Jm = physics.llf(EU, tuple(ad.Jet(a - h * c, b) for a, b, c in zip(w, s, t)),
                         tuple(ad.Jet(a + 0.1 - h * c, b) for a, b, c in zip(w, s, t)), d)
        for k in range(4):
            fd = (Jp[k].d1 - Jm[k].d1) / (2 * h)
            np.testing.assert_allclose(J[k].d12, fd, rtol=1e-6, atol=1e-6)


def test_jet_rules():
    x = ad.Jet(np.array([2.0]), np.array([1.0]), np.array([3.0]), np.array([0.5]))
    # f = sqrt: f' = 1/(2 sqrt x), f'' = -1/(4 x^1.5)
    r = ad.sqrt(x)
    assert r.d12[0] == pytest.approx(0.5 / (2 * math.sqrt(2)) - 3.0 / (4 * 2 ** 1.5))
    r = ad.recip(x)
    assert r.d1[0] == pytest.approx(-0.25) and r.d12[0] == pytest.approx(-0.5 / 4 + 2 * 3 / 8)
    y = x * x                                   # (x^2)'' = 2: d12 = 2 x d12 + 2 d1 d2
    assert y.d12[0] == pytest.approx(2 * 2 * 0.5 + 2 * 1 * 3)
    assert ad.absval(ad.Jet(np.array([0.0]), np.array([1.0]))).d1[0] == 1.0   # sign(0)=+1
    m = ad.maxval(ad.Jet(np.array([1.0]), np.array([5.0])), ad.Jet(np.array([1.0]), np.array([7.0])))
    assert m.d1[0] == 5.0                                                    # tie -> first


def test_viscous_stress_examples():
    """d = 0 -> 0; pure shear u_y = s -> tau_xy = mu s; pure
    dilatation u_x = s -> tau_xx = 4/3 mu s, tau_yy = -2/3 mu s."""
    w = (np.array(1.0), np.array(0.0), np.array(0.0), np.array(2.5))
    z = np.array(0.0)
    s = 0.7
    F = physics.viscous_flux(NS, w, (z, z, z), (z, z, z), 0)
    assert all(float(f) == 0.0 for f in F)
    Fx = physics.viscous_flux(NS, w, (z, z, z), (np.array(s), z, z), 0)
    assert float(Fx[2]) == pytest.approx(1e-3 * s) and float(Fx[1]) == 0.0
    Fx = physics.viscous_flux(NS, w, (np.array(s), z, z), (z, z, z), 0)
    Fy = physics.viscous_flux(NS, w, (np.array(s), z, z), (z, z, z), 1)
    assert float(Fx[1]) == pytest.approx(4 / 3 * 1e-3 * s)
    assert float(Fy[2]) == pytest.approx(-2 / 3 * 1e-3 * s)
    # heat flux: lambda_T = c_p mu / Pr with c_p = 1/(gamma-1) (eps=1)
    Fx = physics.viscous_flux(NS, w, (z, z, np.array(1.0)), (z, z, z), 0)
    assert float(Fx[3]) == pytest.approx(2.5 * 1e-3 / 0.72)


def test_grad_vars_example():
    g = GOLD["grad_vars"]
    w = (np.array(1.0), np.array(0.0), np.array(0.0), np.array(1.0 / 0.4))
    out = physics.grad_vars(NS, w)
    np.testing.assert_allclose([float(x) for x in out], g["wgrad"], atol=1e-15)


def test_glf_paper_flux():
    """The paper's eq:Riemann with Lambda = diag(1/eps,1,1,1/eps),
    eps = 1 (R18): consistency f*(w, w) = F(w); the dissipation is exactly
    1/2 (wL - wR) per variable; conservation under the mirror map; advection:
    lambda = |a.n|, i.e. identical to the upwind / LLF flux."""
    EG = physics.Equation("euler", numflux="glf")
    rng = np.random.default_rng(31)
    wL = (1.2, 0.3, -0.2, 2.6)
    wR = (0.9, -0.1, 0.4, 2.2)
    for d in (0, 1):
        fc = physics.glf(EG, wL, wL, d)
        F = physics.flux(EG, wL, d)
        assert all(abs(a - b) < 1e-15 for a, b in zip(fc, F))
        f = physics.glf(EG, wL, wR, d)
        FL, FR = physics.flux(EG, wL, d), physics.flux(EG, wR, d)
        for v in range(4):
            assert f[v] == pytest.approx(0.5 * (FL[v] + FR[v]) + 0.5 * (wL[v] - wR[v]), abs=1e-15)
    ea = physics.Equation("advection", a=(0.7, -0.4), numflux="glf")
    el = physics.Equation("advection", a=(0.7, -0.4))
    for d in (0, 1):
        l, r = (rng.standard_normal(5),), (rng.standard_normal(5),)
        np.testing.assert_allclose(physics.glf(ea, l, r, d)[0], physics.llf(el, l, r, d)[0], rtol=0, atol=1e-15)


def test_glf_free_stream_and_conservation():
    """R1 with the paper's flux: a constant state has a zero residual; the
    quadrature-weighted sum of R1 vanishes (periodic conservation)."""
    from oracle import basis, dgsem
    eq = physics.Equation("euler", numflux="glf")
    d = dgsem.Disc(basis.build_basis(3, "gll"), dgsem.Mesh(2, 3, 4), eq)
    W = np.zeros(d.field_shape())
    for v, x in enumerate([1.1, 0.2, -0.3, 2.4]):
        W[:, :, v] = x
    R = dgsem.rhs1(d, W.reshape(-1))
    assert np.abs(R).max() < 1e-12
    rng = np.random.default_rng(32)
    W2 = (W.reshape(-1) * (1 + 0.05 * rng.uniform(-1, 1, d.n)))
    R2 = dgsem.rhs1(d, W2).reshape(d.mesh.n_elem, 4, -1)
    B = basis.build_basis(3, "gll")
    wq = np.outer(B.w, B.w).reshape(-1)
    for v in range(4):
        tot = np.sum(R2[:, v] * wq)
        assert abs(tot) <= 1e-12 * np.sum(np.abs(R2[:, v]) * wq)


def test_reference_mach_scaling():
    """eq:Euler with reference Mach number eps is the standard Euler
    system (eps = 1) in the variables W~ = T W, T = diag(1, eps, eps, 1), with time
    scaled by 1/eps: F~(T w) = eps T F_eps(w), and with the LLF flux (lambda~ =
    eps lambda_eps) R1_eps(W) = T^-1 R1_1(T W) / eps node by node."""
    from oracle import basis, dgsem
    eps = 0.1
    rng = np.random.default_rng(33)
    e1 = physics.Equation("euler")
    ee = physics.Equation("euler", mach=eps)
    w = (1.1, 0.3, -0.2, 25.0)
    T = (1.0, eps, eps, 1.0)
    wt = tuple(t * x for t, x in zip(T, w))
    for d in (0, 1):
        F1 = physics.flux(e1, wt, d)
        Fe = physics.flux(ee, w, d)
        for v in range(4):
            assert F1[v] == pytest.approx(eps * T[v] * Fe[v], rel=1e-14)
        assert physics.wave_speed(e1, wt, d) == pytest.approx(eps * physics.wave_speed(ee, w, d), rel=1e-14)
    mesh = dgsem.Mesh(2, 3, 3)
    B = basis.build_basis(3, "gll")
    d1, de = dgsem.Disc(B, mesh, e1), dgsem.Disc(B, mesh, ee)
    W = np.zeros(de.field_shape())
    for v, x in enumerate([1.0, 0.5, -0.3, 30.0]):
        W[:, :, v] = x
    W = W * (1 + 0.02 * rng.uniform(-1, 1, W.shape))
    Wt = (W.reshape(mesh.n_elem, 4, -1) * np.array(T)[None, :, None]).reshape(-1)
    R1e = dgsem.rhs1(de, W.reshape(-1)).reshape(mesh.n_elem, 4, -1)
    R11 = dgsem.rhs1(d1, Wt).reshape(mesh.n_elem, 4, -1)
    np.testing.assert_allclose(R1e, R11 / (eps * np.array(T)[None, :, None]), rtol=1e-10,
                               atol=1e-12 * np.abs(R1e).max())


@pytest.mark.parametrize("numflux", ["llf", "glf"])
def test_reference_mach_free_stream(numflux):
    """eps = 0.01: a constant state has a zero residual with either flux."""
    from oracle import basis, dgsem
    eq = physics.Equation("euler", mach=0.01, numflux=numflux)
    d = dgsem.Disc(basis.build_basis(3, "gll"), dgsem.Mesh(2, 3, 4), eq)
    W = np.zeros(d.field_shape())
    for v, x in enumerate([1.1, 0.2, -0.3, 2.4]):
        W[:, :, v] = x
    R = dgsem.rhs1(d, W.reshape(-1))
    assert np.abs(R).max() < 1e-9
