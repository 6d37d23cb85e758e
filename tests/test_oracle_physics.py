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


def test_glf_paper_flux_worked_example():
    """S:159, the paper's eq:Riemann with lambda = |a.n|:
    a = (0.3, 0.3), n = (1, 0), wL = 1, wR = 0 -> 1/2 (0.3 + 0) + 0.3 (1 - 0) = 0.45
    (golden fstar_glf_paper).  LLF / upwind gives 0.30 on the same data."""
    u = GOLD["llf_upwind"]
    eq = physics.Equation("advection", a=tuple(u["a"]), numflux="glf")
    f = physics.glf(eq, (np.array(u["wL"]),), (np.array(u["wR"]),), 0)[0]
    assert float(f) == pytest.approx(u["fstar_glf_paper"], abs=1e-15)
    assert float(physics.numerical_flux(eq, (np.array(u["wL"]),), (np.array(u["wR"]),), 0)[0]) \
        == pytest.approx(0.45, abs=1e-15)
    # the y-direction and a negative velocity component: lambda = |a_d|
    eq2 = physics.Equation("advection", a=(0.3, -0.5), numflux="glf")
    f = physics.glf(eq2, (np.array(2.0),), (np.array(1.0),), 1)[0]
    assert float(f) == pytest.approx(0.5 * (-1.0 - 0.5) + 0.5 * (2.0 - 1.0), abs=1e-15)   # -0.25


def test_glf_paper_flux_euler_hand_values():
    """eq:Riemann with Lambda = diag(1/eps, 1, 1, 1/eps), values worked by
    hand (gamma = 1.4).  wL = (1, 0, 0, 2.5) (rho = 1, v = 0, p = 1),
    wR = (0.5, 0, 0, 1.25) (rho = 0.5, v = 0, p = 0.5), normal e_x:
    F_x(wL) = (0, 1, 0, 0), F_x(wR) = (0, 0.5, 0, 0);
    eps = 1:   f* = (0 + 0.5, 0.75 + 0, 0, 0 + 1.25) = (0.5, 0.75, 0, 1.25);
    eps = 0.1 (density and energy jumps x10): momentum flux p/eps^2 = 100 p, so
               f* = (0 + 10 * 0.5, 0.5 (100 + 50) + 0, 0, 0 + 10 * 1.25) = (5, 75, 0, 12.5)."""
    wL = (1.0, 0.0, 0.0, 2.5)
    wR = (0.5, 0.0, 0.0, 1.25)
    e1 = physics.Equation("euler", numflux="glf")
    np.testing.assert_allclose(physics.glf(e1, wL, wR, 0), (0.5, 0.75, 0.0, 1.25), rtol=0, atol=1e-15)
    # at eps = 0.1 the same primitive states have E = p/(gamma-1) + eps^2 rho |v|^2 / 2 = same E
    e01 = physics.Equation("euler", numflux="glf", mach=0.1)
    np.testing.assert_allclose(physics.glf(e01, wL, wR, 0), (5.0, 75.0, 0.0, 12.5), rtol=1e-15, atol=1e-13)
    # a momentum jump is not scaled by 1/eps: (1, 0.2, 0, 2.5) vs (1, 0, 0, 2.5) at eps = 0.1
    wa = (1.0, 0.2, 0.0, 2.5 + 0.5 * 0.01 * 0.04)      # p = 1 exactly: E = p/0.4 + eps^2 rho u^2/2
    wb = (1.0, 0.0, 0.0, 2.5)
    f = physics.glf(e01, wa, wb, 0)
    # F_x(wa) = (0.2, 0.04 + 100, 0, 0.2 (E_a + 1)), F_x(wb) = (0, 100, 0, 0)
    Ea = wa[3]
    expect = (0.1 + 10 * 0.0, 0.5 * (100.04 + 100.0) + 0.2, 0.0, 0.1 * (Ea + 1.0) + 10 * (Ea - 2.5))
    np.testing.assert_allclose(f, expect, rtol=1e-14, atol=1e-14)
    # consistency f*(w, w) = F(w) and the mirror conservation
    rng = np.random.default_rng(31)
    a, b = _rand_states(rng, 20), _rand_states(rng, 20)
    for d in (0, 1):
        for x, y in zip(physics.glf(e1, a, a, d), physics.flux(e1, a, d)):
            np.testing.assert_allclose(x, y, rtol=1e-15, atol=1e-15)
        fl = physics.glf(e1, a, b, d)
        mir = lambda w: tuple(-x if k == 1 + d else x for k, x in enumerate(w))
        fr = physics.glf(e1, mir(b), mir(a), d)
        for k in range(4):
            sgn = 1.0 if k == 1 + d else -1.0
            np.testing.assert_allclose(fl[k], sgn * fr[k], rtol=1e-13, atol=1e-13)


def test_euler_flux_moving_state_hand_values():
    """eq:Euler at a state with non-zero velocity, worked by hand
    (gamma = 1.4, eps = 1; every number is a binary fraction, so exact):
    w = (2, 1, -0.5, 5): u = 0.5, v = -0.25, rho|v|^2/2 = 0.3125,
    p = 0.4 (5 - 0.3125) = 1.875, E + p = 6.875;
    F_x = (rho u, rho u^2 + p, rho u v, u (E + p)) = (1, 2.375, -0.25, 3.4375)
    F_y = (rho v, rho u v, rho v^2 + p, v (E + p)) = (-0.5, -0.25, 2.0, -1.71875).
    At eps = 0.5 (p = 0.4 (5 - 0.25 * 0.3125) = 1.96875; momentum p/eps^2 = 7.875):
    F_x = (1, 0.5 + 7.875, -0.25, 0.5 (5 + 1.96875)) = (1, 8.375, -0.25, 3.484375)."""
    w = (2.0, 1.0, -0.5, 5.0)
    ap = lambda a, b: np.testing.assert_allclose(a, b, rtol=4e-16, atol=4e-16)   # gamma-1 = 0.4 rounds
    ap(physics.pressure(EU, w), 1.875)
    ap(physics.flux(EU, w, 0), (1.0, 2.375, -0.25, 3.4375))
    ap(physics.flux(EU, w, 1), (-0.5, -0.25, 2.0, -1.71875))
    e05 = physics.Equation("euler", mach=0.5)
    ap(physics.pressure(e05, w), 1.96875)
    ap(physics.flux(e05, w, 0), (1.0, 8.375, -0.25, 3.484375))


def test_wave_speed_and_llf_hand_values():
    """LLF wave speed lambda_f = max(|v_L.n| + c_L, |v_R.n| + c_R), c = sqrt(gamma p / rho)
    (reading R3), at states chosen so that c is exact (gamma = 1.4):
    wL: rho = 1, u = 0.5, v = -0.25, p = 1.4 -> c = sqrt(1.96) = 1.4,
        E = 1.4/0.4 + 0.3125/2 = 3.65625; speeds: x 1.9, y 1.65.
    wR: rho = 4, u = -1, v = 0, p = 0.7 -> c = sqrt(0.245) = 0.494974746830583...,
        E = 1.75 + 2 = 3.75; speeds: x 1 + c, y c.
    x face: lambda_f = 1.9 (L);  y face: lambda_f = 1.65 (L).
    At eps = 0.5 the sound speed is c/eps (P:395 scaling): wL x speed 0.5 + 2.8 = 3.3."""
    wL = (1.0, 0.5, -0.25, 3.65625)
    wR = (4.0, -4.0, 0.0, 3.75)
    assert physics.pressure(EU, wL) == pytest.approx(1.4, abs=1e-15)
    assert physics.wave_speed(EU, wL, 0) == pytest.approx(1.9, abs=1e-15)
    assert physics.wave_speed(EU, wL, 1) == pytest.approx(1.65, abs=1e-15)
    assert physics.wave_speed(EU, wR, 0) == pytest.approx(1.0 + math.sqrt(0.245), abs=1e-15)
    assert physics.wave_speed(EU, wR, 1) == pytest.approx(math.sqrt(0.245), abs=1e-15)
    # LLF value on the x face: 1/2 (F_L + F_R) + 1/2 * 1.9 (wL - wR), by hand:
    # F_x(wL) = (0.5, 0.25 + 1.4, -0.125, 0.5 (3.65625 + 1.4)) = (0.5, 1.65, -0.125, 2.528125)
    # F_x(wR) = (-4, 4 + 0.7, 0, -1 (3.75 + 0.7)) = (-4, 4.7, 0, -4.45)
    f = physics.llf(EU, wL, wR, 0)
    FL = (0.5, 1.65, -0.125, 2.528125)
    FR = (-4.0, 4.7, 0.0, -4.45)
    expect = tuple(0.5 * (a + b) + 0.95 * (l - r) for a, b, l, r in zip(FL, FR, wL, wR))
    np.testing.assert_allclose(f, expect, rtol=1e-14, atol=1e-14)
    e05 = physics.Equation("euler", mach=0.5)
    wL05 = (1.0, 0.5, -0.25, 1.4 / 0.4 + 0.25 * 0.3125 / 2)     # p = 1.4 at eps = 0.5
    assert physics.wave_speed(e05, wL05, 0) == pytest.approx(0.5 + 2.8, abs=1e-14)


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
