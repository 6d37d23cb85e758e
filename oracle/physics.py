"""Point-wise physics: fluxes, numerical flux, viscous flux, gradient variables.

TEST INFRASTRUCTURE (see oracle/__init__.py).

States are tuples of per-variable components (numpy arrays or ad.Jet), so
every function here is evaluated unchanged on plain values, duals and
hyper-duals.

  advection     F = a w                                   (C1/C2)
  euler         F_x = (rho u, rho u^2 + p, rho u v, u (E + p))      (eq:Euler,
                p = (gamma-1)(E - rho |v|^2 / 2)                     P:388-394)
                in 2D (4 variables) and 3D (5 variables: (rho, rho u, rho v,
                rho w, E), the same system with a third momentum component --
                the paper's 3D Taylor-Green case; NEXT-4)
                and the reference Mach number eps of eq:Euler: momentum flux
                rho v v + p / eps^2, p = (gamma-1)(E - eps^2 rho |v|^2 / 2)
                (configs: eps = 1, reading R18; NS only at eps = 1)
  navier_stokes F - F^v, F^v = (0, tau, tau.v + q), tau = mu(grad v +
                grad v^T - 2/3 div v I), q = lambda_T grad T, lambda_T = c_p mu/Pr,
                c_p = R gamma/(gamma-1), R = 1/gamma, T = p/(rho R)

Numerical flux (reading R3): the paper's
eq:Riemann is a global Lax-Friedrichs flux with a constant lambda; the
BASELINE configs name LLF/Rusanov, so the configs use
    f*(wL, wR; e_d) = 1/2 (F_d(wL) + F_d(wR)) + 1/2 lambda_f (wL - wR),
    lambda_f = max(|v_L.e_d| + c_L, |v_R.e_d| + c_R),
evaluated in the canonical orientation of a face (L = the element on the
-e_d side, normal +e_d); ties take L, sign(0) = +1.  For advection
lambda_f = |a_d| and f* is the exact upwind flux.  numflux = "glf" is the
paper's eq:Riemann literally:
    f*(wL, wR; e_d) = 1/2 (F_d(wL) + F_d(wR)) + Lambda (wL - wR),
Lambda = |a_d| (advection) or diag(1/eps, 1, 1, 1/eps) (Euler / NS), no 1/2
on the jump term (0.45 for a = (0.3, 0.3), wL = 1, wR = 0).
"""
from dataclasses import dataclass

from . import ad


@dataclass(frozen=True)
class Equation:
    kind: str                  # "advection" | "euler" | "navier_stokes"
    a: tuple = (1.0, 1.0)      # advection velocity (3D: three components)
    gamma: float = 1.4
    mu: float = 0.0
    prandtl: float = 0.72
    numflux: str = "llf"       # "llf" (configs, reading R3) | "glf" (the paper's eq:Riemann)
    mach: float = 1.0          # reference Mach number eps of eq:Euler; configs: 1 (R18)
    lifting: str = "br1"       # NS face gradients: "br1" (C5, reading R19) | "br2" (R33)
    eta_br2: float = 2.0       # BR2 stabilisation parameter (the paper gives no value; reading R33)
    dim: int = 2               # space dimension of the Euler system (3: five variables, NEXT-4)

    @property
    def nv(self):
        return 1 if self.kind == "advection" else (5 if self.dim == 3 else 4)

    @property
    def viscous(self):
        return self.kind == "navier_stokes"


def pressure(eq, w):
    """p = (gamma - 1)(E - eps^2/2 rho |v|^2); w = (rho, rho v, E)
    with 2 (2D) or 3 (3D) momentum components."""
    rho, E = w[0], w[-1]
    e2 = eq.mach * eq.mach
    ke = w[1] * w[1]
    for m in w[2:-1]:
        ke = ke + m * m
    return (eq.gamma - 1.0) * (E - 0.5 * e2 * ke / rho)


def flux(eq, w, d):
    """Inviscid physical flux F_d(w) in direction d (0 = x, 1 = y, 2 = z)."""
    if eq.kind == "advection":
        return (eq.a[d] * w[0],)
    rho, E = w[0], w[-1]
    mom = w[1:-1]
    p = pressure(eq, w)
    pe = p / (eq.mach * eq.mach)             # p / eps^2 in the momentum flux (eq:Euler)
    vn = mom[d] / rho
    return ((rho * vn,)
            + tuple(mk * vn + (pe if k == d else 0.0) for k, mk in enumerate(mom))
            + (vn * (E + p),))


def wave_speed(eq, w, d):
    """|v.e_d| + c (Euler/NS), |a_d| (advection)."""
    if eq.kind == "advection":
        return abs(eq.a[d]) + 0.0 * w[0]
    rho = w[0]
    p = pressure(eq, w)
    vn = w[1 + d] / rho
    return ad.absval(vn) + ad.sqrt(eq.gamma * p / rho) / eq.mach   # eigenvalues v.n +- c / eps


def llf(eq, wL, wR, d):
    """Canonical-orientation LLF flux across a face with normal +e_d."""
    FL, FR = flux(eq, wL, d), flux(eq, wR, d)
    lam = ad.maxval(wave_speed(eq, wL, d), wave_speed(eq, wR, d))
    return tuple(0.5 * (fl + fr) + 0.5 * lam * (l - r)
                 for fl, fr, l, r in zip(FL, FR, wL, wR))


def glf(eq, wL, wR, d):
    """The paper's numerical flux eq:Riemann: global Lax-Friedrichs
    with a constant dissipation matrix, lambda = |a.n| for advection and
    Lambda = diag(1/eps, 1, 1, 1/eps) for Euler / NS, eps the reference
    Mach number (configs: eps = 1, reading R18).  Canonical orientation."""
    FL, FR = flux(eq, wL, d), flux(eq, wR, d)
    if eq.kind == "advection":
        lam = (abs(eq.a[d]),)
    else:
        eps = eq.mach
        lam = (1.0 / eps,) + (1.0,) * (len(wL) - 2) + (1.0 / eps,)
    # eq:Riemann: (1/2 (F_L + F_R) + lambda (w_L - w_R)) . n -- the jump term
    # carries the full lambda, no 1/2 (S:159 gives 0.45 for its example),
    # and is not projected on n.
    return tuple(0.5 * (fl + fr) + lv * (l - r)
                 for fl, fr, l, r, lv in zip(FL, FR, wL, wR, lam))


def numerical_flux(eq, wL, wR, d):
    """f*(wL, wR; e_d) of the equation's choice (LLF or the paper's GLF)."""
    return glf(eq, wL, wR, d) if eq.numflux == "glf" else llf(eq, wL, wR, d)


# ---- Navier-Stokes --------------------------------------------------------

def gas_constants(eq):
    R = 1.0 / eq.gamma                      # R = 1/(gamma eps^2), eps = 1
    cp = R * eq.gamma / (eq.gamma - 1.0)
    lam_T = cp * eq.mu / eq.prandtl
    return R, cp, lam_T


def grad_vars(eq, w):
    """w_grad = (v1, v2, T) (eq:LiftingEq), T from p = rho R T."""
    rho, mx, my, E = w
    R, _, _ = gas_constants(eq)
    p = pressure(eq, w)
    return (mx / rho, my / rho, p / (rho * R))


def viscous_flux(eq, w, gx, gy, d):
    """F^v_d(w, grad) with gx = (u_x, v_x, T_x), gy = (u_y, v_y, T_y)."""
    rho, mx, my, E = w
    u, v = mx / rho, my / rho
    _, _, lam_T = gas_constants(eq)
    ux, vx, Tx = gx
    uy, vy, Ty = gy
    div = ux + vy
    mu = eq.mu
    if d == 0:
        txx = mu * (2.0 * ux - (2.0 / 3.0) * div)
        txy = mu * (uy + vx)
        return (0.0 * rho, txx, txy, txx * u + txy * v + lam_T * Tx)
    tyx = mu * (uy + vx)
    tyy = mu * (2.0 * vy - (2.0 / 3.0) * div)
    return (0.0 * rho, tyx, tyy, tyx * u + tyy * v + lam_T * Ty)
