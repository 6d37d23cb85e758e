"""Implicit stage solve: residual G(X), Jacobian-vector products, BJ_ext,
GMRES and Newton (PAPER sec. 3.2 and sec. 4.2).

TEST INFRASTRUCTURE (see oracle/__init__.py).

Extended state X = (W, sigma) is stored as one flat vector of length 2n,
[W | sigma] (same partition for both halves P:630).
c2 := alpha2 dt^2 / 2 throughout.
"""
import math

import numpy as np

from . import ad
from .dgsem import rhs1, rhs1_abs, rhs2, rhs12, Disc

EPS_MACH = 2.0 ** -52            # Fortran epsilon(1d0), reading R7


def split(X, n):
    return X[:n], X[n:]


# ---------------------------------------------------------------------------
# residual  (eq:Newton_Residual P:137-141; extended form P:236-239 as read in
# DESIGN.md R4: G1 = g(W) - b, G2 = sigma - R1(W))

def residual(disc: Disc, a1, a2, dt, b, W, sig):
    c2 = a2 * dt * dt / 2.0
    R1, R2 = rhs12(disc, W, sig)
    G1 = W - a1 * dt * R1 + c2 * R2 - b
    G2 = sig - R1
    return G1, G2


# ---------------------------------------------------------------------------
# Jacobian-vector products

def jvp_exact(disc, a1, a2, dt, W, sig, dW, dsig):
    """J dX with the exact blocks of eq:nonlinear_eqsys:
        top = dW - a1 dt dR1/dW dW + c2 dR2/dW dW + c2 dR2/dsigma dsigma
        bot = -dR1/dW dW + dsigma
    dR1/dW dW  = d2-part of R1(W + e1 sigma + e2 dW)
    dR2/dW dW  = d12-part (the Hessian term)
    dR2/dsigma dsigma = R2(W, dsigma)   (R2 is linear in sigma)."""
    c2 = a2 * dt * dt / 2.0
    J = rhs1(disc, ad.Jet(np.asarray(W, float), np.asarray(sig, float),
                          np.asarray(dW, float), 0.0))
    KdW = np.broadcast_to(J.d2, np.shape(W))
    HdW = np.broadcast_to(J.d12, np.shape(W))
    R2ds = rhs2(disc, W, dsig)
    top = dW - a1 * dt * KdW + c2 * HdW + c2 * R2ds
    bot = -KdW + dsig
    return top, bot


def fd_eps(dv, mach=1.0, eps_machine=EPS_MACH):
    """eps_FD = sqrt(eps_machine) / (eps ||dv||_2); None if
    ||dv|| = 0 (the quotient is then defined as 0)."""
    nrm = float(np.linalg.norm(dv))
    return None if nrm == 0.0 else math.sqrt(eps_machine) / (mach * nrm)


def jvp_fd(disc, a1, a2, dt, W, sig, dW, dsig, eps_override=None,
           sigma_literal=False, mach=None):
    """Matrix-free FD product eq:MatrixFree_nonlinear.
    sigma direction: R2(W, dsigma) exactly (reading R8) unless
    sigma_literal, which uses (R2(W, sig + eps dsig) - R2(W, sig)) / eps."""
    c2 = a2 * dt * dt / 2.0
    if mach is None:                 # the reference Mach number of the equation
        mach = getattr(disc.eq, "mach", 1.0)
    if eps_override is not None:
        ew, es = eps_override
    else:
        ew, es = fd_eps(dW, mach), fd_eps(dsig, mach)
    R1, R2 = rhs12(disc, W, sig)
    if ew is None:
        q1 = np.zeros_like(W)
        q2 = np.zeros_like(W)
    else:
        R1p, R2p = rhs12(disc, W + ew * dW, sig)
        q1 = (R1p - R1) / ew
        q2 = (R2p - R2) / ew
    if sigma_literal:
        q3 = np.zeros_like(W) if es is None else (rhs2(disc, W, sig + es * dsig) - R2) / es
    else:
        q3 = rhs2(disc, W, dsig)
    top = dW - a1 * dt * q1 + c2 * q2 + c2 * q3
    bot = -q1 + dsig
    return top, bot


def jvp_linear(disc, a1, a2, dt, dW, dsig):
    """eq:MatrixFree_linear, for linear fluxes (advection)."""
    c2 = a2 * dt * dt / 2.0
    r1w = rhs1(disc, dW)
    r1s = rhs1(disc, dsig)
    return dW - a1 * dt * r1w + c2 * r1s, -r1w + dsig


def jvp(disc, mode, a1, a2, dt, W, sig, dW, dsig, **kw):
    if mode == "linear":
        return jvp_linear(disc, a1, a2, dt, dW, dsig)
    if mode == "exact":
        return jvp_exact(disc, a1, a2, dt, W, sig, dW, dsig)
    if mode == "fd":
        return jvp_fd(disc, a1, a2, dt, W, sig, dW, dsig, **kw)
    raise ValueError(mode)


def default_jvp_mode(disc):
    """AUTO: linear product for advection, FD otherwise."""
    return "linear" if disc.eq.kind == "advection" else "fd"


# ---------------------------------------------------------------------------
# BJ_ext preconditioner (application)

def _period(n, radius):
    for P in range(radius + 1, n + 1):
        if n % P == 0:
            return P
    return n


def element_jacobians(disc: Disc, W):
    """K_i = element-diagonal block dR1_i/dW_i of every element, (nE, m, m).

    Column c of K_i is the dual part of R1 restricted to element i for the
    seed e_c placed in element i only ("element-internal influence only",
    P:271).  Elements of one colour class carry the seed simultaneously; the
    colouring period exceeds the stencil radius (1 for advection/Euler, 2 for
    NS-BR1), so no two seeded elements influence each other."""
    me = disc.mesh
    nE, m = me.n_elem, disc.m
    radius = 2 if disc.eq.viscous else 1
    Px = _period(me.nx, radius)
    Py = _period(me.ny, radius) if me.dim >= 2 else 1
    Pz = _period(me.nz, radius) if me.dim == 3 else 1
    ex = np.arange(nE) % me.nx
    ey = (np.arange(nE) // me.nx) % (me.ny if me.dim >= 2 else 1)
    ez = np.arange(nE) // (me.nx * (me.ny if me.dim >= 2 else 1))
    K = np.zeros((nE, m, m))
    W = np.asarray(W, float)
    for cz in range(Pz):
      for cy in range(Py):
        for cx in range(Px):
            sel = (ex % Px == cx) & (ey % Py == cy) & (ez % Pz == cz)
            for c in range(m):
                seed = np.zeros((nE, m))
                seed[sel, c] = 1.0
                R = rhs2(disc, W, seed.reshape(-1)).reshape(nE, m)
                K[sel, :, c] = R[sel, :]
    return K


class BJExt:
    """S_i = (I - a1 dt K_i + c2 K_i^2)^-1 by LU with partial pivoting
    (P:296), plus the literal D, E, F, G blocks."""

    def __init__(self, disc, W, a1, a2, dt, K=None):
        self.disc, self.a1, self.a2, self.dt = disc, a1, a2, dt
        self.c2 = a2 * dt * dt / 2.0
        self.K = element_jacobians(disc, W) if K is None else K
        m = disc.m
        I = np.eye(m)
        A = I[None] - a1 * dt * self.K                  # A_i (BJ_ext)
        B = self.c2 * self.K                            # B_i
        C = -self.K                                     # C_i
        self.A, self.B, self.C = A, B, C
        self.M = A - B @ C                              # I - a1 dt K + c2 K^2
        self.S = np.linalg.inv(self.M)                  # LAPACK getrf/getri
        self.D = self.S
        self.E = -B @ self.S
        self.F = -C @ self.S
        self.G = A @ self.S

    def apply(self, XW, Xs):
        """P^-1 X per element: (D W + E s ; F W + G s)."""
        nE, m = self.disc.mesh.n_elem, self.disc.m
        w, s = XW.reshape(nE, m, 1), Xs.reshape(nE, m, 1)
        top = (self.D @ w + self.E @ s).reshape(-1)
        bot = (self.F @ w + self.G @ s).reshape(-1)
        return top, bot

    def apply_sk(self, XW, Xs):
        """Equivalent S+K form: u = S W, v = S s;
        top = u - c2 K v;  bot = v + K (u - a1 dt v)."""
        nE, m = self.disc.mesh.n_elem, self.disc.m
        w, s = XW.reshape(nE, m, 1), Xs.reshape(nE, m, 1)
        u, v = self.S @ w, self.S @ s
        top = u - self.c2 * (self.K @ v)
        bot = v + self.K @ (u - self.a1 * self.dt * v)
        return top.reshape(-1), bot.reshape(-1)


def element_hessian_blocks(disc: Disc, W, sig):
    """H_i = element-diagonal block dR2_i/dW_i at fixed sigma (the Hessian
    contribution of BJ^H_ext), (nE, m, m).

    R2(W, sigma) is the e1 part of R1(W + e1 sigma); column c of H_i is the
    e1e2 part of R1(W + e1 sigma + e2 seed) restricted to element i, with the
    seed e_c in element i only (sigma everywhere, "element-internal influence
    only") -- the hyper-dual product used by jvp_exact.  Same colouring
    as element_jacobians (R2 has the stencil of R1)."""
    me = disc.mesh
    nE, m = me.n_elem, disc.m
    radius = 2 if disc.eq.viscous else 1
    Px = _period(me.nx, radius)
    Py = _period(me.ny, radius) if me.dim >= 2 else 1
    Pz = _period(me.nz, radius) if me.dim == 3 else 1
    ex = np.arange(nE) % me.nx
    ey = (np.arange(nE) // me.nx) % (me.ny if me.dim >= 2 else 1)
    ez = np.arange(nE) // (me.nx * (me.ny if me.dim >= 2 else 1))
    H = np.zeros((nE, m, m))
    W = np.asarray(W, float)
    sig = np.asarray(sig, float)
    for cz in range(Pz):
      for cy in range(Py):
        for cx in range(Px):
            sel = (ex % Px == cx) & (ey % Py == cy) & (ez % Pz == cz)
            for c in range(m):
                seed = np.zeros((nE, m))
                seed[sel, c] = 1.0
                J = rhs1(disc, ad.Jet(W, sig, seed.reshape(-1), 0.0))
                R = np.broadcast_to(J.d12, W.shape).reshape(nE, m)
                H[sel, :, c] = R[sel, :]
    return H


class BJExtH:
    """BJ^H_ext: the extended block-Jacobi preconditioner WITH the
    Hessian contribution,
        A^H_i = I - a1 dt K_i + c2 H_i,   B_i = c2 K_i,   C_i = -K_i,
        D^H = (A^H - B C)^-1,  E^H = -(A^H - B C)^-1 B,
        F^H = -C (A^H - B C)^-1,  G^H = I + C (A^H - B C)^-1 B,
    one inverse per element by LU.  sigma is the build point's
    sigma (the library builds at X = (W, R1(W)), reading R31)."""

    def __init__(self, disc, W, sig, a1, a2, dt, K=None, H=None):
        self.disc, self.a1, self.a2, self.dt = disc, a1, a2, dt
        self.c2 = a2 * dt * dt / 2.0
        self.K = element_jacobians(disc, W) if K is None else K
        self.H = element_hessian_blocks(disc, W, sig) if H is None else H
        m = disc.m
        I = np.eye(m)
        A = I[None] - a1 * dt * self.K + self.c2 * self.H     # A^H_i
        B = self.c2 * self.K                                  # B_i
        C = -self.K                                           # C_i
        self.A, self.B, self.C = A, B, C
        self.M = A - B @ C                                    # I - a1 dt K + c2 (H + K^2)
        self.S = np.linalg.inv(self.M)                        # LAPACK getrf/getri
        self.D = self.S
        self.E = -self.S @ B
        self.F = -C @ self.S
        self.G = I[None] + C @ self.S @ B

    def apply(self, XW, Xs):
        """P^-1 X per element: (D x + E y ; F x + G y)."""
        nE, m = self.disc.mesh.n_elem, self.disc.m
        w, s = XW.reshape(nE, m, 1), Xs.reshape(nE, m, 1)
        top = (self.D @ w + self.E @ s).reshape(-1)
        bot = (self.F @ w + self.G @ s).reshape(-1)
        return top, bot

    def apply_sk(self, XW, Xs):
        """Equivalent S+K form: u = S (x - c2 K y);  top = u;  bot = y + K u."""
        nE, m = self.disc.mesh.n_elem, self.disc.m
        w, s = XW.reshape(nE, m, 1), Xs.reshape(nE, m, 1)
        u = self.S @ (w - self.c2 * (self.K @ s))
        bot = s + self.K @ u
        return u.reshape(-1), bot.reshape(-1)


def make_precond(kind, disc, W, a1, a2, dt):
    """'bjext' or 'bjext_h' (sigma = R1(W))."""
    if kind == "bjext":
        return BJExt(disc, W, a1, a2, dt)
    if kind == "bjext_h":
        return BJExtH(disc, W, rhs1(disc, W), a1, a2, dt)
    raise ValueError(kind)


# ---------------------------------------------------------------------------
# GMRES (right preconditioned, modified Gram-Schmidt, restarted)

STAGNATION = 0.9          # a restart cycle must reduce the true residual below 0.9x its start (R34)


def gmres(matvec, rhs, precond=None, rtol=1e-6, restart=50, max_total=7000):
    """Solve A x = rhs with x0 = 0 by restarted GMRES on A P^-1 y = rhs,
    x = P^-1 y (right preconditioning).  Converged when the Arnoldi
    residual estimate <= rtol ||rhs||.  Returns (x, iterations, converged).

    Stagnation (reading R34): with restarts, every cycle starts from
    the true residual rhs - A x, which an FD JVP only resolves down
    to its own truncation/rounding level.  A cycle that lowers the true
    residual by less than 10 % (||r_new|| > 0.9 ||r_cycle_start||) ends the
    solve as converged-as-far-as-possible: x is returned to Newton, whose outer
    iteration re-evaluates G and continues (inexact Newton)."""
    Pinv = precond if precond is not None else (lambda v: v)
    x = np.zeros_like(rhs)
    beta0 = float(np.linalg.norm(rhs))
    if beta0 == 0.0:
        return x, 0, True
    total = 0
    r = rhs.copy()
    converged = False
    beta_start = None
    while True:
        beta = float(np.linalg.norm(r))
        if beta <= rtol * beta0:
            converged = True
            break
        if beta_start is not None and beta > STAGNATION * beta_start:
            converged = True                           # stagnated at the operator's noise level (R34)
            break
        if total >= max_total:
            break
        beta_start = beta
        V = [r / beta]
        H = np.zeros((restart + 1, restart))
        cs, sn = np.zeros(restart), np.zeros(restart)
        g = np.zeros(restart + 1)
        g[0] = beta
        k = 0
        for j in range(restart):
            w = matvec(Pinv(V[j]))
            for i in range(j + 1):                     # modified Gram-Schmidt
                H[i, j] = float(np.dot(w, V[i]))
                w = w - H[i, j] * V[i]
            H[j + 1, j] = float(np.linalg.norm(w))
            for i in range(j):                         # previous rotations
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = math.hypot(H[j, j], H[j + 1, j])
            cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            total += 1
            k = j + 1
            hnext = float(np.linalg.norm(w))
            if abs(g[j + 1]) <= rtol * beta0 or total >= max_total or hnext == 0.0:
                break
            V.append(w / hnext)
        y = np.zeros(k)
        for i in range(k - 1, -1, -1):                 # back substitution
            y[i] = (g[i] - np.dot(H[i, i + 1:k], y[i + 1:k])) / H[i, i]
        x = x + Pinv(sum(y[i] * V[i] for i in range(k)))
        r = rhs - matvec(x)                            # true residual
        if abs(g[k]) <= rtol * beta0:
            converged = True
            break
    return x, total, converged


# ---------------------------------------------------------------------------
# Newton on the extended system (eq:Newton)

class NewtonOpts:
    def __init__(self, rtol=1e-10, atol_dw=1e-12, max_newton=50, gmres_rtol=1e-6,
                 restart=700, max_krylov=7000, precond="bjext",
                 precond_policy="per_step_per_alpha", jvp_mode="auto", schur=False):
        self.rtol, self.atol_dw, self.max_newton = rtol, atol_dw, max_newton
        self.gmres_rtol, self.restart, self.max_krylov = gmres_rtol, restart, max_krylov
        self.precond, self.precond_policy, self.jvp_mode = precond, precond_policy, jvp_mode
        self.schur = schur           # solve the Schur complement system instead of eq:Newton


class NewtonFailure(RuntimeError):
    pass


def newton_solve(disc, a1, a2, dt, b, W_guess, opts: NewtonOpts, pc=None, stats=None):
    """Solve G(X) = 0 from X0 = (W_g, R1(W_g)).  Stops when
    ||G(X^r)|| <= max(rtol ||G(X^0)||, 64 eps ||b||) or after a step with
    ||dW|| <= atol_dw (reading R10).  The floor also
    covers the rounding level of the sigma block sigma - R1(W), which cannot
    be evaluated below ~eps ||R1_abs|| (R1 with |Dhat|, |F|, |f*|): the
    reason P:924 gives for adding an absolute criterion (reading R10b):
        floor = max(64 eps ||b||, 4 eps ||R1_abs(W_g)||)."""
    n = disc.n
    mode = default_jvp_mode(disc) if opts.jvp_mode == "auto" else opts.jvp_mode
    W = np.array(W_guess, float)
    sig = rhs1(disc, W)
    floor = max(64.0 * EPS_MACH * float(np.linalg.norm(b)),
                4.0 * EPS_MACH * float(np.linalg.norm(rhs1_abs(disc, W))))
    g0 = None
    for r in range(opts.max_newton + 1):
        G1, G2 = residual(disc, a1, a2, dt, b, W, sig)
        gn = float(np.sqrt(np.dot(G1, G1) + np.dot(G2, G2)))
        if g0 is None:
            g0 = gn
        if gn <= max(opts.rtol * g0, floor):
            break
        if r == opts.max_newton:
            raise NewtonFailure(f"Newton did not converge: ||G||={gn:.3e}, ||G0||={g0:.3e}")
        if opts.precond in ("bjext", "bjext_h") and opts.precond_policy == "per_newton":
            pc = make_precond(opts.precond, disc, W, a1, a2, dt)
            if stats is not None:
                stats["precond_builds"] += 1
        Wc, sc = W.copy(), sig.copy()
        if opts.schur:
            # Schur complement: J_S dw = -G1 + c2 dR2/dsigma G2, dsigma = -G2 + dR1/dW dw,
            # J_S = I - a1 dt K + c2 dR2/dW + c2 K^2 (eq:nonlinear_eqsys_Schur) applied matrix-free as
            # the top block of J (v, K v); K v = dR1/dW v = R2(W, v) exactly (R2 linear in sigma)
            c2 = a2 * dt * dt / 2.0
            Kv = lambda v: rhs2(disc, Wc, v)

            def matvec_s(v):
                return jvp(disc, mode, a1, a2, dt, Wc, sc, v, Kv(v))[0]

            precond_s = None
            if pc is not None:       # element-block Jacobi of J_S: the D block of BJ_ext / BJ^H_ext (reading R32)
                precond_s = lambda v: (pc.S @ v.reshape(-1, disc.m, 1)).reshape(-1)
            dw, its, ok = gmres(matvec_s, -G1 + c2 * Kv(G2), precond_s,
                                opts.gmres_rtol, opts.restart, opts.max_krylov)
            dX = np.concatenate([dw, -G2 + Kv(dw)])
        else:
            def matvec(v):
                t, bt = jvp(disc, mode, a1, a2, dt, Wc, sc, v[:n], v[n:])
                return np.concatenate([t, bt])

            precond = None
            if pc is not None:
                precond = lambda v: np.concatenate(pc.apply(v[:n], v[n:]))
            dX, its, ok = gmres(matvec, -np.concatenate([G1, G2]), precond,
                                opts.gmres_rtol, opts.restart, opts.max_krylov)
        if stats is not None:
            stats["gmres_its"] += its
            stats["newton_its"] += 1
        if not ok:
            raise NewtonFailure(f"GMRES did not converge in {its} iterations")
        W = W + dX[:n]
        sig = sig + dX[n:]
        if float(np.linalg.norm(dX[:n])) <= opts.atol_dw:
            break
    return W, sig
