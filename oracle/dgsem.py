"""DGSEM spatial operators R^(1)_h and R^(2)_h on periodic Cartesian meshes.

TEST INFRASTRUCTURE (see oracle/__init__.py).

Layout L: a field is a flat fp64 vector indexed
[elem][var][j][i] (i fastest), elem = ey*nx + ex.  Internally it is viewed
as (ny, nx, nv, p, p) in 2D and (nx, nv, p) in 1D.

R^(1)_h follows eq:DGSEM_wt on affine Cartesian elements, where
J_geo = dx dy/4 and s-hat = dy/2 (xi_1 faces), dx/2 (xi_2 faces), so
    R1_ij = -[ (2/dx) ( sum_l Dhat_il Fx_lj + f*_E,j lhat_i(1) - f*_W,j lhat_i(-1) )
             + (2/dy) ( sum_m Dhat_jm Fy_im + f*_N,i lhat_j(1) - f*_S,i lhat_j(-1) ) ].
f*_E/W/N/S are the canonical (normal +e_d) face fluxes; the outward normal
of the element's W and S faces is -e_d, hence the minus signs.  Traces are
the solution polynomial evaluated at xi = +-1: w(+-1) = sum_i l_i(+-1) w_i.

R^(2)_h(W, sigma) is *defined* by differentiating the discrete equations in
time with w_t = sigma (P:211-213 and eq:DGSEM_wtt; NS: P:869-905), i.e. the
directional derivative of R^(1)_h at W in direction sigma.  It is computed
with forward-mode AD (oracle.ad), which reproduces the volume term
(dF/dw) sigma and the linearised face flux f~* of P:226-228 (including the
derivative of the LLF wave speed, reading R3).

Navier-Stokes (C5): BR1 lifting (reading R19; the paper uses BR2,
P:834): d = lifted gradient of w_grad = (u, v, T) from the weak form
eq:Lifting with the central surface value 1/2(g_L + g_R);
face gradients d^L, d^R are the traces of the lifted polynomial.  The
viscous surface flux is 1/2(F^v_L + F^v_R).n.  Equation.lifting =
"br2": the volume keeps d, the face gradients come from the per-face local
lifting of P:865 (lifting_br2_faces, reading R33).
"""
from dataclasses import dataclass

import numpy as np

from . import ad, physics
from .basis import Basis


@dataclass(frozen=True)
class Mesh:
    dim: int
    nx: int
    ny: int = 1
    xmin: float = 0.0
    xmax: float = 1.0
    ymin: float = 0.0
    ymax: float = 1.0
    nz: int = 1                # 3D (NEXT-4): elements and extent in z
    zmin: float = 0.0
    zmax: float = 1.0

    @property
    def dx(self):
        return (self.xmax - self.xmin) / self.nx

    @property
    def dy(self):
        return (self.ymax - self.ymin) / self.ny

    @property
    def dz(self):
        return (self.zmax - self.zmin) / self.nz

    @property
    def n_elem(self):
        return self.nx * (self.ny if self.dim >= 2 else 1) * (self.nz if self.dim == 3 else 1)


@dataclass
class Disc:
    basis: Basis
    mesh: Mesh
    eq: physics.Equation

    @property
    def p(self):
        return self.basis.p

    @property
    def nv(self):
        return self.eq.nv

    @property
    def m(self):
        return self.nv * self.p ** self.mesh.dim

    @property
    def n(self):
        return self.mesh.n_elem * self.m

    def field_shape(self):
        p, nv, me = self.p, self.nv, self.mesh
        if me.dim == 3:
            return (me.nz, me.ny, me.nx, nv, p, p, p)      # [ez][ey][ex][var][k][j][i]
        return (me.ny, me.nx, nv, p, p) if me.dim == 2 else (me.nx, nv, p)

    def to_field(self, x):
        return ad.apply_linear(lambda c: np.reshape(c, self.field_shape()), x)

    def to_flat(self, F):
        return ad.apply_linear(lambda c: np.reshape(c, -1), F)

    def node_coords(self):
        """Physical node coordinates, each of field shape without the var
        axis broadcast: x(ex, i) = xmin + ex dx + (xi_i + 1) dx/2."""
        me, xi = self.mesh, self.basis.xi
        xs = me.xmin + np.arange(me.nx)[:, None] * me.dx + (xi[None, :] + 1.0) * me.dx / 2
        if me.dim == 1:
            return (xs,)                                  # (nx, p)
        ys = me.ymin + np.arange(me.ny)[:, None] * me.dy + (xi[None, :] + 1.0) * me.dy / 2
        if me.dim == 3:
            zs = me.zmin + np.arange(me.nz)[:, None] * me.dz + (xi[None, :] + 1.0) * me.dz / 2
            p = self.p
            sh = (me.nz, me.ny, me.nx, p, p, p)
            X = np.broadcast_to(xs[None, None, :, None, None, :], sh)
            Y = np.broadcast_to(ys[None, :, None, None, :, None], sh)
            Z = np.broadcast_to(zs[:, None, None, :, None, None], sh)
            return (X, Y, Z)                              # (nz, ny, nx, p(k), p(j), p(i))
        X = np.broadcast_to(xs[None, :, None, :], (me.ny, me.nx, self.p, self.p))
        Y = np.broadcast_to(ys[:, None, :, None], (me.ny, me.nx, self.p, self.p))
        return (X, Y)                                     # (ny, nx, p(j), p(i))


# ---------------------------------------------------------------------------
# field helpers (2D axes: 0 ey, 1 ex, 2 var, 3 j, 4 i;  1D: 0 ex, 1 var, 2 i)

def _split(F, var_axis):
    n = F.shape[var_axis]
    idx = [slice(None)] * (var_axis + 1)
    out = []
    for v in range(n):
        idx[var_axis] = v
        out.append(F[tuple(idx)])
    return tuple(out)


def _lin(f, x):
    return ad.apply_linear(f, x)


def _roll(x, shift, axis):
    return _lin(lambda c: np.roll(c, shift, axis=axis), x)


class _Ops:
    """Tensor-product derivative/trace operators of one discretization.
    absolute=True builds the magnitude version used for rounding estimates
    (|Dhat|, |lhat|, and the - face added instead of subtracted)."""

    def __init__(self, disc: Disc, absolute=False):
        b = disc.basis
        self.disc = disc
        self.Dh, self.lp, self.lm = b.Dhat, b.l_plus, b.l_minus
        self.lhp, self.lhm = b.lhat_plus, b.lhat_minus
        if absolute:
            self.Dh, self.lhp, self.lhm = np.abs(self.Dh), np.abs(self.lhp), -np.abs(self.lhm)
        self.dim = disc.mesh.dim

    # traces: polynomial evaluated at the element end
    def trace(self, F, d, side):
        l = self.lp if side > 0 else self.lm
        if self.dim == 3:                # node axis of direction d: -1 - d  ([k][j][i])
            return _lin(lambda c: np.tensordot(c, l, axes=([c.ndim - 1 - d], [0])), F)
        if self.dim == 1:
            return _lin(lambda c: np.einsum("...i,i->...", c, l), F)
        if d == 0:
            return _lin(lambda c: np.einsum("...ji,i->...j", c, l), F)
        return _lin(lambda c: np.einsum("...ji,j->...i", c, l), F)

    def volume(self, F, d):
        """sum_l Dhat_il F_lj (d = 0) or sum_m Dhat_jm F_im (d = 1)."""
        Dh = self.Dh
        if self.dim == 3:                # sum_l Dhat_il F_..l.. along the node axis of d
            def vol3(c):
                ax = c.ndim - 1 - d
                return np.moveaxis(np.tensordot(c, Dh, axes=([ax], [1])), -1, ax)
            return _lin(vol3, F)
        if self.dim == 1:
            return _lin(lambda c: np.einsum("il,...l->...i", Dh, c), F)
        if d == 0:
            return _lin(lambda c: np.einsum("il,...jl->...ji", Dh, c), F)
        return _lin(lambda c: np.einsum("jm,...mi->...ji", Dh, c), F)

    def surface(self, fplus, fminus, d):
        """f+ lhat(1) - f- lhat(-1) spread onto the element nodes; f+/f- are
        canonical (normal +e_d) fluxes on the element's +/- face."""
        hp, hm = self.lhp, self.lhm
        if self.dim == 3:                # face values spread along the node axis of d
            def spread(h):
                def f(c):
                    ax = c.ndim - d          # the inserted axis sits at -1 - d of the result
                    sh = [1] * (c.ndim + 1)
                    sh[ax] = h.size
                    return np.expand_dims(c, ax) * h.reshape(sh)
                return f
            return _lin(spread(hp), fplus) - _lin(spread(hm), fminus)
        if self.dim == 1:
            return _lin(lambda c: c[..., None] * hp, fplus) - _lin(lambda c: c[..., None] * hm, fminus)
        if d == 0:
            return (_lin(lambda c: c[..., :, None] * hp[None, :], fplus)
                    - _lin(lambda c: c[..., :, None] * hm[None, :], fminus))
        return (_lin(lambda c: c[..., None, :] * hp[:, None], fplus)
                - _lin(lambda c: c[..., None, :] * hm[:, None], fminus))

    def elem_axis(self, d):
        """Array axis along which elements neighbour in direction d."""
        if self.dim == 1:
            return 0
        if self.dim == 3:
            return 2 - d                 # (ez, ey, ex)
        return 1 if d == 0 else 0

    def faces(self, F, d):
        """Own traces on the +/- faces and the matching neighbour traces:
        returns (own_plus, nbr_plus, nbr_minus, own_minus), where nbr_plus is
        the neighbour across the + face (its - trace) and nbr_minus the
        neighbour across the - face (its + trace)."""
        ax = self.elem_axis(d)
        tp, tm = self.trace(F, d, +1), self.trace(F, d, -1)
        return tp, _roll(tm, -1, ax), _roll(tp, +1, ax), tm


def _scale(d, me):
    return 2.0 / (me.dx if d == 0 else (me.dy if d == 1 else me.dz))


def lifting(disc: Disc, Wf, ops=None):
    """BR1 lifted gradients of w_grad (eq:Lifting, central surface
    value P:861):  d^d = (2/h_d) [ sum Dhat g + g*_+ lhat(1) - g*_- lhat(-1) ].
    Returns (gx, gy), each a tuple (u_d, v_d, T_d) of field-shaped arrays."""
    ops = ops or _Ops(disc)
    eq, me = disc.eq, disc.mesh
    g = physics.grad_vars(eq, _split(Wf, 2))
    G = ad.stack(list(g), axis=2)                       # (ny, nx, 3, p, p)
    out = []
    for d in range(2):
        own_p, nbr_p, nbr_m, own_m = ops.faces(G, d)
        gstar_p = 0.5 * (own_p + nbr_p)                 # canonical L = own, R = nbr
        gstar_m = 0.5 * (nbr_m + own_m)                 # canonical L = nbr, R = own
        D = _scale(d, me) * (ops.volume(G, d) + ops.surface(gstar_p, gstar_m, d))
        out.append(_split(D, 2))
    return out[0], out[1]


def _deriv_strong(disc: Disc, G, d):
    """Strong-form derivative (2/h_d) sum_l D_il g_l along direction d (nodal)."""
    D = disc.basis.D
    sc = _scale(d, disc.mesh)
    if d == 0:
        return sc * _lin(lambda c: np.einsum("il,...jl->...ji", D, c), G)
    return sc * _lin(lambda c: np.einsum("jm,...mi->...ji", D, c), G)


def lifting_br2_faces(disc: Disc, Wf, ops=None):
    """BR2 face gradients (reading R33).  For each face f of an element,
    the local lifting keeps the volume part of eq:Lifting and only the surface
    contribution of f, scaled by eta_BR2; in the strong form that is
        d_f = grad_h g + eta (2/h_d) (+-) (g*_f - g_f) lhat(+-1)      (normal component d only),
    evaluated on f:  d_f = trace_f(grad_h g) + eta (2/h_d) (+-) (g*_f - g_f) c_+-,
    c_+- = sum_i l_i(+-1) lhat_i(+-1) (GLL: 1/w_N, 1/w_0), with g* = 1/2 (g_L + g_R).
    Returns, per direction d, the canonical tuple (own_plus, nbr_plus, nbr_minus, own_minus) of
    (gx, gy) face gradients, each a pair of (ny, nx, 3, p) arrays (as ops.faces of Gx, Gy)."""
    ops = ops or _Ops(disc)
    eq, me = disc.eq, disc.mesh
    b = disc.basis
    eta = eq.eta_br2
    cp = float(np.dot(b.l_plus, b.lhat_plus))
    cm = float(np.dot(b.l_minus, b.lhat_minus))
    g = physics.grad_vars(eq, _split(Wf, 2))
    G = ad.stack(list(g), axis=2)                       # (ny, nx, 3, p, p)
    DG = [_deriv_strong(disc, G, 0), _deriv_strong(disc, G, 1)]
    out = []
    for d in range(2):
        own_p, nbr_p, nbr_m, own_m = ops.faces(G, d)
        gstar_p = 0.5 * (own_p + nbr_p)
        gstar_m = 0.5 * (nbr_m + own_m)
        sc = _scale(d, me)
        fp = []            # own plus-face gradient, components (x, y)
        fm = []
        for c in range(2):
            tp = ops.trace(DG[c], d, +1)
            tm = ops.trace(DG[c], d, -1)
            if c == d:
                tp = tp + (eta * sc * cp) * (gstar_p - own_p)
                tm = tm - (eta * sc * cm) * (gstar_m - own_m)
            fp.append(tp)
            fm.append(tm)
        ax = ops.elem_axis(d)
        nbp = [_roll(x, -1, ax) for x in fm]           # neighbour across + face: its minus-face gradient
        nbm = [_roll(x, +1, ax) for x in fp]           # neighbour across - face: its plus-face gradient
        out.append((fp, nbp, nbm, fm))
    return out


def rhs1_field(disc: Disc, Wf, absolute=False):
    """R^(1)_h on a field-shaped array (values, duals or hyper-duals).
    absolute=True returns R1_abs (plain values only): every term of
    eq:DGSEM_wt replaced by its magnitude -- the scale of R1's rounding."""
    ops = _Ops(disc, absolute)
    ab = (lambda xs: [np.abs(x) for x in xs]) if absolute else (lambda xs: xs)
    eq, me = disc.eq, disc.mesh
    dim = me.dim
    va = dim                                            # variable axis: after the element axes
    assert dim < 3 or not eq.viscous, "3D: inviscid (Euler / advection) only (NEXT-4 scope)"
    w = _split(Wf, va)
    if eq.viscous:
        gx, gy = lifting(disc, Wf, ops)
        Gx, Gy = ad.stack(list(gx), axis=2), ad.stack(list(gy), axis=2)
        if eq.lifting == "br2":
            br2 = lifting_br2_faces(disc, Wf, _Ops(disc))
    total = 0.0
    for d in range(dim):
        # volume flux at the nodes
        F = list(physics.flux(eq, w, d))
        if eq.viscous:
            Fv = physics.viscous_flux(eq, w, gx, gy, d)
            F = [f - fv for f, fv in zip(F, Fv)]
        Fa = ad.stack(F, axis=va)
        # traces of the state (and of the lifted gradients for NS)
        wp, wnp, wnm, wm = [_split(t, va) for t in ops.faces(Wf, d)]
        fp = list(physics.numerical_flux(eq, wp, wnp, d))   # + face: L = own, R = nbr
        fm = list(physics.numerical_flux(eq, wnm, wm, d))   # - face: L = nbr, R = own
        if eq.viscous and eq.lifting == "br2":
            faces = br2[d]                                  # (own+, nbr+, nbr-, own-), each (x, y)
            gxp, gxnp, gxnm, gxm = [_split(t[0], 2) for t in faces]
            gyp, gynp, gynm, gym = [_split(t[1], 2) for t in faces]
        elif eq.viscous:
            gxp, gxnp, gxnm, gxm = [_split(t, 2) for t in ops.faces(Gx, d)]
            gyp, gynp, gynm, gym = [_split(t, 2) for t in ops.faces(Gy, d)]
        if eq.viscous:
            fvL = physics.viscous_flux(eq, wp, gxp, gyp, d)
            fvR = physics.viscous_flux(eq, wnp, gxnp, gynp, d)
            fp = [f - 0.5 * (a + b) for f, a, b in zip(fp, fvL, fvR)]
            fvL = physics.viscous_flux(eq, wnm, gxnm, gynm, d)
            fvR = physics.viscous_flux(eq, wm, gxm, gym, d)
            fm = [f - 0.5 * (a + b) for f, a, b in zip(fm, fvL, fvR)]
        if absolute:
            Fa = ad.stack(ab(F), axis=va)
        fpa = ad.stack(ab(fp), axis=va)
        fma = ad.stack(ab(fm), axis=va)
        total = total + _scale(d, me) * (ops.volume(Fa, d) + ops.surface(fpa, fma, d))
    return total if absolute else -total


def rhs1(disc: Disc, W):
    """R^(1)_h(W) for a flat layout-L vector (or Jet of flat vectors)."""
    return disc.to_flat(rhs1_field(disc, disc.to_field(W)))


def rhs1_abs(disc: Disc, W):
    """R1_abs(W): magnitude version of R1 (rounding scale, reading R10b)."""
    return disc.to_flat(rhs1_field(disc, disc.to_field(np.asarray(W, float)), absolute=True))


def rhs2(disc: Disc, W, sigma):
    """R^(2)_h(W, sigma): dual part of R^(1)_h(W + e1 sigma)."""
    return rhs1(disc, ad.Jet(np.asarray(W, float), np.asarray(sigma, float))).d1


def rhs12(disc: Disc, W, sigma):
    """(R^(1)_h(W), R^(2)_h(W, sigma)) from one dual evaluation."""
    r = rhs1(disc, ad.Jet(np.asarray(W, float), np.asarray(sigma, float)))
    return r.v, r.d1
