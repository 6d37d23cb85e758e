"""Hyper-dual numbers x = v + d1*e1 + d2*e2 + d12*e1*e2 with e1^2 = e2^2 = 0.

TEST INFRASTRUCTURE (see oracle/__init__.py).

Why: the paper defines R^(2)_h by differentiating the discrete weak form in
time with w_t = sigma (eq:Euler_wtt; NS: P:869-890).  That is the
directional derivative of R^(1)_h in direction sigma, which forward-mode
automatic differentiation computes exactly (to rounding), without any
hand-derived flux Jacobian.  A hyper-dual evaluation
    f(W + e1*a + e2*b) = f + e1 f'a + e2 f'b + e1e2 f''[a,b]
additionally yields the Hessian term dR^(2)/dW * dW of eq:nonlinear_eqsys
 for the EXACT Jacobian-vector product.

Components may be numpy arrays or python/numpy scalars (a scalar 0.0 stands
for an all-zero component and broadcasts).
"""
import numpy as np


def _isz(c):
    return np.ndim(c) == 0 and c == 0.0


class Jet:
    __slots__ = ("v", "d1", "d2", "d12")

    def __init__(self, v, d1=0.0, d2=0.0, d12=0.0):
        self.v, self.d1, self.d2, self.d12 = v, d1, d2, d12

    # ---- construction helpers -------------------------------------------
    @staticmethod
    def lift(x):
        return x if isinstance(x, Jet) else Jet(x)

    def comps(self):
        return (self.v, self.d1, self.d2, self.d12)

    # ---- ring operations --------------------------------------------------
    def __add__(self, o):
        if not isinstance(o, Jet):
            return Jet(self.v + o, self.d1, self.d2, self.d12)
        return Jet(self.v + o.v, self.d1 + o.d1, self.d2 + o.d2, self.d12 + o.d12)

    __radd__ = __add__

    def __neg__(self):
        return Jet(-self.v, -self.d1, -self.d2, -self.d12)

    def __sub__(self, o):
        if not isinstance(o, Jet):
            return Jet(self.v - o, self.d1, self.d2, self.d12)
        return Jet(self.v - o.v, self.d1 - o.d1, self.d2 - o.d2, self.d12 - o.d12)

    def __rsub__(self, o):
        return (-self) + o

    def __mul__(self, o):
        if not isinstance(o, Jet):
            return Jet(self.v * o, self.d1 * o, self.d2 * o, self.d12 * o)
        a, b = self, o
        return Jet(a.v * b.v,
                   a.v * b.d1 + a.d1 * b.v,
                   a.v * b.d2 + a.d2 * b.v,
                   a.v * b.d12 + a.d1 * b.d2 + a.d2 * b.d1 + a.d12 * b.v)

    __rmul__ = __mul__

    def __truediv__(self, o):
        if not isinstance(o, Jet):
            return Jet(self.v / o, self.d1 / o, self.d2 / o, self.d12 / o)
        q = self * recip(o)
        q.v = self.v / o.v           # value part rounds exactly like plain a/b
        return q

    def __rtruediv__(self, o):
        q = recip(self) * o
        q.v = o / self.v
        return q

    # ---- linear structural maps (indexing, reshaping) ---------------------
    def __getitem__(self, idx):
        return Jet(*[c if np.ndim(c) == 0 else c[idx] for c in self.comps()])

    @property
    def shape(self):
        return np.shape(self.v)


def apply_linear(f, x):
    """Apply a linear map f (einsum, roll, slicing, ...) component-wise."""
    if not isinstance(x, Jet):
        return f(x)
    return Jet(*[c if _isz(c) else f(c) for c in x.comps()])


def _scalar_fn(x, f0, f1, f2):
    """Chain rule for a scalar function with value f0, derivative f1 and
    second derivative f2 at x.v:
      f(x) = f0 + f1 d1 e1 + f1 d2 e2 + (f1 d12 + f2 d1 d2) e1 e2."""
    return Jet(f0, f1 * x.d1, f1 * x.d2, f1 * x.d12 + f2 * x.d1 * x.d2)


def recip(x):
    if not isinstance(x, Jet):
        return 1.0 / x
    r = 1.0 / x.v
    return _scalar_fn(x, r, -r * r, 2.0 * r * r * r)


def sqrt(x):
    if not isinstance(x, Jet):
        return np.sqrt(x)
    s = np.sqrt(x.v)
    return _scalar_fn(x, s, 0.5 / s, -0.25 / (s * x.v))


def absval(x):
    """|x| with sign(0) := +1."""
    if not isinstance(x, Jet):
        return np.abs(x)
    sg = np.where(x.v >= 0.0, 1.0, -1.0)
    return Jet(sg * x.v, sg * x.d1, sg * x.d2, sg * x.d12)


def maxval(a, b):
    """max(a, b) branch-wise on the value part; ties take a (the first, i.e.
    the canonical left state)."""
    if not isinstance(a, Jet) and not isinstance(b, Jet):
        return np.where(a >= b, a, b)
    a, b = Jet.lift(a), Jet.lift(b)
    pick = a.v >= b.v
    return Jet(*[np.where(pick, ca, cb) for ca, cb in zip(a.comps(), b.comps())])


def value(x):
    return x.v if isinstance(x, Jet) else x


def stack(xs, axis):
    """np.stack for a list of Jets/arrays (zero components broadcast)."""
    if not any(isinstance(x, Jet) for x in xs):
        return np.stack(xs, axis=axis)
    xs = [Jet.lift(x) for x in xs]
    shape = np.broadcast_shapes(*[np.shape(c) for x in xs for c in x.comps()])
    out = []
    for k in range(4):
        cs = [x.comps()[k] for x in xs]
        if all(_isz(c) for c in cs):
            out.append(0.0)
        else:
            out.append(np.stack([np.broadcast_to(c, shape) for c in cs], axis=axis))
    return Jet(*out)


def strip(x):
    """Drop all derivative parts (used for 'frozen neighbour' evaluations)."""
    return value(x)
