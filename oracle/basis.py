"""1D nodal basis of the DGSEM (eq:Interpolation, eq:DGSEM_wt).

TEST INFRASTRUCTURE (see oracle/__init__.py).

Everything is computed in 50-digit arithmetic (mpmath) and rounded once to
fp64:
  * nodes xi_i and weights omega_i: Gauss-Legendre (the paper's
    choice) or Gauss-Lobatto (BASELINE.json configs);
  * D_ij = l'_j(xi_i) (nodal differentiation matrix);
  * Dhat := -M^{-1} D^T M, i.e. Dhat_ij = -(omega_j/omega_i) l'_i(xi_j).
    PAPER P:192 prints the weight ratio as omega_i/omega_j; that version
    violates free-stream preservation for N >= 2, so the
    SPEC reading S:35/S:49 is used (reading R2);
  * l(+-1) = Lagrange polynomials at the element ends, lhat(+-1) = l(+-1)/omega
    (P:192).
"""
from dataclasses import dataclass

import mpmath as mp
import numpy as np

_DPS = 50


def _legendre(n, x):
    """P_n(x) and P_n'(x) by the three-term recurrence."""
    p0, p1 = mp.mpf(1), x
    if n == 0:
        return p0, mp.mpf(0)
    for k in range(2, n + 1):
        p0, p1 = p1, ((2 * k - 1) * x * p1 - (k - 1) * p0) / k
    if x * x == 1:                      # P_n'(+-1) = (+-1)^(n-1) n(n+1)/2
        return p1, (x ** (n - 1)) * n * (n + 1) / 2
    dp = n * (x * p1 - p0) / (x * x - 1)
    return p1, dp


def _newton(f, x0):
    x = mp.mpf(x0)
    for _ in range(200):
        fx, dfx = f(x)
        dx = fx / dfx
        x -= dx
        if abs(dx) < mp.mpf(10) ** (-_DPS + 5):
            break
    return x


def gauss_legendre(N):
    """N+1 Gauss-Legendre nodes (roots of P_{N+1}) and weights
    2 / ((1-x^2) P'_{N+1}(x)^2)."""
    with mp.workdps(_DPS):
        n = N + 1
        xs, ws = [], []
        for k in range(n):
            x0 = -mp.cos(mp.pi * (k + mp.mpf(3) / 4) / (n + mp.mpf(1) / 2))
            x = _newton(lambda t: _legendre(n, t), x0)
            _, dp = _legendre(n, x)
            xs.append(x)
            ws.append(2 / ((1 - x * x) * dp * dp))
        return xs, ws


def gauss_lobatto(N):
    """N+1 Gauss-Lobatto nodes (+-1 and the roots of P'_N) and weights
    2 / (N(N+1) P_N(x)^2)."""
    assert N >= 1
    with mp.workdps(_DPS):
        xs = [mp.mpf(-1)]
        for k in range(1, N):
            x0 = -mp.cos(mp.pi * k / N)

            def f(t):
                # g = P'_N, g' = P''_N from the Legendre ODE
                p, dp = _legendre(N, t)
                ddp = (2 * t * dp - N * (N + 1) * p) / (1 - t * t)
                return dp, ddp

            xs.append(_newton(f, x0))
        xs.append(mp.mpf(1))
        ws = []
        for x in xs:
            p, _ = _legendre(N, x)
            ws.append(mp.mpf(2) / (N * (N + 1) * p * p))
        return xs, ws


def _lagrange_at(xs, t):
    """[l_0(t), ..., l_N(t)]."""
    out = []
    for j, xj in enumerate(xs):
        v = mp.mpf(1)
        for k, xk in enumerate(xs):
            if k != j:
                v *= (t - xk) / (xj - xk)
        out.append(v)
    return out


def _diff_matrix(xs):
    """D_ij = l'_j(xi_i) via barycentric weights; D_ii = -sum_{j!=i} D_ij."""
    n = len(xs)
    bw = []
    for j in range(n):
        v = mp.mpf(1)
        for k in range(n):
            if k != j:
                v *= xs[j] - xs[k]
        bw.append(1 / v)
    D = [[mp.mpf(0)] * n for _ in range(n)]
    for i in range(n):
        for j in range(n):
            if i != j:
                D[i][j] = (bw[j] / bw[i]) / (xs[i] - xs[j])
        D[i][i] = -sum(D[i][j] for j in range(n) if j != i)
    return D


@dataclass
class Basis:
    N: int
    kind: str             # "gll" or "gl"
    xi: np.ndarray        # nodes
    w: np.ndarray         # quadrature weights omega
    D: np.ndarray         # D_ij = l'_j(xi_i)
    Dhat: np.ndarray      # -M^{-1} D^T M
    l_minus: np.ndarray   # l_i(-1)
    l_plus: np.ndarray    # l_i(+1)
    lhat_minus: np.ndarray
    lhat_plus: np.ndarray

    @property
    def p(self):
        return self.N + 1


def build_basis(N, kind="gll"):
    with mp.workdps(_DPS):
        xs, ws = gauss_lobatto(N) if kind == "gll" else gauss_legendre(N)
        D = _diff_matrix(xs)
        n = len(xs)
        Dhat = [[-(ws[j] / ws[i]) * D[j][i] for j in range(n)] for i in range(n)]
        lm = _lagrange_at(xs, mp.mpf(-1))
        lp = _lagrange_at(xs, mp.mpf(1))
        f = lambda a: np.array([[float(v) for v in r] for r in a]) if isinstance(a[0], list) \
            else np.array([float(v) for v in a])
        return Basis(N=N, kind=kind, xi=f(xs), w=f(ws), D=f(D), Dhat=f(Dhat),
                     l_minus=f(lm), l_plus=f(lp),
                     lhat_minus=f([lm[i] / ws[i] for i in range(n)]),
                     lhat_plus=f([lp[i] / ws[i] for i in range(n)]))
