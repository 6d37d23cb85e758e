"""Pins for oracle.basis.  CPU only."""
import json
import os

import numpy as np
import pytest

from oracle.basis import build_basis

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_gl_N1_worked_example():
    g = GOLD["gl_N1"]
    b = build_basis(1, "gl")
    np.testing.assert_allclose(b.xi, g["xi"], rtol=0, atol=2.3e-16)   # printed to 16 digits
    np.testing.assert_allclose(b.w, g["w"], rtol=0, atol=1e-16)
    np.testing.assert_allclose(b.Dhat, g["Dhat"], rtol=0, atol=1e-15)


def test_gl_N0_midpoint():
    b = build_basis(0, "gl")
    assert b.xi[0] == 0.0 and b.w[0] == 2.0


@pytest.mark.parametrize("kind", ["gl", "gll"])
@pytest.mark.parametrize("N", [1, 2, 3, 5, 7, 8])
def test_basis_invariants(kind, N):
    b = build_basis(N, kind)
    # weights sum to 2, nodes symmetric and increasing
    assert abs(b.w.sum() - 2.0) < 1e-14
    assert np.all(np.diff(b.xi) > 0)
    np.testing.assert_allclose(b.xi, -b.xi[::-1], atol=1e-15)
    # polynomial exactness of D: D xi^k = k xi^(k-1)
    for k in range(N + 1):
        lhs = b.D @ b.xi ** k
        rhs = k * b.xi ** (k - 1) if k > 0 else 0 * b.xi
        np.testing.assert_allclose(lhs, rhs, atol=1e-12)
    # summation by parts: MD + (MD)^T = l(1)l(1)^T - l(-1)l(-1)^T
    M = np.diag(b.w)
    B = np.outer(b.l_plus, b.l_plus) - np.outer(b.l_minus, b.l_minus)
    np.testing.assert_allclose(M @ b.D + (M @ b.D).T, B, atol=1e-12)
    # quadrature exactness: degree 2N+1 (GL), 2N-1 (GLL)
    deg = 2 * N + 1 if kind == "gl" else 2 * N - 1
    for k in range(deg + 1):
        exact = 0.0 if k % 2 else 2.0 / (k + 1)
        assert abs(np.dot(b.w, b.xi ** k) - exact) < 1e-13
    # ... and NOT for degree deg+1 (the rule is not over-exact by accident)
    k = deg + 1
    assert abs(np.dot(b.w, b.xi ** k) - (0.0 if k % 2 else 2.0 / (k + 1))) > 1e-6
    # partition of unity at the ends
    assert abs(b.l_plus.sum() - 1) < 1e-13 and abs(b.l_minus.sum() - 1) < 1e-13
    # free-stream row identity sum_l Dhat_il = -lhat_i(1) + lhat_i(-1)
    np.testing.assert_allclose(b.Dhat.sum(axis=1), -b.lhat_plus + b.lhat_minus,
                               atol=1e-13 * max(1, np.abs(b.Dhat).max()))


@pytest.mark.parametrize("N", [2, 3, 5, 7])
def test_gll_closed_forms(N):
    """GLL: xi_0 = -1, xi_N = 1, omega_end = 2/(N(N+1)), l(+-1) = unit vectors,
    hence lhat_N(1) = N(N+1)/2."""
    b = build_basis(N, "gll")
    assert b.xi[0] == -1.0 and b.xi[-1] == 1.0
    assert abs(b.w[0] - 2.0 / (N * (N + 1))) < 1e-15
    np.testing.assert_array_equal(b.l_plus, np.eye(N + 1)[-1])
    np.testing.assert_array_equal(b.l_minus, np.eye(N + 1)[0])
    assert abs(b.lhat_plus[-1] - N * (N + 1) / 2) < 1e-12


@pytest.mark.parametrize("kind", ["gl", "gll"])
def test_printed_dhat_ratio_breaks_free_stream(kind):
    """Reading R2: P:192 prints Dhat_ij = -(w_i/w_j) l'_i(xi_j).  That form
    violates the free-stream row identity for N >= 2, the transposed ratio
     satisfies it -- this is why the oracle uses the latter."""
    b = build_basis(5, kind)
    printed = -(b.w[:, None] / b.w[None, :]) * b.D.T
    resid = np.abs(printed.sum(1) + b.lhat_plus - b.lhat_minus).max()
    assert resid > 1.0
    assert np.abs(b.Dhat.sum(1) + b.lhat_plus - b.lhat_minus).max() < 1e-13
