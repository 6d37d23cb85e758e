"""Pins for oracle.tableau.  CPU only, exact rationals."""
import json
import os
from fractions import Fraction as Fr

import pytest

from oracle.tableau import tableau_exact, tableau

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


@pytest.mark.parametrize("q", [4, 6, 8])
def test_quadrature_exactness(q):
    """sum_j B1_lj c_j^m + m sum_j B2_lj c_j^(m-1) = c_l^(m+1)/(m+1) for
    0 <= m <= q-1: I_l integrates t^m over [0, c_l] exactly with f = t^m,
    f' = m t^(m-1) (order q per P:93-99).  Exact arithmetic."""
    c, B1, B2 = tableau_exact(q)
    s = len(c)
    for l in range(s):
        for m in range(q):
            lhs = sum(B1[l][j] * c[j] ** m for j in range(s))
            if m > 0:
                lhs += m * sum(B2[l][j] * c[j] ** (m - 1) for j in range(s))
            assert lhs == c[l] ** (m + 1) / (m + 1), (q, l, m)


@pytest.mark.parametrize("q", [4, 6, 8])
def test_structure(q):
    c, B1, B2 = tableau_exact(q)
    assert c[0] == 0 and c[-1] == 1
    assert all(x == 0 for x in B1[0]) and all(x == 0 for x in B2[0])
    # predictor pairs (alpha1, alpha2) = (dc/2, dc^2/6) are stage-independent
    dcs = {c[l] - c[l - 1] for l in range(1, len(c))}
    assert len(dcs) == 1
    dc = dcs.pop()
    want = [Fr(x) for x in GOLD["predictor_pairs"][str(q)]]
    assert [dc / 2, dc * dc / 6] == want


def test_printed_values():
    g = GOLD["tableau_q4"]
    c, B1, B2 = tableau_exact(4)
    assert c == [Fr(x) for x in g["c"]]
    assert B1 == [[Fr(x) for x in r] for r in g["B1"]]
    assert B2 == [[Fr(x) for x in r] for r in g["B2"]]
    assert tableau_exact(8)[0] == [Fr(x) for x in GOLD["tableau_q8_c"]["c"]]
    cf, _, _ = tableau(6)
    assert list(cf) == [0.0, 0.5, 1.0]


def test_unsupported():
    with pytest.raises(ValueError):
        tableau_exact(5)
