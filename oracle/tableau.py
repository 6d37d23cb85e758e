"""Two-derivative Butcher tableaux (c, B^(1), B^(2)) of PAPER App. A.

TEST INFRASTRUCTURE (see oracle/__init__.py).

Transcribed as exact rationals from eq:butcher4, eq:butcher6
 and eq:butcher8.  They define the stage
quadrature I_l = dt sum_j B1_lj R1_j + dt^2 sum_j B2_lj R2_j.
Pinned in tests/test_oracle_tableau.py by the quadrature exactness
conditions (exact rational arithmetic).
"""
from fractions import Fraction as Fr

import numpy as np

_TAB = {
    4: dict(
        c=[Fr(0), Fr(1)],
        B1=[[Fr(0), Fr(0)],
            [Fr(1, 2), Fr(1, 2)]],
        B2=[[Fr(0), Fr(0)],
            [Fr(1, 12), Fr(-1, 12)]]),
    6: dict(
        c=[Fr(0), Fr(1, 2), Fr(1)],
        B1=[[Fr(0), Fr(0), Fr(0)],
            [Fr(101, 480), Fr(8, 30), Fr(55, 2400)],
            [Fr(7, 30), Fr(16, 30), Fr(7, 30)]],
        B2=[[Fr(0), Fr(0), Fr(0)],
            [Fr(65, 4800), Fr(-25, 600), Fr(-25, 8000)],
            [Fr(5, 300), Fr(0), Fr(-5, 300)]]),
    8: dict(
        c=[Fr(0), Fr(1, 3), Fr(2, 3), Fr(1)],
        B1=[[Fr(0), Fr(0), Fr(0), Fr(0)],
            [Fr(6893, 54432), Fr(313, 2016), Fr(89, 2016), Fr(397, 54432)],
            [Fr(223, 1701), Fr(20, 63), Fr(13, 63), Fr(20, 1701)],
            [Fr(31, 224), Fr(81, 224), Fr(81, 224), Fr(31, 224)]],
        B2=[[Fr(0), Fr(0), Fr(0), Fr(0)],
            [Fr(1283, 272160), Fr(-851, 30240), Fr(-269, 30240), Fr(-163, 272160)],
            [Fr(43, 8505), Fr(-16, 945), Fr(-19, 945), Fr(-8, 8505)],
            [Fr(19, 3360), Fr(-9, 1120), Fr(9, 1120), Fr(-19, 3360)]]),
}


def tableau_exact(q):
    """Exact rational (c, B1, B2) for q in {4, 6, 8}."""
    if q not in _TAB:
        raise ValueError(f"unsupported order q={q}")
    t = _TAB[q]
    return t["c"], t["B1"], t["B2"]


def tableau(q):
    """fp64 (c, B1, B2) as numpy arrays."""
    c, B1, B2 = tableau_exact(q)
    return (np.array([float(x) for x in c]),
            np.array([[float(x) for x in r] for r in B1]),
            np.array([[float(x) for x in r] for r in B2]))
