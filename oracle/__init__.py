"""CPU oracle for the HBPC(q, k_max) two-derivative DGSEM hot path (arXiv 2109.04804).

TEST INFRASTRUCTURE ONLY.  This package is the plain, slow, obviously-correct
fp64 reference the CUDA path is checked against.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product path
(``paper_2109_04804_b200``) never imports anything from here and shares no
code with it.

Citation convention: ``P:n`` = line n of the paper's LaTeX source,
``S:n`` = line n of SPEC.md, equations by their ``\\label{}`` name.

Modules
  ad        -- hyper-dual numbers (forward-mode AD: value, two directions, mixed)
  basis     -- Gauss-Lobatto / Gauss-Legendre nodes, weights, D, D-hat, l(+-1)
  tableau   -- Butcher tableaux of App. A (exact rationals)
  physics   -- advection / Euler / Navier-Stokes fluxes, LLF flux, viscous flux
  dgsem     -- mesh, R^(1)_h (eq:DGSEM_wt), BR1 lifting, R^(2)_h as d/dt of R^(1)_h
  implicit  -- residual G(X), JVPs, BJ_ext blocks, GMRES, Newton
  hbpc      -- Alg. 1 (predictor, corrector, FSAL)
  linear    -- closed forms used as pins (dense operator, Pade, expm)

Parity status of every function is listed in DESIGN.md section "Oracle pins".
"""
