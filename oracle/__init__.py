"""CPU oracle for the IgA curl-div hot path -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct fp64 implementation of what the CUDA path computes,
written from PAPER.md (arxiv 1805.10058, Mazza-Manni-Ratnani-Serra-Capizzano-Speleers).
Every function cites the passage it follows as  PAPER.md:<line> (<section / equation>).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything under ``oracle/``.  The product path
(``paper_1805_10058_b200``) never imports it, and the oracle never imports the product:
the two share no code, no tables, no helpers.  Seeded inputs come from ``inputs/``.

Modules
  bspline    -- knot vector, Cox-de Boor basis, cardinal B-splines, Gauss rule (Sec. 3.1)
  matrices1d -- M, A, S by element-wise Gauss quadrature (Sec. 3.2, eq:matr_M..S)
  operator   -- d x d block operator assembled element by element (Sec. 1 L_A, Sec. 4)
  transfer   -- knot-insertion prolongation and R = P^T (Sec. 6.1 Galerkin approach)
  multigrid  -- Galerkin hierarchy, damped Jacobi, V-cycle (Sec. 6.1 steps 1-3)
  krylov     -- preconditioned CG (Sec. 6.1 remark, Sec. 6.2 P_MIM usage)
  symbol     -- spectral symbols m_p, a_p, s_p, f^{p,alpha,beta} (Sec. 3.2, 5.1-5.2)

Parity pins live in tests/test_oracle_*.py; DESIGN.md lists them per function.
"""
