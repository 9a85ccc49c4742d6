"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU (NumPy, FP64) implementation of the
interpolation-and-lookup formation of K (Hirschler, Antolin, Buffa,
arXiv 2107.09568 — /root/reference/PAPER.md) and of the standard
full-Gauss-quadrature assembly K^• it is compared with.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import this package.  It shares no code with the
CUDA path (`paper_2107_09568_b200/`); the only common input is `synth/`
(seeded placement and random draws, none of the method's arithmetic).

Modules (each function cites the PAPER.md passage it follows):
  bspline      Cox–de Boor B-splines (Eq. 2), Bernstein basis (Eq. 21), Gauss–Legendre rules
  macro        macro field Ā_ij (Eq. 37 / App. A.2), three routes; interpolation onto Q_q (Eq. 42, reading R1)
  tables       sparsity set I_coo (Eq. 56) and lookup tables 𝔎 (Eqs. 51–52, 57)
  dofmap       DofMap, CSR pattern and block map (readings R9, R10)
  assemble     lookup K^π (Eqs. 50, 58) + scatter; standard K^• (Eq. 49 with Eq. 10)
  sensitivity  g = uᵀ(∂K^π/∂P)v via the lookup-table adjoint (Eqs. 70–73) and complex step

Parity pinned by tests/test_oracle_*.py except where a function header says
"parity unpinned" (also listed in DESIGN.md §4).
"""
