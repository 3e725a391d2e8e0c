"""CPU ORACLE for arXiv 2010.00881 (hierarchical p-multigrid for the finite cell method).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import or run
anything under ``oracle/``.  The product path (``paper_2010_00881_b200``) never
imports it and the oracle never imports the product path; the two share no code.
Only the seeded input generators in ``workloads/`` (no method arithmetic) feed both.

Plain, slow, obviously-correct numpy/scipy in fp64, following PAPER.md:
  basis.py      integrated-Legendre 1D modes, tensor/trunk element modes
  geometry.py   exact point/box classification against spherical voids (P:55 alpha(x))
  quadrature.py space-tree cut-cell quadrature, element matrices and loads (Eq. weakform)
  dofmap.py     global DOF numbering, Dirichlet elimination, p-levels
  assembly.py   global CSR assembly and element-by-element operator
  mg.py         additive Schwarz (Eq. AdditiveSchwarz), Algorithm 1 V-cycle
                (P:150-183), coarse solve, flexible PCG
  problem.py    builds a whole workload from a workloads.Config

Every function cites the passage it follows.  Readings of ambiguous passages are
listed in DESIGN.md ("Readings").  Parity-unpinned functions: none are knowingly
unpinned -- see tests/test_oracle_*.py for the pins of each module.
"""
