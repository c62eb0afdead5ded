"""CPU ORACLE for arXiv 1805.11930's matrix-free DG hot path — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct fp64 numpy code written from PAPER.md. Only
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import it. The CUDA product path
(`paper_1805_11930_b200/`) never imports it and shares no code with it; the only
shared module is `synth/` (seeded inputs, no method arithmetic).

Modules
  basis   1D Gauss-Lobatto nodal basis + Gauss rule (§2.1; §3.1)
  tier_a  global dense A by brute-force 3D quadrature of a_h term by term
          (P:333-360 eq. bilinear_form_split) and l_h (P:361-371 eq. rhs)
  tier_b  per-cell dense blocks from 1D brute-force quadrature matrices and
          Kronecker products (derivation in SURVEY.md §8(c) step 3, re-derived in
          DESIGN.md); matrix-free-free reference apply, D_T, LU local solves and the
          block-Jacobi sweep of Alg. 2
  hybrid  the hybrid multigrid of Alg. 1 with the P0 subspace: P, R = P^T
          (P:725-735), A^ = P^T A P by brute force and by the rescaled finite-volume
          construction of App. A.1, the V-cycle with an exact coarse solve,
          and the V-cycle-preconditioned flexible CG
  sor     block SOR / SSOR of Alg. 3 written out for a traversal order, and its
          red-black coloured form

Pins: every function is checked in tests/test_oracle_*.py against closed forms,
invariants or the other tier (never against itself or the CUDA path).
"""
