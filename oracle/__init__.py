"""CPU ORACLE for arXiv 2104.12916 — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct fp64 CPU implementation (NumPy / SciPy) of
what the B200 hot path computes: the single-factorization inexact IPM whose
inner solve is PCG on the inequality-constraint-reduced system

    K_F Δν = r_ν,   K_F = D − [C 0] F⁻¹ [Cᵀ; 0],   F = [−H Aᵀ; A 0]
                                                

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2104_12916_b200``) never imports, links or calls it,
and this package never imports the product: the two share no code; only the
seeded input generator ``qpgen`` (problem data, no method arithmetic) serves
both.

Modules
-------
fsolve    F-solves: dense block formula f-inv, sparse SuperLU
kkt       residuals, slack elimination, r_ν, K_F·p, recovery, P_L, P_H
pcg       textbook left-preconditioned CG
ipm       the IPM loop (readings: SURVEY.md §8(c) c3)
symbolic  elimination tree, column counts, supernodes, levels (structure parity)
costs     the paper's flop-cost model
spectral  dense K_F two ways, preconditioned spectra

Pins: every function is checked in ``tests/test_oracle_*.py`` against
something other than itself (closed forms, brute-force dense KKT, the
paper's theorems, SPEC hand examples, textbook routines).  Functions without
such a pin would say "parity unpinned" here; there are none.
"""
