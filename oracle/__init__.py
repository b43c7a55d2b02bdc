"""CPU oracle for the TT apply / round / dot / axpby / GMRES-cycle path of arXiv:1906.06785.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product package
``paper_1906_06785_b200`` never imports it and has no CPU fallback.

Plain, slow, obviously-correct NumPy/SciPy in float64, following the paper step by step
(every function cites the passage it restates).  It shares no code with the CUDA path; both
consume the seeded inputs of ``synth/``.

Pins (tests/test_oracle_*.py, all ``-m "not gpu"``):
  * tt.apply_op      vs the explicit sparse Kronecker matvec (kron_dense.py)       — exact
  * tt.round_tt      vs dense TT-SVD of the full tensor (tt.tt_svd_dense, Alg. 2),
                     the bound ||x~ - x|| <= eps ||x||, orthonormal cores,
                     closed-form spectra, rank monotonicity, zero-padding             — exact/invariants
  * tt.dot/axpby/norm vs dense inner products and sums                             — exact
  * gpc_quadrature   vs the closed-form G_l of synth.gpc (and vice versa)          — exact
  * gmres.gmres_cycle at tol 1e-14 vs dense GMRES on the explicit matrix            — exact
  * gmres.gmres_cycle at tol 1e-6: parity unpinned beyond GPU-vs-oracle agreement
  * gpc_quadrature.h_by_quadrature vs the closed-form H_l (synth.gpc), H_1 = I, H_{e_i} = G_i
  * convection.dense_convection (the definition) vs the Kronecker-sum N(u)
                     of eq:N_kron (convection.convection_operator); n_of vs w.grad f  — exact
"""
