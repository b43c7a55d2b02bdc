"""Seeded synthetic inputs shared by the CPU oracle and the CUDA path.

This package holds NO arithmetic of the method under test (TT apply, TT rounding,
TT dot/axpby, GMRES).  It only builds the *inputs* of that path:

* ``gpc``      — multi-index ordering of the Legendre chaos basis and the closed-form
                 Galerkin matrices G_l = <xi_l psi_r psi_s>  (R13)
* ``fd``       — the synthetic finite-difference Oseen blocks that stand in for the
                 paper's IFISS Q2-Q1 matrices (BASELINE.json configs; R10/R11)
* ``configs``  — the five named configurations c1..c5 of BASELINE.json
* ``operator`` — the Kronecker-sum term list  A = sum_k T_k (x) G_k (x) K_k  (PAPER.md:157 eq:F)
* ``tt``       — seeded input tensor trains

Both ``oracle/`` and the product package consume these objects; neither imports the other.
"""
from .configs import CONFIGS, get_config  # noqa: F401
from .operator import KronSumOp, Term, build_operator  # noqa: F401
from .tt import make_input_tt, make_rhs_tt  # noqa: F401
