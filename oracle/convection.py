"""The stochastic Galerkin convection matrix N(u) from its DEFINITION, dense (tests only).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:317-322: with the velocity coefficient tensor u(k, l, j) (time k, chaos index l,
spatial dof j), the k-th diagonal time block of N(u) is

    sum_{l=1}^{n_xi} H_l (x) N(u_{h,l}^k),   u_{h,l}^k = sum_j u(k, l, j) phi_j,

i.e. the convection matrix is block diagonal in time and, per time step, a Galerkin sum over
the chaos modes of the velocity.  Here the full coefficient tensor is formed from the TT
cores (x, xi, t order, R1) and every block is built from that definition: no TT
structure (no alpha sums, eq:N_kron) is used.  N_of(w_vec) maps a spatial coefficient vector
to its (sparse) convection matrix and H the list of H_l — both passed in, so this module holds
no stencil or chaos arithmetic of its own.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def full_tensor(U1, U2, U3) -> np.ndarray:
    """u[j, l, k] = sum_{a,b} U1[j, a] U2[a, l, b] U3[b, k]."""
    return np.einsum("ja,alb,bk->jlk", U1, U2, U3)


def dense_convection(U1, U2, U3, H, N_of) -> sp.csr_matrix:
    """N(u) on the vector ordered (t, xi, x) with x fastest (vec of the TT, R1)."""
    u = full_tensor(U1, U2, U3)
    n_x, n_xi, n_t = u.shape
    blocks = []
    for k in range(n_t):
        bk = None
        for l in range(n_xi):
            term = sp.kron(sp.csr_matrix(H[l]), N_of(u[:, l, k]))
            bk = term if bk is None else bk + term
        blocks.append(bk)
    return sp.block_diag(blocks, format="csr")
