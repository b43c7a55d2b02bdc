"""The stochastic Galerkin convection matrix N(u): its DEFINITION (dense, tests only) and the
Kronecker-sum form of eq:N_kron that the oracle applies.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:317-322: with the velocity coefficient tensor u(k, l, j) (time k, chaos index l,
spatial dof j), the k-th diagonal time block of N(u) is

    sum_{l=1}^{n_xi} H_l (x) N(u_{h,l}^k),   u_{h,l}^k = sum_j u(k, l, j) phi_j,

i.e. the convection matrix is block diagonal in time and, per time step, a Galerkin sum over
the chaos modes of the velocity.  Here the full coefficient tensor is formed from the TT
cores (x, xi, t order, R1) and every block is built from that definition: no TT
structure (no alpha sums, eq:N_kron) is used.  N_of(w_vec) maps a spatial coefficient vector
to its (sparse) convection matrix and H the list of H_l — both passed in.

convection_operator() is eq:N_kron written out: one term per (alpha_1,
alpha_2) with a diagonal time factor, the chaos factor sum_l u2 H_l and the spatial factor
N(u^(3)_{alpha_2}); n_of() is the spatial convection matrix of a velocity coefficient vector
(PAPER.md:126 [N(w)]_ij = (w . grad phi_j, phi_i), with the difference operators D_c of the
discretisation standing for the derivatives: N(w) = sum_c diag(w_c) D_c on every velocity
component, R10/R18).  The stencils D_c and the H_l are input data (synth/).
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


def n_of(w: np.ndarray, D, n_v: int, n_x: int) -> sp.csr_matrix:
    """N(w) = blkdiag over the d = len(D) velocity components of sum_c diag(w_c) D_c, zero on
    the rows/columns beyond d n_v (the pressure does not convect); w_c = w[c n_v:(c+1) n_v]."""
    d = len(D)
    blk = None
    for c in range(d):
        t = sp.diags(w[c * n_v:(c + 1) * n_v]) @ D[c]
        blk = t if blk is None else blk + t
    blocks = [blk] * d
    rest = n_x - d * n_v
    if rest:
        blocks.append(sp.csr_matrix((rest, rest)))
    return sp.block_diag(blocks, format="csr")


class Term:
    """One Kronecker term T (x) G (x) K of an oracle operator (dense T, dense G, sparse K)."""

    def __init__(self, T: np.ndarray, G: np.ndarray, K: sp.csr_matrix):
        self.T, self.G, self.K = T, G, K

    def T_dense(self) -> np.ndarray:
        return self.T


class Operator:
    """sum_k terms[k] on modes (n_x, n_xi, n_t) — what oracle.tt.apply_op consumes."""

    def __init__(self, n_x: int, n_xi: int, n_t: int, terms: list):
        self.n_x, self.n_xi, self.n_t, self.terms = n_x, n_xi, n_t, terms

    @property
    def T(self) -> int:
        return len(self.terms)


def convection_operator(U1, U2, U3, H, D, n_v: int) -> Operator:
    """eq:N_kron in this repo's core order (R18):

        N(u) = sum_{alpha_1, alpha_2} diag(u^(1)_{alpha_1}) (x) sum_l u^(2)(alpha_1, l, alpha_2) H_l
                                      (x) N(u^(3)_{alpha_2})

    with u^(1)(k, alpha_1) = U3[alpha_1, k], u^(2)(alpha_1, l, alpha_2) = U2[alpha_2, l, alpha_1],
    u^(3)(alpha_2, j) = U1[j, alpha_2]; terms ordered a = alpha_2 (space bond) major,
    b = alpha_1 (time bond) minor: term a r2 + b."""
    n_x, r1 = U1.shape
    r2, n_t = U3.shape
    n_xi = U2.shape[1]
    terms = []
    for a in range(r1):
        K = n_of(U1[:, a], D, n_v, n_x)
        for b in range(r2):
            G = sum(U2[a, l, b] * H[l] for l in range(n_xi))
            terms.append(Term(np.diag(U3[b, :]), G, K))
    return Operator(n_x, n_xi, n_t, terms)
