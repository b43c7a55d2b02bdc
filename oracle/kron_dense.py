"""Explicit Kronecker-sum matrix, used to PIN the TT apply (tests only).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:157 (eq:F) writes each block as sum_l X^(1) (x) X^(2) (x) X^(3) acting on the vector
whose index is i3 + (i2-1) n_x + (i1-1) n_xi n_x: the last (space) factor
runs fastest, exactly the convention of scipy.sparse.kron(T, kron(G, K)).
"""
from __future__ import annotations

import scipy.sparse as sp


def kron_matrix(op) -> sp.csr_matrix:
    a = None
    for t in op.terms:
        tk = sp.csr_matrix(t.T_dense())
        blk = sp.kron(tk, sp.kron(sp.csr_matrix(t.G), t.K, format="csr"), format="csr")
        a = blk if a is None else a + blk
    return a.tocsr()
