"""Synthetic finite-difference Oseen blocks (stand-in for the paper's IFISS Q2-Q1 matrices).

The paper's spatial matrices (mass M, stiffness A_l, convection N(w),
divergence B) come from IFISS on the step domain, which is not available.  BASELINE.json
configs replace them by a seeded finite-difference Oseen family on the unit square; the
reading fixed in DESIGN.md (R10, R11):

* N x N interior nodes, h = 1/(N+1), homogeneous Dirichlet, node (ix, iy) -> iy*N + ix.
* L = -Delta_h, 5-point stencil (SPD, the sign of A_l).
* N(w) = diag(w1) D_x + diag(w2) D_y, central differences (no stabilisation).
* B1, B2 forward differences; velocity rows carry B1^T, B2^T.
* velocity mass M = I, pressure mass 0 (no pressure time derivative).
* spatial dofs are stacked [u1; u2; p], n_x = 3 N^2 (one spatial TT mode, BASELINE.json:7).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def _shift_ops(n: int):
    """1-D shift matrices with zero Dirichlet extension: (E u)_i = u_{i+1}, (W u)_i = u_{i-1}."""
    e = sp.diags([np.ones(n - 1)], [1], shape=(n, n), format="csr")
    w = sp.diags([np.ones(n - 1)], [-1], shape=(n, n), format="csr")
    return e, w


def grid_coords(n: int):
    h = 1.0 / (n + 1)
    x = (np.arange(n) + 1) * h
    xx, yy = np.meshgrid(x, x, indexing="xy")  # xx[iy, ix]
    return xx.ravel(), yy.ravel(), h


def laplacian(n: int) -> sp.csr_matrix:
    """-Delta_h on the N x N interior grid (x fastest)."""
    h = 1.0 / (n + 1)
    i1 = sp.identity(n, format="csr")
    t = sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1], format="csr")
    return ((sp.kron(i1, t) + sp.kron(t, i1)) / (h * h)).tocsr()


def central_dx(n: int) -> sp.csr_matrix:
    h = 1.0 / (n + 1)
    e, w = _shift_ops(n)
    return (sp.kron(sp.identity(n), (e - w)) / (2 * h)).tocsr()


def central_dy(n: int) -> sp.csr_matrix:
    h = 1.0 / (n + 1)
    e, w = _shift_ops(n)
    return (sp.kron((e - w), sp.identity(n)) / (2 * h)).tocsr()


def forward_dx(n: int) -> sp.csr_matrix:
    h = 1.0 / (n + 1)
    e, _ = _shift_ops(n)
    return (sp.kron(sp.identity(n), (e - sp.identity(n))) / h).tocsr()


def forward_dy(n: int) -> sp.csr_matrix:
    h = 1.0 / (n + 1)
    e, _ = _shift_ops(n)
    return (sp.kron((e - sp.identity(n)), sp.identity(n)) / h).tocsr()


def convection(n: int, w1: np.ndarray, w2: np.ndarray) -> sp.csr_matrix:
    """N(w) = diag(w1) D_x + diag(w2) D_y (central)."""
    return (sp.diags(w1) @ central_dx(n) + sp.diags(w2) @ central_dy(n)).tocsr()


def sinusoid_wind(n: int, rng: np.random.Generator, scale: float = 1.0):
    """One wind field: each component sum_{s=1..3} a_s sin(pi(k_s x + l_s y) + phi_s),
    a_s ~ N(0,1), k_s, l_s in {1,2,3}, phi_s ~ U[0, 2pi)  (R11)."""
    xs, ys, _ = grid_coords(n)
    comps = []
    for _c in range(2):
        a = rng.standard_normal(3)
        k = rng.integers(1, 4, size=3)
        l = rng.integers(1, 4, size=3)
        phi = rng.uniform(0.0, 2.0 * np.pi, size=3)
        w = np.zeros_like(xs)
        for s in range(3):
            w += a[s] * np.sin(np.pi * (k[s] * xs + l[s] * ys) + phi[s])
        comps.append(scale * w)
    return comps[0], comps[1]


def _z(n2: int) -> sp.csr_matrix:
    return sp.csr_matrix((n2, n2))


def stacked(blocks) -> sp.csr_matrix:
    """3 x 3 block matrix over [u1; u2; p] with None -> zero block."""
    n2 = next(b.shape[0] for row in blocks for b in row if b is not None)
    rows = [[(b if b is not None else _z(n2)) for b in row] for row in blocks]
    m = sp.bmat(rows, format="csr")
    m.sum_duplicates()
    m.sort_indices()
    return m


def mass_block(n: int) -> sp.csr_matrix:
    """blkdiag(I, I, 0): velocity identity mass, no pressure mass."""
    i = sp.identity(n * n, format="csr")
    return stacked([[i, None, None], [None, i, None], [None, None, None]])


def oseen_block(n: int, nu0: float, w0) -> sp.csr_matrix:
    """[[nu0 L + N(w0), 0, B1^T], [0, nu0 L + N(w0), B2^T], [B1, B2, 0]]."""
    f = (nu0 * laplacian(n) + convection(n, *w0)).tocsr()
    b1 = forward_dx(n)
    b2 = forward_dy(n)
    return stacked([[f, None, b1.T.tocsr()], [None, f, b2.T.tocsr()], [b1, b2, None]])


def viscous_block(n: int, nu: float) -> sp.csr_matrix:
    """blkdiag(nu L, nu L, 0)."""
    l = (nu * laplacian(n)).tocsr()
    return stacked([[l, None, None], [None, l, None], [None, None, None]])


def wind_block(n: int, w) -> sp.csr_matrix:
    """blkdiag(N(w), N(w), 0)."""
    c = convection(n, *w)
    return stacked([[c, None, None], [None, c, None], [None, None, None]])
