"""NEXT-1: the TT-format convection operator N(u) of eq:N_kron.

Pins, all -m "not gpu":
  * H_l closed form (synth.gpc.h_matrices, Wigner-3j product) vs Gauss-Legendre quadrature of
    the definition <psi_l psi_r psi_s> (oracle.gpc_quadrature.h_by_quadrature); H_1 = I
    (psi_1 = 1); H_{e_i} = G_i (psi_{e_i} = xi_i); symmetry; parity selection;
  * the Kronecker-sum operator (synth.operator.convection_operator, alpha sums of eq:N_kron) vs
    the dense block definition sum_l H_l (x) N(u_{h,l}^k) per time step (oracle.convection);
  * linearity in u and the kappa -> kappa^2 rank growth of the apply.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import gpc_quadrature as gq
from oracle import tt
from oracle.convection import dense_convection
from oracle.kron_dense import kron_matrix
from synth import fd, gpc
from synth.operator import convection_operator
from synth.tt import random_tt


@pytest.mark.parametrize("m,p", [(1, 4), (2, 2), (3, 3), (4, 3)])
def test_h_closed_form_vs_quadrature(m, p):
    idx = gpc.multi_indices(m, p)
    H = gpc.h_matrices(m, p)
    Hq = gq.h_by_quadrature(idx, m, p)
    assert len(H) == gpc.n_xi(m, p)
    for a, b in zip(H, Hq):
        assert np.abs(a - b).max() <= 1e-14
        assert np.abs(a - a.T).max() == 0.0
    assert np.array_equal(H[0], np.eye(len(idx)))
    G = gpc.g_matrices(m, p)
    for i in range(m):  # degree-1 multi-index e_i sits at position 1 + i
        assert np.abs(H[1 + i] - G[1 + i]).max() <= 1e-15
    # parity: <psi_l psi_r psi_s> = 0 when the total degree |l| + |r| + |s| is odd
    for li, lam in enumerate(idx):
        for r, al in enumerate(idx):
            for s, be in enumerate(idx):
                if (sum(lam) + sum(al) + sum(be)) % 2:
                    assert H[li][r, s] == 0.0


def _n_of(n):
    return lambda w: fd.wind_block(n, (w[: n * n], w[n * n: 2 * n * n]))


@pytest.mark.parametrize("ranks,seed", [((1, 1), 0), ((2, 3), 1), ((3, 2), 2)])
def test_kron_sum_equals_definition(ranks, seed):
    rng = np.random.default_rng(seed)
    n, m, p, nt = 4, 2, 2, 3
    H = gpc.h_matrices(m, p)
    u = random_tt(rng, 3 * n * n, len(H), nt, *ranks)
    op = convection_operator(n, len(H), nt, H, *u)
    assert op.T == ranks[0] * ranks[1]
    D = dense_convection(*u, H, _n_of(n))
    A = kron_matrix(op)
    assert abs(D - A).max() <= 1e-14 * abs(D).max()


def test_linear_in_u_and_rank_growth():
    rng = np.random.default_rng(7)
    n, m, p, nt = 3, 1, 3, 4
    H = gpc.h_matrices(m, p)
    u = random_tt(rng, 3 * n * n, len(H), nt, 2, 2)
    v = random_tt(rng, 3 * n * n, len(H), nt, 1, 2)
    w = tt.axpby(1.0, u, 1.0, v)
    A = lambda c: kron_matrix(convection_operator(n, len(H), nt, H, *c))
    assert abs(A(w) - (A(u) + A(v))).max() <= 1e-13 * abs(A(w)).max()
    x = random_tt(rng, 3 * n * n, len(H), nt, 2, 3)
    op = convection_operator(n, len(H), nt, H, *u)
    y = tt.apply_op(op, x)
    assert tt.ranks(y) == (4 * 2, 4 * 3)  # kappa_u^2 terms times the ranks of x
    ref = A(u) @ tt.vec(tt.full(x))
    assert np.linalg.norm(tt.vec(tt.full(y)) - ref) <= 1e-13 * np.linalg.norm(ref)
