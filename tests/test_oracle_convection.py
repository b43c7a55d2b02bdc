"""NEXT-1: the TT-format convection operator N(u) of eq:N_kron.

Pins, all -m "not gpu":
  * H_l closed form (synth.gpc.h_matrices, Wigner-3j product) vs Gauss-Legendre quadrature of
    the definition <psi_l psi_r psi_s> (oracle.gpc_quadrature.h_by_quadrature); H_1 = I
    (psi_1 = 1); H_{e_i} = G_i (psi_{e_i} = xi_i); symmetry; parity selection;
  * the Kronecker-sum operator (oracle.convection.convection_operator, alpha sums of eq:N_kron)
    vs the dense block definition sum_l H_l (x) N(u_{h,l}^k) per time step (oracle.convection);
  * the spatial N(w) (oracle.convection.n_of) vs the convective derivative w . grad f of
    quadratic fields (central differences are exact on quadratics) on every velocity component;
  * linearity in u and the kappa -> kappa^2 rank growth of the apply.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import gpc_quadrature as gq
from oracle import tt
from oracle.convection import convection_operator, dense_convection, n_of
from oracle.kron_dense import kron_matrix
from synth import fd, gpc
from synth.operator import convection_stencils
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


def _conv(n, H, u):
    D, n_v = convection_stencils(n)
    return convection_operator(*u, H, D, n_v), (lambda w: n_of(w, D, n_v, 3 * n_v))


def test_n_of_is_the_convective_derivative():
    """[N(w) f]_i = w1_i df/dx + w2_i df/dy at nodes whose 4 neighbours are interior, for a
    quadratic f on each velocity component (and zero on the pressure rows)."""
    n = 7
    D, n_v = convection_stencils(n)
    xs, ys, _ = fd.grid_coords(n)
    rng = np.random.default_rng(3)
    w = rng.standard_normal(3 * n_v)
    f = xs ** 2 + 3 * xs * ys - ys          # df/dx = 2x + 3y, df/dy = 3x - 1
    g = -2 * ys ** 2 + xs * ys + 0.5 * xs   # dg/dx = y + 0.5,  dg/dy = -4y + x
    v = np.concatenate([f, g, rng.standard_normal(n_v)])
    out = n_of(w, D, n_v, 3 * n_v) @ v
    ix, iy = np.arange(n_v) % n, np.arange(n_v) // n
    inner = (ix > 0) & (ix < n - 1) & (iy > 0) & (iy < n - 1)
    w1, w2 = w[:n_v], w[n_v:2 * n_v]
    ref_f = w1 * (2 * xs + 3 * ys) + w2 * (3 * xs - 1)
    ref_g = w1 * (ys + 0.5) + w2 * (-4 * ys + xs)
    assert np.abs(out[:n_v][inner] - ref_f[inner]).max() <= 1e-11
    assert np.abs(out[n_v:2 * n_v][inner] - ref_g[inner]).max() <= 1e-11
    assert not np.any(out[2 * n_v:])


@pytest.mark.parametrize("ranks,seed", [((1, 1), 0), ((2, 3), 1), ((3, 2), 2)])
def test_kron_sum_equals_definition(ranks, seed):
    rng = np.random.default_rng(seed)
    n, m, p, nt = 4, 2, 2, 3
    H = gpc.h_matrices(m, p)
    u = random_tt(rng, 3 * n * n, len(H), nt, *ranks)
    op, N_of = _conv(n, H, u)
    assert op.T == ranks[0] * ranks[1]
    D = dense_convection(*u, H, N_of)
    A = kron_matrix(op)
    assert abs(D - A).max() <= 1e-14 * abs(D).max()


def test_linear_in_u_and_rank_growth():
    rng = np.random.default_rng(7)
    n, m, p, nt = 3, 1, 3, 4
    H = gpc.h_matrices(m, p)
    u = random_tt(rng, 3 * n * n, len(H), nt, 2, 2)
    v = random_tt(rng, 3 * n * n, len(H), nt, 1, 2)
    w = tt.axpby(1.0, u, 1.0, v)
    A = lambda c: kron_matrix(_conv(n, H, c)[0])
    assert abs(A(w) - (A(u) + A(v))).max() <= 1e-13 * abs(A(w)).max()
    x = random_tt(rng, 3 * n * n, len(H), nt, 2, 3)
    op = _conv(n, H, u)[0]
    y = tt.apply_op(op, x)
    assert tt.ranks(y) == (4 * 2, 4 * 3)  # kappa_u^2 terms times the ranks of x
    ref = A(u) @ tt.vec(tt.full(x))
    assert np.linalg.norm(tt.vec(tt.full(y)) - ref) <= 1e-13 * np.linalg.norm(ref)
