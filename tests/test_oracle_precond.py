"""Pins of the NEXT-3 oracle (oracle/precond.py): the mean-based LSC preconditioner and the
inner (F0 + C) solve of PAPER.md section 5, against things other than themselves — dense
solves with the explicitly assembled Kronecker matrices, the paper's two exactness claims
(LSC is exact for F = a multiple of the mass matrix; the ideal block-triangular P makes
right-preconditioned GMRES converge in two iterations), and the
closed-form (I - C)^{-1} (a cumulative sum)."""
import dataclasses

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import tt
from oracle.gmres import gmres_cycle
from oracle.kron_dense import kron_matrix
from oracle.precond import MeanLSC, time_cumsum
from synth.configs import CONFIGS
from synth.operator import build_operator, mean_blocks
from synth.tt import random_tt

# a tiny Oseen config: N = 3 (n_x = 27), m = 1, p = 2 (n_xi = 3), n_t = 4
TINY = dataclasses.replace(CONFIGS["c1"], grid=3, m=1, p=2, n_t=4, tau=0.1, nus=(0.05, 0.01),
                           ranks=(2, 2))


def vec(x):
    return tt.vec(tt.full(x))


def from_vec(v, n_x, n_xi, n_t):
    """A TT of a full vector (Alg. 2 at tol 0: exact)."""
    return tt.tt_svd_dense(v.reshape((n_x, n_xi, n_t), order="F"), 0.0)


@pytest.fixture(scope="module")
def tiny():
    op = build_operator(TINY)
    F0s, B = mean_blocks(TINY)
    A = kron_matrix(op).toarray()
    n_x, n_xi, n_t = op.n_x, op.n_xi, op.n_t
    nv = 2 * TINY.grid ** 2
    idx = np.arange(n_x * n_xi * n_t)
    sx = idx % n_x
    vel, prs = np.where(sx < nv)[0], np.where(sx >= nv)[0]
    return op, F0s, B, A, vel, prs


def test_time_cumsum_is_inverse_of_I_minus_C():
    rng = np.random.default_rng(0)
    x = random_tt(rng, 5, 3, 6, 2, 3)
    n_t = 6
    ImC = np.eye(n_t) - np.eye(n_t, k=-1)
    y = time_cumsum(x)
    ref = sp.kron(sp.csr_matrix(np.linalg.inv(ImC)), sp.identity(5 * 3)) @ vec(x)
    assert np.abs(vec(y) - ref).max() <= 1e-13 * np.abs(ref).max()


def test_m_inv_is_the_solve_with_the_kronecker_M(tiny):
    """eq:11_prec: M = (I - C) (x) I (x) blkdiag(K_s, K_s) on the velocity; M^{-1} x vs a dense
    solve (pressure rows of the result are zero)."""
    op, F0s, B, A, vel, prs = tiny
    P = MeanLSC(F0s, B, TINY.tau, op.n_xi, op.n_t, tol=0.0)
    rng = np.random.default_rng(1)
    x = random_tt(rng, op.n_x, op.n_xi, op.n_t, 2, 2)
    ImC = np.eye(op.n_t) - np.eye(op.n_t, k=-1)
    Ks = np.eye(F0s.shape[0]) / TINY.tau + F0s.toarray()
    M = np.kron(ImC, np.kron(np.eye(op.n_xi), np.block([[Ks, 0 * Ks], [0 * Ks, Ks]])))
    nvv = 2 * F0s.shape[0]
    vmask = (np.arange(op.n_x * op.n_xi * op.n_t) % op.n_x) < nvv
    ref = np.linalg.solve(M, vec(x)[vmask])
    got = vec(P.m_inv(x))
    assert np.abs(got[vmask] - ref).max() <= 1e-12 * np.abs(ref).max()
    assert not np.any(got[~vmask])


def test_lsc_is_exact_when_F_is_the_mass(tiny):
    """With nu = 0 and no wind, F0 + C = ((I - C)/tau) (x) I (x) I_v, and S_LSC,0^{-1} equals the
    true S_0^{-1} = (B (F0 + C)^{-1} B^T)^{-1} (the LSC identity is exact when
    F commutes with B^T B, here F a multiple of the identity in space)."""
    op, F0s, B, A, vel, prs = tiny
    Z = sp.csr_matrix(F0s.shape)
    P = MeanLSC(Z, B, TINY.tau, op.n_xi, op.n_t, tol=0.0)
    ImC = np.eye(op.n_t) - np.eye(op.n_t, k=-1)
    Ix = np.eye(op.n_xi)
    Bd = B.toarray()
    F0C = np.kron(ImC / TINY.tau, np.kron(Ix, np.eye(Bd.shape[1])))
    BB = np.kron(np.eye(op.n_t), np.kron(Ix, Bd))
    S0 = BB @ np.linalg.solve(F0C, BB.T)
    rng = np.random.default_rng(2)
    x = random_tt(rng, op.n_x, op.n_xi, op.n_t, 2, 2)
    from oracle.precond import restrict_rows
    nvv = Bd.shape[1]
    v_p = restrict_rows(x, nvv, op.n_x)
    got = vec(P.schur_inv(v_p))
    pm = (np.arange(op.n_x * op.n_xi * op.n_t) % op.n_x) >= nvv
    ref = np.linalg.solve(S0, vec(v_p)[pm])
    assert np.abs(got[pm] - ref).max() <= 1e-11 * np.abs(ref).max()
    assert not np.any(got[~pm])


def test_ideal_block_triangular_P_converges_in_two_steps(tiny):
    """with the exact (F + C)^{-1} and the exact Schur complement
    S = B (F + C)^{-1} B^T plugged into P = [[F + C, B^T], [0, -S]], right-preconditioned GMRES
    converges in two iterations.  Pins the block back substitution of MeanLSC.apply (the
    restrictions, the sign of S, the B^T coupling) with the flexible oracle GMRES."""
    op, F0s, B, A, vel, prs = tiny
    n = (op.n_x, op.n_xi, op.n_t)
    FC = A[np.ix_(vel, vel)]
    Bb = A[np.ix_(prs, vel)]
    S = Bb @ np.linalg.solve(FC, Bb.T)
    N = A.shape[0]

    def embed(part, idx):
        v = np.zeros(N)
        v[idx] = part
        return from_vec(v, *n)

    f_inv = lambda w: embed(np.linalg.solve(FC, vec(w)[vel]), vel)
    s_inv = lambda v: embed(np.linalg.solve(S, vec(v)[prs]), prs)
    P = MeanLSC(F0s, B, TINY.tau, op.n_xi, op.n_t, tol=1e-14, schur_inv=s_inv, f_inv=f_inv)
    rng = np.random.default_rng(3)
    b = random_tt(rng, *n, 2, 2)
    res = gmres_cycle(op, b, steps=3, tol=1e-14, prec=P.apply)
    h = res["history"]
    assert h[2] <= 1e-9 * h[0], h
    assert res["explicit"] <= 1e-9 * h[0]


def test_apply_inverts_the_dense_block_triangular_P(tiny):
    """eq:prec: P = [[F + C, B^T], [0, -S]] assembled densely; with the exact solves plugged
    in, P (P^{-1} v) = v on every component (pins the sign of S and the B^T coupling, which the
    two-step convergence alone does not: [[F, B^T], [0, +S]] also gives a degree-2 minimal
    polynomial)."""
    op, F0s, B, A, vel, prs = tiny
    n = (op.n_x, op.n_xi, op.n_t)
    FC = A[np.ix_(vel, vel)]
    Bb = A[np.ix_(prs, vel)]
    S = Bb @ np.linalg.solve(FC, Bb.T)
    N = A.shape[0]

    def embed(part, idx):
        v = np.zeros(N)
        v[idx] = part
        return from_vec(v, *n)

    P = MeanLSC(F0s, B, TINY.tau, op.n_xi, op.n_t, tol=0.0,
                f_inv=lambda w: embed(np.linalg.solve(FC, vec(w)[vel]), vel),
                schur_inv=lambda v: embed(np.linalg.solve(S, vec(v)[prs]), prs))
    Pd = np.zeros((N, N))
    Pd[np.ix_(vel, vel)] = FC
    Pd[np.ix_(vel, prs)] = Bb.T
    Pd[np.ix_(prs, prs)] = -S
    rng = np.random.default_rng(8)
    v = random_tt(rng, *n, 2, 3)
    got = Pd @ vec(P.apply(v))
    assert np.abs(got - vec(v)).max() <= 1e-10 * np.abs(vec(v)).max()


def test_inner_solve_meets_its_tolerance(tiny):
    """eq:11_sys with the inner stopping rule ||y - (F0 + C) v|| <= tol ||y||:
    the returned v satisfies it, checked with the dense F0 + C."""
    op, F0s, B, A, vel, prs = tiny
    P = MeanLSC(F0s, B, TINY.tau, op.n_xi, op.n_t, tol=1e-12,
                inner=dict(tol=1e-6, restart=12, max_cycles=6))
    rng = np.random.default_rng(4)
    from oracle.precond import restrict_rows
    w = restrict_rows(random_tt(rng, op.n_x, op.n_xi, op.n_t, 2, 2), 0, 2 * F0s.shape[0])
    u = P.f_inv(w)
    F0C = kron_matrix(P.op_F0C)
    r = vec(w) - F0C @ vec(u)
    assert np.linalg.norm(r) <= 1.01e-6 * np.linalg.norm(vec(w))


def test_flexible_gmres_with_identity_prec_is_unchanged(tiny):
    op, F0s, B, A, vel, prs = tiny
    rng = np.random.default_rng(5)
    b = random_tt(rng, op.n_x, op.n_xi, op.n_t, 2, 2)
    r0 = gmres_cycle(op, b, steps=4, tol=1e-10)
    r1 = gmres_cycle(op, b, steps=4, tol=1e-10, prec=lambda v: v)
    assert np.array_equal(r0["history"], r1["history"])


def test_mean_lsc_accelerates_gmres(tiny):
    """The practical P (LSC + inner GMRES at tol 1e-1) reduces the residual faster than no
    preconditioner on the tiny Oseen problem (the purpose of PAPER.md section 5)."""
    op, F0s, B, A, vel, prs = tiny
    rng = np.random.default_rng(6)
    b = random_tt(rng, op.n_x, op.n_xi, op.n_t, 2, 2)
    P = MeanLSC(F0s, B, TINY.tau, op.n_xi, op.n_t, tol=1e-10)
    hp = gmres_cycle(op, b, steps=6, tol=1e-10, prec=P.apply)["history"]
    h0 = gmres_cycle(op, b, steps=6, tol=1e-10)["history"]
    assert hp[-1] < 0.5 * h0[-1]
