"""Pins of the NEXT-4 oracle (oracle/picard.py, Alg. 1) against things other
than itself: a dense Picard fixed-point iteration on the explicitly assembled all-at-once
Navier-Stokes matrix (eq:ns_sys_all_iter: dense Stokes Kronecker matrix +
the dense per-time-step convection definition sum_l H_l (x) N(u_{h,l}^k), dense direct solves),
the nonlinear residual of eq:ns_sys_all at the converged iterate, and the stopping rule."""
import dataclasses

import numpy as np
import pytest

from oracle import tt
from oracle.convection import dense_convection, n_of
from oracle.kron_dense import kron_matrix
from oracle.picard import picard, residual, system_operator
from synth import gpc
from synth.configs import CONFIGS
from synth.operator import build_operator, convection_stencils, picard_forcing

SMALL = dataclasses.replace(CONFIGS["c7"], grid=3, n_t=3)


def problem(cfg):
    op = build_operator(cfg)
    H = gpc.h_matrices(cfg.m, cfg.p)
    D, nv = convection_stencils(cfg.grid)
    f = picard_forcing(cfg, op.n_xi)
    return op, H, D, nv, f


def dense_N(zvec, H, D, nv, n):
    """N(u) from the DEFINITION for the full coefficient vector u = z."""
    n_x, n_xi, n_t = n
    u = zvec.reshape((n_x, n_xi, n_t), order="F")
    return dense_convection(np.eye(n_x), u, np.eye(n_t), H,
                            lambda w: n_of(w, D, nv, n_x)).toarray()


def dense_picard(S, fvec, H, D, nv, n, iters=80):
    z = np.linalg.solve(S, fvec)  # Stokes (N = 0)
    for _ in range(iters):
        z_new = np.linalg.solve(S + dense_N(z, H, D, nv, n), fvec)
        if np.linalg.norm(z_new - z) <= 1e-14 * np.linalg.norm(z_new):
            return z_new
        z = z_new
    return z


@pytest.fixture(scope="module")
def small():
    op, H, D, nv, f = problem(SMALL)
    n = (op.n_x, op.n_xi, op.n_t)
    S = kron_matrix(op).toarray()
    fvec = tt.vec(tt.full(f))
    zs = dense_picard(S, fvec, H, D, nv, n)
    return op, H, D, nv, f, n, S, fvec, zs


def test_dense_fixed_point_solves_the_nonlinear_system(small):
    """The reference itself: f - (S + N(z*)) z* = 0 (eq:ns_sys_all) to roundoff."""
    op, H, D, nv, f, n, S, fvec, zs = small
    r = fvec - (S + dense_N(zs, H, D, nv, n)) @ zs
    assert np.linalg.norm(r) <= 1e-12 * np.linalg.norm(fvec)
    assert np.linalg.norm(zs[:2 * nv]) > 0.1 * np.linalg.norm(zs)  # a real flow, not p only


def test_system_operator_is_stokes_plus_dense_convection(small):
    """L(z) = stokes + N(T(z)) as a Kronecker sum equals the dense stokes + N(z) definition."""
    op, H, D, nv, f, n, S, fvec, zs = small
    rng = np.random.default_rng(0)
    from synth.tt import random_tt
    z = random_tt(rng, *n, 3, 2)
    L = system_operator(op, z, H, D, nv, 0.0)
    Ld = S + dense_N(tt.vec(tt.full(z)), H, D, nv, n)
    assert np.abs(kron_matrix(L).toarray() - Ld).max() <= 1e-12 * np.abs(Ld).max()


def test_low_rank_picard_converges_to_the_dense_fixed_point(small):
    """Alg. 1 with near-exact truncation (eps 1e-12) reaches z* of the dense iteration."""
    op, H, D, nv, f, n, S, fvec, zs = small
    res = picard(op, H, D, nv, f, tol_picard=1e-11, maxit=60, tol_gmres=1e-3, eps_gmres=1e-13,
                 restart=30, max_cycles=10)
    z = tt.vec(tt.full(res["z"]))
    assert res["residuals"][-1] <= 1e-11 * res["fnorm"]
    assert np.linalg.norm(z - zs) <= 1e-9 * np.linalg.norm(zs)


def test_picard_stopping_rule_and_contraction():
    """c7 (the GPU parity config): the loop stops at the first ||r_i|| <= tol_picard ||f||
    (line 2), the residual contracts every step (a Picard fixed point at this Reynolds
    number), and every inner solve met eq:inexact_solve (||s|| <= tol_gmres ||r||)."""
    cfg = CONFIGS["c7"]
    op, H, D, nv, f = problem(cfg)
    tol_picard, tol_gmres = 1e-3, 1e-1
    res = picard(op, H, D, nv, f, tol_picard=tol_picard, maxit=10, tol_gmres=tol_gmres,
                 eps_gmres=cfg.tol)
    r = np.array(res["residuals"]) / res["fnorm"]
    assert r[-1] <= tol_picard and np.all(r[:-1] > tol_picard)
    assert np.all(np.diff(r) < 0)
    for cycles, expl in res["solves"]:
        assert expl[-1] <= tol_gmres * expl[0] * 1.0000001
    # the final residual, recomputed from the definition (dense), agrees with the TT one
    n = (op.n_x, op.n_xi, op.n_t)
    z = tt.vec(tt.full(res["z"]))
    L = system_operator(op, res["z"], H, D, nv, cfg.tol)
    rd = tt.vec(tt.full(f)) - kron_matrix(L) @ z
    assert abs(np.linalg.norm(rd) - res["residuals"][-1]) <= 2 * cfg.tol * res["fnorm"]
    assert tt.norm(residual(f, L, res["z"], 0.0)) == pytest.approx(np.linalg.norm(rd), rel=1e-10)
