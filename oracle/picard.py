"""NEXT-4: the inexact Picard iteration of PAPER.md Alg. 1 (alg:picard, :199-213) on the
all-at-once stochastic Galerkin Navier-Stokes system eq:ns_sys_all (:148-156), in TT format.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The system matrix at the iterate u (eq:ns_sys_all_iter, :182-189):
    L(u) = stokes + N(u),   stokes = (I - C)/tau (x) I (x) M + sum_l I (x) G_l (x) A_l + B/B^T
                            (synth.operator.build_stokes_operator: input data),
    N(u) = eq:N_kron (:324-329) built by oracle.convection.convection_operator from the TT
           T_eps_conv(z) of the current iterate z = [u; p] (eq:eps_conv, :331-336: the velocity
           is truncated before the convection matrix is formed; N only reads the velocity rows)
Readings (R21):
    line 1  z_0 = Stokes solve  gmres_solve(stokes, f) with ||s|| <= tol_gmres ||f||   (:538)
            r_0 = T(f - L(z_0) z_0)                                                    (:193)
    line 2  while ||r_i|| > tol_picard ||f|| and i < maxit                            (:544)
    line 4  dz  = gmres_solve(L(z_{i-1}), r_{i-1}) with ||s|| <= tol_gmres ||r_{i-1}|| (eq:inexact_solve)
    line 5  z_i = T(z_{i-1} + dz)
    line 6-7 L(z_i), r_i = T(f - L(z_i) z_i)
    every T at eps_gmres (the paper: eps_gmres = 1e-2 tol_gmres, :537), GMRES restarted every
    `restart` steps with at most `max_cycles` cycles, z_0 = 0 inside each solve, optional right
    preconditioner.
"""
from __future__ import annotations

from . import tt
from .convection import Operator, Term, convection_operator
from .gmres import gmres_solve


def system_operator(stokes, z, H, D, n_v: int, eps_conv: float) -> Operator:
    """L(u) = stokes + N(T_eps_conv(z)) as one Kronecker sum (stokes terms first)."""
    u = tt.round_tt(z, eps_conv)
    conv = convection_operator(u[0], u[1], u[2], H, D, n_v)
    fixed = [Term(t.T_dense(), t.G, t.K) for t in stokes.terms]
    return Operator(stokes.n_x, stokes.n_xi, stokes.n_t, fixed + conv.terms)


def residual(f, L, z, eps: float):
    """r = T_eps(f - L z)  (:190-195)."""
    return tt.round_tt(tt.axpby(1.0, f, -1.0, tt.apply_op(L, z)), eps)


def picard(stokes, H, D, n_v: int, f, tol_picard: float = 1e-5, maxit: int = 10,
           tol_gmres: float = 1e-1, eps_gmres: float = 1e-3, eps_conv: float | None = None,
           restart: int = 20, max_cycles: int = 5, prec=None):
    """Alg. 1.  Returns dict(z, residuals = [||r_0||, ||r_1||, ...], iterations, solves =
    per-linear-solve (cycles, explicit residual history), ranks of every iterate)."""
    eps_conv = eps_gmres if eps_conv is None else eps_conv
    fn = tt.norm(f)
    s = gmres_solve(stokes, f, restart=restart, max_cycles=max_cycles, tol=eps_gmres,
                    tol_gmres=tol_gmres, prec=prec)                                      # line 1
    z = s["z"] if s["z"] is not None else tt.zero_tt(stokes.n_x, stokes.n_xi, stokes.n_t)
    solves = [(s["cycles"], list(s["explicit"]))]
    L = system_operator(stokes, z, H, D, n_v, eps_conv)
    r = residual(f, L, z, eps_gmres)
    res = [tt.norm(r)]
    ranks = [tt.ranks(z)]
    i = 0
    while res[-1] > tol_picard * fn and i < maxit:                                      # line 2
        i += 1
        s = gmres_solve(L, r, restart=restart, max_cycles=max_cycles, tol=eps_gmres,
                        tol_gmres=tol_gmres, prec=prec)                                  # line 4
        solves.append((s["cycles"], list(s["explicit"])))
        if s["z"] is not None:
            z = tt.round_tt(tt.axpby(1.0, z, 1.0, s["z"]), eps_gmres)                     # line 5
        L = system_operator(stokes, z, H, D, n_v, eps_conv)                              # line 6
        r = residual(f, L, z, eps_gmres)                                                 # line 7
        res.append(tt.norm(r))
        ranks.append(tt.ranks(z))
    return dict(z=z, residuals=res, iterations=i, solves=solves, ranks=ranks, fnorm=fn)
