"""One cycle of low-rank GMRES (Alg. 3) with P = I (BASELINE.json c5).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Readings (R15):
  * z_0 = 0, s_0 = T(b), beta = ||s_0||, v_1 = s_0 / beta                    (Alg. 3 line 1)
  * x = T(L v_k)                                                             (line 5)
  * modified Gram-Schmidt, h_ik = <x, v_i>, x = T(x - h_ik v_i)  — the config rounds after
    EVERY update (BASELINE.json c5), where Alg. 3 rounds only at lines 5/10/13/14
  * h_{k+1,k} = ||x||, v_{k+1} = x / h_{k+1,k}                                (line 10)
  * least-squares residual |g_{k+1}| from Givens rotations of H-bar after every step (line 12)
  * breakdown when h_{k+1,k} <= 1e-14 ||T(L v_k)||
  * z = sum_i y_i v_i accumulated as z <- T(z + y_i v_i); explicit residual ||T(b - L z)||.
gmres_solve: the complete, restarted Alg. 3 (NEXT-2; reading R19 in its docstring).
Both take an optional right preconditioner (NEXT-3, oracle/precond.py): flexible GMRES.
"""
from __future__ import annotations

import math

import numpy as np

from . import tt


def givens(a: float, b: float):
    if b == 0.0:
        return 1.0, 0.0
    r = math.hypot(a, b)
    return a / r, b / r


def gmres_cycle(op, b, steps: int = 20, tol: float = 1e-6, stop_abs: float = 0.0,
                explicit: bool = True, prec=None):
    """One cycle.  stop_abs > 0: stop once the least-squares residual |g_{k+1}| <= stop_abs
    (Alg. 3 line 2 with the Givens estimate, R19).  explicit=False skips the explicit
    residual T(b - L z) (the restarted solver forms its own).  prec (callable TT -> TT): the
    right preconditioner of Alg. 3 line 4, v^_k = P^{-1} v_k; the flexible variant keeps the
    v^_k and forms z = z_0 + V^_k y_k (lines 11, 13)."""
    s0 = tt.round_tt(b, tol)
    beta = tt.norm(s0)
    v = [tt.scale(1.0 / beta, s0)]
    H = np.zeros((steps + 1, steps))
    cs, sn = [], []
    g = np.zeros(steps + 1)
    g[0] = beta
    hist = [beta]
    ranks = [tt.ranks(v[0])]
    k_done = 0
    vhat = []
    for k in range(steps):
        vh = prec(v[k]) if prec is not None else v[k]                # line 4
        vhat.append(vh)
        x = tt.round_tt(tt.apply_op(op, vh), tol)                     # line 5
        nav = tt.norm(x)
        for i in range(k + 1):
            h = tt.dot(x, v[i])
            H[i, k] = h
            x = tt.round_tt(tt.axpby(1.0, x, -h, v[i]), tol)
        hn = tt.norm(x)
        H[k + 1, k] = hn
        # apply previous rotations to column k, then a new one
        col = H[: k + 2, k].copy()
        for i in range(k):
            t0 = cs[i] * col[i] + sn[i] * col[i + 1]
            col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1]
            col[i] = t0
        c, s = givens(col[k], col[k + 1])
        cs.append(c)
        sn.append(s)
        col[k] = c * col[k] + s * col[k + 1]
        col[k + 1] = 0.0
        H[: k + 2, k] = col
        g[k + 1] = -s * g[k]
        g[k] = c * g[k]
        hist.append(abs(g[k + 1]))
        k_done = k + 1
        if hn <= 1e-14 * nav or hist[-1] <= stop_abs:
            break
        v.append(tt.scale(1.0 / hn, x))
        ranks.append(tt.ranks(v[-1]))
    # least squares solve: H[:k,:k] y = g[:k] (upper triangular after rotations)
    R = H[:k_done, :k_done]
    y = np.linalg.solve(np.triu(R), g[:k_done])
    z = tt.scale(y[0], vhat[0])
    for i in range(1, k_done):
        z = tt.round_tt(tt.axpby(1.0, z, y[i], vhat[i]), tol)
    if not explicit:
        return dict(history=np.array(hist), explicit=None, y=y, z=z, ranks=ranks, steps=k_done)
    r = tt.round_tt(tt.axpby(1.0, b, -1.0, tt.apply_op(op, z)), tol)
    return dict(history=np.array(hist), explicit=tt.norm(r), y=y, z=z, ranks=ranks, steps=k_done)


def gmres_solve(op, b, restart: int = 20, max_cycles: int = 5, tol: float = 1e-6,
                tol_gmres: float = 1e-8, eps_soln: float | None = None, prec=None):
    """Complete low-rank GMRES (NEXT-2): Alg. 3 with P = I,
    restarted every `restart` steps (z_0 <- z), the stopping test ||s_k|| <= tol_gmres ||b||
    (line 2) and the truncated solution update of eq:eps_soln.  Reading
    R19: inside a cycle the test uses the Givens least-squares residual; z_k (line 13, here
    z <- T_eps_soln(z + sum_i y_i v_i)) and the explicit s_k = T(b - L z_k) (line 14) are formed
    at the end of every cycle (and their norm decides the outer stop).  Returns the solution
    TT, the explicit residual norms (s_0 first) and the per-cycle least-squares histories."""
    eps_soln = tol if eps_soln is None else eps_soln
    bnorm = tt.norm(b)
    s = tt.round_tt(b, tol)  # z_0 = 0: s_0 = T(b)
    explicit = [tt.norm(s)]
    ls = []
    z = None
    for _cycle in range(max_cycles):
        if explicit[-1] <= tol_gmres * bnorm:
            break
        res = gmres_cycle(op, s, restart, tol, stop_abs=tol_gmres * bnorm, explicit=False,
                          prec=prec)
        ls.append(res["history"])
        dz = res["z"]
        z = tt.round_tt(dz if z is None else tt.axpby(1.0, z, 1.0, dz), eps_soln)
        s = tt.round_tt(tt.axpby(1.0, b, -1.0, tt.apply_op(op, z)), tol)
        explicit.append(tt.norm(s))
    return dict(z=z, explicit=np.array(explicit), ls=ls, cycles=len(ls))
