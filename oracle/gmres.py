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


def gmres_cycle(op, b, steps: int = 20, tol: float = 1e-6):
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
    for k in range(steps):
        x = tt.round_tt(tt.apply_op(op, v[k]), tol)
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
        if hn <= 1e-14 * nav:
            break
        v.append(tt.scale(1.0 / hn, x))
        ranks.append(tt.ranks(v[-1]))
    # least squares solve: H[:k,:k] y = g[:k] (upper triangular after rotations)
    R = H[:k_done, :k_done]
    y = np.linalg.solve(np.triu(R), g[:k_done])
    z = tt.scale(y[0], v[0])
    for i in range(1, k_done):
        z = tt.round_tt(tt.axpby(1.0, z, y[i], v[i]), tol)
    r = tt.round_tt(tt.axpby(1.0, b, -1.0, tt.apply_op(op, z)), tol)
    return dict(history=np.array(hist), explicit=tt.norm(r), y=y, z=z, ranks=ranks, steps=k_done)
