"""NEXT-3: the mean-based preconditioner of PAPER.md section 5 in tensor-train form.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain NumPy/SciPy float64; the sparse
direct solves are scipy's SuperLU (a library primitive standing in for "solve with").

The all-at-once system (eq:ns_sys_all) on the stacked spatial mode
[u1; u2; p] of this repo (R8/R10):

    L = [[F + C, B^T], [B, 0]],     B = I (x) I (x) B,  B = [B1 B2]  (n_p x 2 n_v)

Right preconditioner (eq:prec):  P = [[F + C, B^T], [0, -S]], so

    P^{-1} [v_u; v_p]:   p^ = -S^{-1} v_p,    u^ = (F + C)^{-1} (v_u - B^T p^)

with the two approximations of the paper:
  * S^{-1} ~ S_LSC,0^{-1} = (B M*^-1 B^T)^{-1} (B M*^-1 (F0 + C) M*^-1 B^T) (B M*^-1 B^T)^{-1}
    (eq:mean_lsc); here M = I on the velocity (BASELINE.json configs), so
    M* = I and B M*^-1 B^T = B B^T, a pressure Laplacian;
    F0 + C = tau^-1 (I - C_nt) (x) I (x) M + I (x) I (x) A0 + N0
           = ((I - C_nt) / tau) (x) I (x) I_v  +  I (x) I (x) F0s_v,
    F0s_v = blkdiag(F0s, F0s), F0s = nu0 L + N(w0) the mean convection-diffusion block;
  * (F + C)^{-1} ~ the inner low-rank GMRES on (F0 + C) v = y (eq:11_sys)
    to the relative tolerance tol_in (1e-1), right-preconditioned with
    M = (I - C_nt) (x) I (x) (tau^-1 M + A0 + N(w_avg))   (eq:11_prec)
    whose inverse is (I - C_nt)^{-1} = a cumulative sum over time on the time core and a
    spatial solve with K_s = tau^-1 I + F0s on each velocity component of the space core.
    The synthetic wind is time independent, so w_avg = w0 (R20).

Reading R20 of where the truncations go (the paper truncates every quantity it
forms): every TT op that grows ranks is followed by T_eps:
    1  v_p = Pi_p v                          (restriction to the pressure rows: rank kept)
    2  q1  = (B B^T)^{-1} v_p                (spatial solve: rank kept)
    3  q2  = T(O_S q1),  O_S = B (F0 + C) B^T = ((I-C)/tau) (x) I (x) B B^T + I (x) I (x) B F0s_v B^T
    4  p^  = -(B B^T)^{-1} q2
    5  w   = T(Pi_u v - B^T p^)
    6  u^  = inner GMRES (F0 + C) u^ = w, preconditioner M, z_0 = 0
    7  P^{-1} v = T(u^ + p^)
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import tt
from .convection import Operator, Term


def time_cumsum(x):
    """(I - C_nt)^{-1} on the time mode: C_nt is the unit sub-diagonal shift,
    so (I - C) y = x is y_t = x_t + y_{t-1}, a cumulative sum of every time vector U3[b, :]."""
    return x[0], x[1], np.cumsum(x[2], axis=1)


def restrict_rows(x, lo: int, hi: int):
    """The TT with its space core zeroed outside rows [lo, hi) (a projector on the space mode:
    ranks unchanged)."""
    u1 = np.zeros_like(x[0])
    u1[lo:hi] = x[0][lo:hi]
    return u1, x[1], x[2]


def spatial_solve(x, lu, lo: int, n: int, reps: int = 1):
    """(I (x) I (x) K^{-1}) x restricted to rows [lo, lo + reps n): the n x n factor K (a
    SuperLU object) applied to each of `reps` consecutive diagonal blocks of the space core;
    the other rows of the result are zero.  Ranks unchanged (PAPER.md:244 with X^(3) = K^-1)."""
    u1 = np.zeros_like(x[0])
    for s in range(reps):
        a, b = lo + s * n, lo + (s + 1) * n
        u1[a:b] = lu.solve(np.ascontiguousarray(x[0][a:b]))
    return u1, x[1], x[2]


class MeanLSC:
    """P^{-1} of eq:prec with S_LSC,0 (eq:mean_lsc) and the inner (F0 + C) solve (eq:11_sys,
    eq:11_prec) on the stacked [u1; u2; p] spatial mode.

    F0s (n_v x n_v): the mean convection-diffusion block nu0 L + N(w0) of one velocity
    component; B (n_p x 2 n_v): the divergence [B1 B2]; tau, n_xi, n_t: the discretisation.
    tol: truncation eps of every T; inner: dict(tol, restart, max_cycles) of the inner GMRES.
    schur_inv / f_inv: replace the two approximate solves (the pins plug exact ones in)."""

    def __init__(self, F0s, B, tau: float, n_xi: int, n_t: int, tol: float,
                 inner=None, schur_inv=None, f_inv=None):
        self.n_v = F0s.shape[0]
        self.n_p = B.shape[0]
        self.n_x = 2 * self.n_v + self.n_p
        self.n_xi, self.n_t, self.tau, self.tol = n_xi, n_t, tau, tol
        self.inner = {**dict(tol=1e-1, restart=10, max_cycles=3), **(inner or {})}
        nv, npr, nx = self.n_v, self.n_p, self.n_x
        F0s = sp.csr_matrix(F0s)
        B = sp.csr_matrix(B)
        Bt = B.T.tocsr()
        F0v = sp.block_diag([F0s, F0s], format="csr")
        BBt = (B @ Bt).tocsc()
        BFBt = (B @ F0v @ Bt).tocsr()
        z = lambda m, n: sp.csr_matrix((m, n))
        # embedded spatial factors on the stacked mode
        Iv = sp.block_diag([sp.identity(2 * nv), z(npr, npr)], format="csr")
        F0emb = sp.block_diag([F0v, z(npr, npr)], format="csr")
        S_mass = sp.block_diag([z(2 * nv, 2 * nv), BBt], format="csr")
        S_conv = sp.block_diag([z(2 * nv, 2 * nv), BFBt], format="csr")
        Bt_emb = sp.bmat([[z(2 * nv, 2 * nv), Bt], [z(npr, 2 * nv), z(npr, npr)]], format="csr")
        It, Ix = np.eye(n_t), np.eye(n_xi)
        ImC = np.eye(n_t) - np.eye(n_t, k=-1)
        # F0 + C on the velocity rows
        self.op_F0C = Operator(nx, n_xi, n_t, [Term(ImC / tau, Ix, Iv), Term(It, Ix, F0emb)])
        # O_S = B (F0 + C) B^T on the pressure rows (M* = I)
        self.op_S = Operator(nx, n_xi, n_t, [Term(ImC / tau, Ix, S_mass), Term(It, Ix, S_conv)])
        # B^T: pressure rows -> velocity rows
        self.op_Bt = Operator(nx, n_xi, n_t, [Term(It, Ix, Bt_emb)])
        self.lu_p = spla.splu(BBt)
        Ks = (sp.identity(nv) / tau + F0s).tocsc()   # tau^-1 M + A0 + N(w_avg), M = I
        self.lu_v = spla.splu(Ks)
        self._schur_inv = schur_inv
        self._f_inv = f_inv
        self.inner_stats = []

    # ------------------------------------------------------------------ pieces
    def m_inv(self, x):
        """M^{-1} of eq:11_prec: (I - C)^{-1} on the time core, K_s^{-1} on both velocity
        blocks of the space core (the pressure rows become zero: M acts on the velocity)."""
        return spatial_solve(time_cumsum(x), self.lu_v, 0, self.n_v, reps=2)

    def schur_inv(self, v_p):
        """S_LSC,0^{-1} v_p (eq:mean_lsc, steps 2-3 of R20; positive sign)."""
        if self._schur_inv is not None:
            return self._schur_inv(v_p)
        q1 = spatial_solve(v_p, self.lu_p, 2 * self.n_v, self.n_p)
        q2 = tt.round_tt(tt.apply_op(self.op_S, q1), self.tol)
        return spatial_solve(q2, self.lu_p, 2 * self.n_v, self.n_p)

    def f_inv(self, w):
        """(F + C)^{-1} w ~ inner low-rank GMRES on (F0 + C) u = w with M (step 6 of R20)."""
        if self._f_inv is not None:
            return self._f_inv(w)
        from .gmres import gmres_solve
        res = gmres_solve(self.op_F0C, w, restart=self.inner["restart"],
                          max_cycles=self.inner["max_cycles"], tol=self.tol,
                          tol_gmres=self.inner["tol"], prec=self.m_inv)
        self.inner_stats.append((res["cycles"], res["explicit"][-1] / max(tt.norm(w), 1e-300)))
        if res["z"] is None:
            return tt.zero_tt(self.n_x, self.n_xi, self.n_t)
        return res["z"]

    # ------------------------------------------------------------------ P^{-1}
    def apply(self, v):
        """P^{-1} v, steps 1-7 of R20 (eq:prec block back substitution)."""
        nv2 = 2 * self.n_v
        v_p = restrict_rows(v, nv2, self.n_x)                            # 1
        p_hat = tt.scale(-1.0, self.schur_inv(v_p))                       # 2-4
        v_u = restrict_rows(v, 0, nv2)
        btp = tt.apply_op(self.op_Bt, p_hat)
        w = tt.round_tt(tt.axpby(1.0, v_u, -1.0, btp), self.tol)         # 5
        u_hat = self.f_inv(w)                                             # 6
        return tt.round_tt(tt.axpby(1.0, u_hat, 1.0, p_hat), self.tol)   # 7
