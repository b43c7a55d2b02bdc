"""Tensor-train arithmetic of PAPER.md section 4.1, plain NumPy/SciPy float64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

A TT is a tuple (U1, U2, U3): U1 (n_x, r1), U2 (r1, n_xi, r2), U3 (r2, n_t); the represented
tensor is X(i_x,i_xi,i_t) = sum_{a,b} U1[i_x,a] U2[a,i_xi,b] U3[b,i_t] (PAPER.md:228-232 eq:z_tt
with the core order reversed to (space, stoch, time), R1), and vec(X) runs space
fastest.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.linalg as sla


# ----------------------------------------------------------------------------- basics
def ranks(x):
    return x[0].shape[1], x[2].shape[0]


def full(x) -> np.ndarray:
    """Entrywise evaluation of eq:z_tt."""
    u1, u2, u3 = x
    return np.einsum("xa,aib,bt->xit", u1, u2, u3)


def vec(xfull: np.ndarray) -> np.ndarray:
    """vec with i_x fastest, then i_xi, then i_t."""
    return xfull.reshape(-1, order="F")


def storage(x) -> int:
    """Number of stored entries n_x r1 + r1 n_xi r2 + r2 n_t."""
    return x[0].size + x[1].size + x[2].size


def zero_tt(n_x: int, n_xi: int, n_t: int):
    """Canonical zero tensor: ranks (1,1), zero cores (R17)."""
    return np.zeros((n_x, 1)), np.zeros((1, n_xi, 1)), np.zeros((1, n_t))


# ----------------------------------------------------------------------------- apply
def apply_op(op, x):
    """y = A x with A = sum_k T_k (x) G_k (x) K_k   (eq:Xz).

    Each term maps the cores factor by factor, "with the same ranks as in z":
    K_k U1, G_k x_2 U2, U3 T_k^T.  The sum over k concatenates the cores
    ("additions ... increase the ranks"): U1 side by side, U2 block
    diagonal, U3 stacked.  Output ranks (T r1, T r2).
    """
    u1, u2, u3 = x
    r1, r2 = u1.shape[1], u3.shape[0]
    T = len(op.terms)
    n_xi = u2.shape[1]
    y1 = np.zeros((u1.shape[0], T * r1))
    y2 = np.zeros((T * r1, n_xi, T * r2))
    y3 = np.zeros((T * r2, u3.shape[1]))
    for k, term in enumerate(op.terms):
        y1[:, k * r1:(k + 1) * r1] = term.K @ u1
        y2[k * r1:(k + 1) * r1, :, k * r2:(k + 1) * r2] = np.einsum("ij,ajb->aib", term.G, u2)
        y3[k * r2:(k + 1) * r2, :] = u3 @ term.T_dense().T
    return y1, y2, y3


# ----------------------------------------------------------------------------- rounding
def rank_rule(sigma: np.ndarray, delta: float, rmax: int = 0) -> int:
    """Smallest r >= 1 with (sum_{j>r} sigma_j^2)^{1/2} <= delta  (Alg. 2
    line 4 ||E||_F <= delta_j); values tied with the last kept one are kept;
    then min(r, rmax) when rmax > 0 (BASELINE.json:5; R4)."""
    s = np.asarray(sigma, dtype=np.float64)
    n = s.size
    if n == 0:
        return 1
    tail = np.sqrt(np.cumsum((s ** 2)[::-1])[::-1])  # tail[r] = ||sigma[r:]||
    r = n
    for cand in range(1, n + 1):
        rest = tail[cand] if cand < n else 0.0
        if rest <= delta:
            r = cand
            break
    while r < n and s[r] == s[r - 1]:
        r += 1
    if rmax and rmax > 0:
        r = min(r, rmax)
    return max(r, 1)


def round_tt(x, tol: float, rmax: int = 0, return_info: bool = False):
    """TT truncation T_eps: result x~ with ||x~ - x||_F <= eps ||x||_F,
    using delta_1 = delta_2 = eps ||x||_F / sqrt(d-1), d = 3, computed on
    the cores only in the north-star direction (R2): a right-to-left
    QR sweep over the small cores, then truncated SVDs left to right (space bond first).

    Steps:
      1  Q3^T, L3^T = qr(Y3^T)                      (time core)
      2  Y2 <- Y2 x_3 L3
      3  Q2^T, L2^T = qr(Y2_(1)^T),  Y2_(1) = reshape(Y2, R1, n_xi k3)
      4  Q1, R_Y = qr(Y1)                           (LAPACK Householder)
      5  M = R_Y L2
      6  delta = tol ||M||_F / sqrt(2),  ||M||_F = ||x||_F
      7  U, s, V^T = svd(M);  r1 = rank_rule(s, delta, rmax)
      8  U1' = Q1 U[:, :r1]
      9  C = (diag(s) V^T)[:r1] Q2  -> (r1, n_xi, k3)
     10  U, s', V^T = svd(reshape(C, r1 n_xi, k3));  r2 = rank_rule(s', delta, rmax)
     11  U2' = reshape(U[:, :r2], r1, n_xi, r2),  U3' = (diag(s') V^T)[:r2] Q3
    """
    if tol < 0:
        raise ValueError("tol must be >= 0")
    y1, y2, y3 = x
    n_x, R1 = y1.shape
    R2, n_t = y3.shape
    n_xi = y2.shape[1]
    # 1
    q, r = np.linalg.qr(y3.T, mode="reduced")        # y3.T = q r
    q3, l3 = q.T, r.T                                 # y3 = l3 q3
    k3 = q3.shape[0]
    # 2
    y2 = np.einsum("aib,bc->aic", y2, l3)
    # 3
    y2m = y2.reshape(R1, n_xi * k3)
    q, r = np.linalg.qr(y2m.T, mode="reduced")
    q2, l2 = q.T, r.T                                 # y2m = l2 q2
    # 4
    q1, ry = np.linalg.qr(y1, mode="reduced")
    # 5
    m = ry @ l2
    nrm = np.linalg.norm(m)
    if nrm == 0.0:
        z = zero_tt(n_x, n_xi, n_t)
        info = dict(norm=0.0, delta=0.0, sigma1=np.zeros(1), sigma2=np.zeros(1), ranks=(1, 1))
        return (z, info) if return_info else z
    # 6
    delta = tol * nrm / math.sqrt(2.0)
    # 7
    u, s, vt = sla.svd(m, full_matrices=False, lapack_driver="gesvd")
    r1 = rank_rule(s, delta, rmax)
    # 8
    u1n = q1 @ u[:, :r1]
    # 9
    c = (s[:r1, None] * vt[:r1]) @ q2
    c = c.reshape(r1 * n_xi, k3)
    # 10
    u_, s2, vt2 = sla.svd(c, full_matrices=False, lapack_driver="gesvd")
    r2 = rank_rule(s2, delta, rmax)
    # 11
    u2n = u_[:, :r2].reshape(r1, n_xi, r2)
    u3n = (s2[:r2, None] * vt2[:r2]) @ q3
    out = (u1n, u2n, u3n)
    if return_info:
        info = dict(norm=nrm, delta=delta, sigma1=s, sigma2=s2, ranks=(r1, r2),
                    discarded=(float(np.linalg.norm(s[r1:])), float(np.linalg.norm(s2[r2:]))))
        return out, info
    return out


def tt_svd_dense(xfull: np.ndarray, tol: float, rmax: int = 0):
    """Alg. 2 (TT-SVD) on a full n_x x n_xi x n_t tensor, splitting the
    space mode first (north-star order), delta_j = tol ||X||_F / sqrt(2)."""
    n_x, n_xi, n_t = xfull.shape
    nrm = np.linalg.norm(xfull)
    if nrm == 0.0:
        return zero_tt(n_x, n_xi, n_t)
    delta = tol * nrm / math.sqrt(2.0)
    z = xfull.reshape(n_x, n_xi * n_t)                               # line 3, j=1
    u, s, vt = sla.svd(z, full_matrices=False, lapack_driver="gesvd")  # line 4
    k1 = rank_rule(s, delta, rmax)
    core1 = u[:, :k1]                                                 # line 5
    z = s[:k1, None] * vt[:k1]                                        # line 6
    z = z.reshape(k1 * n_xi, n_t)                                     # line 3, j=2
    u, s, vt = sla.svd(z, full_matrices=False, lapack_driver="gesvd")
    k2 = rank_rule(s, delta, rmax)
    core2 = u[:, :k2].reshape(k1, n_xi, k2)
    core3 = s[:k2, None] * vt[:k2]                                    # line 8
    return core1, core2, core3


# ----------------------------------------------------------------------------- dot / axpby
def dot(x, y) -> float:
    """<x, y>_F contracted core by core ("inner products"):
    W1 = X1^T Y1;  W2 = sum_i X2[:,i,:]^T W1 Y2[:,i,:];  <x,y> = sum W2 .* (X3 Y3^T)."""
    w1 = x[0].T @ y[0]
    w2 = np.zeros((x[1].shape[2], y[1].shape[2]))
    for i in range(x[1].shape[1]):
        w2 += x[1][:, i, :].T @ w1 @ y[1][:, i, :]
    return float(np.sum(w2 * (x[2] @ y[2].T)))


def norm(x) -> float:
    """||x||_F = ||vec x||_2, via sqrt(<x,x>)."""
    return math.sqrt(max(dot(x, x), 0.0))


def axpby(a: float, x, b: float, y):
    """a x + b y by core concatenation: U1 = [x1 | y1],
    U2 = blockdiag(x2, y2), U3 = [a x3; b y3]; ranks add."""
    (x1, x2, x3), (y1, y2, y3) = x, y
    if x1.shape[0] != y1.shape[0] or x2.shape[1] != y2.shape[1] or x3.shape[1] != y3.shape[1]:
        raise ValueError("mode size mismatch")
    r1 = x1.shape[1] + y1.shape[1]
    r2 = x3.shape[0] + y3.shape[0]
    u1 = np.concatenate([x1, y1], axis=1)
    u2 = np.zeros((r1, x2.shape[1], r2))
    u2[: x1.shape[1], :, : x3.shape[0]] = x2
    u2[x1.shape[1]:, :, x3.shape[0]:] = y2
    u3 = np.concatenate([a * x3, b * y3], axis=0)
    return u1, u2, u3


def scale(a: float, x):
    """a x: scale the time core."""
    return x[0], x[1], a * x[2]
