"""Legendre polynomial-chaos basis: multi-index order and closed-form G_l.

PAPER.md:93  — {psi_r} are m-variate orthonormal polynomials, <psi_r psi_s> = delta_rs.
PAPER.md:130-134 — [G_l]_rs = <xi_l psi_r psi_s>, xi_0 == 1.
PAPER.md:414 — psi_1 == 1, hence G_0 = I.
PAPER.md:514-518 — xi_l i.i.d. uniform on [-sqrt3, sqrt3]; total degree <= d_psi;
                   n_xi = (m+d_psi)!/(m! d_psi!).

Univariate factor (reading R13): psi_n(xi) = sqrt(2n+1) P_n(xi/sqrt3).
Three-term recurrence x P_n = ((n+1) P_{n+1} + n P_{n-1})/(2n+1) and <P_n^2> = 1/(2n+1)
under the uniform density on [-1,1] give the only non-zero 1-D moments

    <xi psi_n psi_{n+1}> = sqrt3 (n+1) / sqrt((2n+1)(2n+3)),

so [G_l]_{ab} is that number when multi-indices a, b differ by one in coordinate l
(k = min(a_l, b_l)) and agree elsewhere, and 0 otherwise.  This closed form is an INPUT
(operator descriptor data); tests pin it against Gauss-Legendre quadrature of the
definition (oracle/gpc_quadrature.py).
"""
from __future__ import annotations

import itertools
import math

import numpy as np


def n_xi(m: int, p: int) -> int:
    """Number of basis functions: (m+p)!/(m! p!)."""
    return math.comb(m + p, p)


def multi_indices(m: int, p: int) -> list[tuple[int, ...]]:
    """Graded order: total degree 0,1,..,p; within a degree, descending lexicographic
    (so (1,0,..) precedes (0,1,..) and psi_2 is the degree-1 polynomial in xi_1;
    SPEC.md:220 'graded lexicographic', SPEC.md:249 [G_1]_12 = 1)."""
    out: list[tuple[int, ...]] = []
    for d in range(p + 1):
        level = [a for a in itertools.product(range(d + 1), repeat=m) if sum(a) == d]
        level.sort(reverse=True)
        out.extend(level)
    assert len(out) == n_xi(m, p)
    return out


def g_matrices(m: int, p: int) -> list[np.ndarray]:
    """[G_0, G_1, ..., G_m] as dense float64 n_xi x n_xi arrays (closed form above)."""
    idx = multi_indices(m, p)
    pos = {a: i for i, a in enumerate(idx)}
    n = len(idx)
    gs = [np.eye(n)]
    for l in range(m):
        g = np.zeros((n, n))
        for i, a in enumerate(idx):
            b = list(a)
            b[l] += 1
            j = pos.get(tuple(b))
            if j is None:
                continue
            k = a[l]
            v = math.sqrt(3.0) * (k + 1) / math.sqrt((2 * k + 1) * (2 * k + 3))
            g[i, j] = v
            g[j, i] = v
        gs.append(g)
    return gs


def _triple_1d(a: int, b: int, c: int) -> float:
    """<psi_a psi_b psi_c> in one variable (psi_n = sqrt(2n+1) P_n(xi/sqrt3), xi ~ U[-sqrt3,
    sqrt3]): sqrt((2a+1)(2b+1)(2c+1)) times E[P_a P_b P_c] = (a b c; 0 0 0)^2 (the squared
    Wigner 3j symbol with zero projections; Adams/Neumann closed form):
        s = a+b+c even, |a-b| <= c <= a+b, g = s/2:
        (a b c; 0 0 0)^2 = (s-2a)! (s-2b)! (s-2c)! / (s+1)! * (g! / ((g-a)! (g-b)! (g-c)!))^2
    and 0 otherwise."""
    s = a + b + c
    if s % 2 or c > a + b or c < abs(a - b):
        return 0.0
    g = s // 2
    f = math.factorial
    w2 = (f(s - 2 * a) * f(s - 2 * b) * f(s - 2 * c) / f(s + 1)) * \
        (f(g) / (f(g - a) * f(g - b) * f(g - c))) ** 2
    return math.sqrt((2 * a + 1) * (2 * b + 1) * (2 * c + 1)) * w2


def h_matrices(m: int, p: int) -> list[np.ndarray]:
    """[H_1, ..., H_{n_xi}] with [H_l]_{rs} = <psi_l psi_r psi_s> (the Galerkin
    matrices of a random field expanded in the chaos basis itself, used by the TT convection
    operator eq:N_kron PAPER.md:327), l in the multi_indices order; product of 1-D triple
    products over the m variables.  H_1 = I (psi_1 = 1) and H_{e_i} = G_i (psi_{e_i} = xi_i)."""
    idx = multi_indices(m, p)
    n = len(idx)
    t1 = {}
    out = []
    for lam in idx:
        h = np.zeros((n, n))
        for r, al in enumerate(idx):
            for s_, be in enumerate(idx):
                v = 1.0
                for d in range(m):
                    key = (lam[d], al[d], be[d])
                    if key not in t1:
                        t1[key] = _triple_1d(*key)
                    v *= t1[key]
                    if v == 0.0:
                        break
                h[r, s_] = v
        out.append(h)
    return out
