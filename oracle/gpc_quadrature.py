"""G_l from its definition by tensorised Gauss-Legendre quadrature (tests only).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:130-134: [G_l]_rs = <xi_l psi_r psi_s>, xi_0 = 1, expectation over xi uniform on
[-sqrt3, sqrt3]^m.  psi_r = prod_l sqrt(2 a_l + 1) P_{a_l}(xi_l / sqrt3)
(orthonormal Legendre).  Each 1-D factor integrand has degree <= 2p+1,
so q = p + 2 Gauss-Legendre points are exact.  The multi-index list is taken as an argument
so this module shares no arithmetic with synth.gpc.
"""
from __future__ import annotations

import math

import numpy as np
from numpy.polynomial import legendre as npleg


def _psi_1d(n: int, xi: np.ndarray) -> np.ndarray:
    c = np.zeros(n + 1)
    c[n] = 1.0
    return math.sqrt(2 * n + 1) * npleg.legval(xi / math.sqrt(3.0), c)


def g_by_quadrature(indices, m: int, p: int) -> list[np.ndarray]:
    q = p + 2
    x, w = npleg.leggauss(q)      # on [-1, 1]
    w = w / 2.0                   # uniform density 1/2 on [-1, 1]
    xi = math.sqrt(3.0) * x       # nodes for xi uniform on [-sqrt3, sqrt3]
    n = len(indices)
    # 1-D moment tables  <xi^e psi_a psi_b>, e in {0, 1}
    mom = np.zeros((2, p + 1, p + 1))
    for a in range(p + 1):
        for b in range(p + 1):
            pa, pb = _psi_1d(a, xi), _psi_1d(b, xi)
            mom[0, a, b] = np.sum(w * pa * pb)
            mom[1, a, b] = np.sum(w * xi * pa * pb)
    out = []
    for l in range(m + 1):
        g = np.zeros((n, n))
        for r, al in enumerate(indices):
            for s, be in enumerate(indices):
                v = 1.0
                for d in range(m):
                    e = 1 if (l >= 1 and d == l - 1) else 0
                    v *= mom[e, al[d], be[d]]
                g[r, s] = v
        out.append(g)
    return out


def gauss_legendre_nodes(q: int) -> np.ndarray:
    """Roots of P_q (library routine), for the m = 1 eigenvalue pin."""
    return npleg.leggauss(q)[0]


def h_by_quadrature(indices, m: int, p: int) -> list[np.ndarray]:
    """[H_l]_rs = <psi_l psi_r psi_s> for every multi-index l (PAPER.md:132 with the random field
    expanded in the chaos basis, as eq:N_kron PAPER.md:327 uses it), by tensorised
    Gauss-Legendre quadrature: each 1-D integrand has degree <= 3p, q = (3p)//2 + 2 points are
    exact."""
    q = (3 * p) // 2 + 2
    x, w = npleg.leggauss(q)
    w = w / 2.0
    xi = math.sqrt(3.0) * x
    psi = [_psi_1d(a, xi) for a in range(p + 1)]
    t1 = np.zeros((p + 1, p + 1, p + 1))
    for a in range(p + 1):
        for b in range(p + 1):
            for c in range(p + 1):
                t1[a, b, c] = np.sum(w * psi[a] * psi[b] * psi[c])
    n = len(indices)
    out = []
    for lam in indices:
        h = np.zeros((n, n))
        for r, al in enumerate(indices):
            for s, be in enumerate(indices):
                v = 1.0
                for d in range(m):
                    v *= t1[lam[d], al[d], be[d]]
                h[r, s] = v
        out.append(h)
    return out
