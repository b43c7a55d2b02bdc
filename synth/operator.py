"""Kronecker-sum operator descriptor  A = sum_k T_k (x) G_k (x) K_k.

PAPER.md:157-161 (eq:F) and :453: every block of the all-at-once system is a sum of
triple Kronecker products time (x) stochastic (x) space.  The term list of the synthetic
configs (R8):

  k=0        time-mass   T_0 = (I - C_{n_t})/tau  (x) G_0 = I (x) blkdiag(I, I, 0)
  k=1        mean Oseen  I (x) G_0 (x) [[nu0 L + N(w0), 0, B1^T], [0, nu0 L + N(w0), B2^T], [B1, B2, 0]]
  k=2..m+1   KL terms    I (x) G_l (x) blkdiag(nu_l L, nu_l L, 0)           l = 1..m
  then       wind terms  I (x) G_j (x) blkdiag(N(w_j), N(w_j), 0)           j = 1..R_w-1

T_0 merges tau^{-1} I (x) I (x) M with the all-at-once shift  C = -tau^{-1} C_{n_t} (x) I (x) M
(PAPER.md:157).  T_k are banded (stored LAPACK general-band, column major), G_k dense,
K_k CSR with int32 indices — the descriptor of BASELINE.json:5.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import fd, gpc
from .configs import Config


@dataclass
class Term:
    name: str
    kl: int                 # sub-diagonals of T_k
    ku: int                 # super-diagonals of T_k
    band: np.ndarray        # (kl+ku+1, n_t) LAPACK band: band[ku + i - j, j] = T[i, j]
    G: np.ndarray           # (n_xi, n_xi) dense
    K: sp.csr_matrix        # (n_x, n_x) CSR, int32 indices, sorted

    def T_dense(self) -> np.ndarray:
        n = self.band.shape[1]
        t = np.zeros((n, n))
        for j in range(n):
            for i in range(max(0, j - self.ku), min(n, j + self.kl + 1)):
                t[i, j] = self.band[self.ku + i - j, j]
        return t


@dataclass
class KronSumOp:
    n_x: int
    n_xi: int
    n_t: int
    terms: list

    @property
    def T(self) -> int:
        return len(self.terms)


def band_identity(n: int) -> tuple[int, int, np.ndarray]:
    return 0, 0, np.ones((1, n))


def band_backward_euler(n: int, tau: float) -> tuple[int, int, np.ndarray]:
    """(I - C_n)/tau: 1/tau on the diagonal, -1/tau on the sub-diagonal."""
    band = np.zeros((2, n))
    band[0, :] = 1.0 / tau
    band[1, : n - 1] = -1.0 / tau
    return 1, 0, band


def _csr32(k: sp.csr_matrix) -> sp.csr_matrix:
    k = sp.csr_matrix(k)
    k.sum_duplicates()
    k.eliminate_zeros()
    k.sort_indices()
    k.indices = k.indices.astype(np.int32)
    k.indptr = k.indptr.astype(np.int32)
    return k


def build_operator(cfg: Config) -> KronSumOp:
    if cfg.operator == "picard":
        return build_stokes_operator(cfg)
    if cfg.operator == "convection":
        raise ValueError("the convection operator is built by the library (tk_op_convection) "
                         "or by oracle.convection from synth.operator.convection_stencils")
    rng = np.random.default_rng([cfg.index, 0])
    n = cfg.grid
    winds = [fd.sinusoid_wind(n, rng, scale=0.5 ** j) for j in range(cfg.wind_rank)]
    gs = gpc.g_matrices(cfg.m, cfg.p)
    nxi = gs[0].shape[0]
    terms = []
    kl, ku, b = band_backward_euler(cfg.n_t, cfg.tau)
    terms.append(Term("time-mass", kl, ku, b, gs[0], _csr32(fd.mass_block(n))))
    kl, ku, b = band_identity(cfg.n_t)
    terms.append(Term("oseen", kl, ku, b, gs[0], _csr32(fd.oseen_block(n, cfg.nus[0], winds[0]))))
    for l in range(1, cfg.m + 1):
        kl, ku, b = band_identity(cfg.n_t)
        terms.append(Term(f"kl{l}", kl, ku, b, gs[l], _csr32(fd.viscous_block(n, cfg.nus[l]))))
    for j in range(1, cfg.wind_rank):
        kl, ku, b = band_identity(cfg.n_t)
        terms.append(Term(f"wind{j}", kl, ku, b, gs[j], _csr32(fd.wind_block(n, winds[j]))))
    op = KronSumOp(cfg.n_x, nxi, cfg.n_t, terms)
    assert op.T == cfg.n_terms
    return op


def random_operator(rng: np.random.Generator, n_x: int, n_xi: int, n_t: int, T: int,
                    density: float = 0.3, max_band: int = 2) -> KronSumOp:
    """Small random descriptor for parity tests (random sparse K, dense G, banded T)."""
    terms = []
    for k in range(T):
        kl = int(rng.integers(0, max_band + 1))
        ku = int(rng.integers(0, max_band + 1))
        band = rng.standard_normal((kl + ku + 1, n_t))
        g = rng.standard_normal((n_xi, n_xi))
        kmat = sp.random(n_x, n_x, density=density, random_state=rng, format="csr",
                         data_rvs=rng.standard_normal)
        terms.append(Term(f"rand{k}", kl, ku, band, g, _csr32(kmat)))
    return KronSumOp(n_x, n_xi, n_t, terms)


def convection_stencils(n: int):
    """The discretisation data of the convection operator (input data, no method arithmetic):
    the central-difference operators (D_x, D_y) on the N x N velocity grid and n_v = N^2 dofs
    per velocity component; the spatial mode is [u1; u2; p] (R10).  N(w) itself is
    formed by the library (tk_conv_create / tk_op_convection) and by oracle.convection."""
    return [_csr32(fd.central_dx(n)), _csr32(fd.central_dy(n))], n * n


def mean_blocks(cfg: Config):
    """Input data of the mean-based preconditioner (NEXT-3, section 5) for an Oseen
    config: the mean convection-diffusion block F0s = nu_0 L + N(w_0) of ONE velocity component
    (the same w_0 as build_operator's mean Oseen term) and the divergence B = [B1 B2]
    (n_p x 2 n_v).  Returns (F0s, B) as CSR; no preconditioner arithmetic."""
    rng = np.random.default_rng([cfg.index, 0])
    n = cfg.grid
    if cfg.operator == "picard":  # no fixed wind: the Stokes mean block (w_avg = 0, R21)
        f0 = _csr32(cfg.nus[0] * fd.laplacian(n))
        b = _csr32(sp.hstack([fd.forward_dx(n), fd.forward_dy(n)]))
        return f0, b
    winds = [fd.sinusoid_wind(n, rng, scale=0.5 ** j) for j in range(cfg.wind_rank)]
    f0 = _csr32(cfg.nus[0] * fd.laplacian(n) + fd.convection(n, *winds[0]))
    b = _csr32(sp.hstack([fd.forward_dx(n), fd.forward_dy(n)]))
    return f0, b


def build_stokes_operator(cfg: Config) -> KronSumOp:
    """The fixed part of the all-at-once Navier-Stokes matrix (eq:ns_sys_all, eq:F without
    N(u)): time-mass (I - C)/tau (x) I (x) blkdiag(I, I, 0), the mean Stokes block
    I (x) G_0 (x) [[nu0 L, 0, B1^T], [0, nu0 L, B2^T], [B1, B2, 0]] and the KL terms
    I (x) G_l (x) blkdiag(nu_l L, nu_l L, 0) — the Stokes operator of Alg. 1 line 1
    (PAPER.md:197).  The convection N(u) of the current iterate is added by the Picard driver."""
    n = cfg.grid
    gs = gpc.g_matrices(cfg.m, cfg.p)
    nxi = gs[0].shape[0]
    zero = np.zeros(n * n)
    terms = []
    kl, ku, b = band_backward_euler(cfg.n_t, cfg.tau)
    terms.append(Term("time-mass", kl, ku, b, gs[0], _csr32(fd.mass_block(n))))
    kl, ku, b = band_identity(cfg.n_t)
    terms.append(Term("stokes", kl, ku, b, gs[0],
                      _csr32(fd.oseen_block(n, cfg.nus[0], (zero, zero)))))
    for l in range(1, cfg.m + 1):
        kl, ku, b = band_identity(cfg.n_t)
        terms.append(Term(f"kl{l}", kl, ku, b, gs[l], _csr32(fd.viscous_block(n, cfg.nus[l]))))
    return KronSumOp(cfg.n_x, nxi, cfg.n_t, terms)


def picard_forcing(cfg: Config, n_xi: int, amp: float = 1.0):
    """Right-hand side f = [f^u; f^p] of eq:ns_sys_all for the Picard problem (input data):
    a seeded smooth body force in the mean chaos mode, constant in time, f^p = 0 — rank (1, 1).
    f^u_c = amp * sum of 3 random sinusoids (the wind recipe of DESIGN.md R11)."""
    rng = np.random.default_rng([cfg.index, 4])
    n = cfg.grid
    f1, f2 = fd.sinusoid_wind(n, rng)
    u1 = np.concatenate([f1, f2, np.zeros(n * n)])[:, None] * amp
    u2 = np.zeros((1, n_xi, 1))
    u2[0, 0, 0] = 1.0
    u3 = np.ones((1, cfg.n_t))
    return u1, u2, u3
