"""Seeded input tensor trains (north-star core order, R1).

A TT is a plain tuple (U1, U2, U3) of float64 arrays:
  U1: (n_x, r1)          space core       (paper's z^(3) transposed)
  U2: (r1, n_xi, r2)     stochastic core  (paper's z^(2) with bond indices swapped)
  U3: (r2, n_t)          time core        (paper's z^(1) transposed)
X(i_x, i_xi, i_t) = sum_{a,b} U1[i_x,a] U2[a,i_xi,b] U3[b,i_t];  vec(X) runs space fastest
(PAPER.md:224-227).

Recipes (R14):
  "gauss": all cores N(0,1).
  "decay": U1 = orth(N(0,1)_{n_x x r1}) diag(0.7^i),  U3 = diag(0.7^j) orth_rows(N(0,1)_{r2 x n_t}),
           U2 ~ N(0,1).   (orth via numpy QR: input preparation, not the method.)
Seeds: numpy default_rng([config index, 1]).
"""
from __future__ import annotations

import numpy as np

from .configs import Config


def _orth_cols(a: np.ndarray) -> np.ndarray:
    q, _ = np.linalg.qr(a)
    return q


def random_tt(rng: np.random.Generator, n_x: int, n_xi: int, n_t: int, r1: int, r2: int,
              kind: str = "gauss"):
    if kind == "gauss":
        u1 = rng.standard_normal((n_x, r1))
        u2 = rng.standard_normal((r1, n_xi, r2))
        u3 = rng.standard_normal((r2, n_t))
        return u1, u2, u3
    if kind == "decay":
        u1 = _orth_cols(rng.standard_normal((n_x, r1)))
        u1 = u1 * (0.7 ** np.arange(u1.shape[1]))[None, :]
        if u1.shape[1] < r1:  # n_x < r1: pad (not used by the named configs)
            u1 = np.concatenate([u1, np.zeros((n_x, r1 - u1.shape[1]))], axis=1)
        u3 = _orth_cols(rng.standard_normal((n_t, r2))).T
        u3 = u3 * (0.7 ** np.arange(u3.shape[0]))[:, None]
        if u3.shape[0] < r2:
            u3 = np.concatenate([u3, np.zeros((r2 - u3.shape[0], n_t))], axis=0)
        u2 = rng.standard_normal((r1, n_xi, r2))
        return np.ascontiguousarray(u1), u2, np.ascontiguousarray(u3)
    raise ValueError(kind)


def make_input_tt(cfg: Config, n_xi: int):
    rng = np.random.default_rng([cfg.index, 1])
    return random_tt(rng, cfg.n_x, n_xi, cfg.n_t, cfg.ranks[0], cfg.ranks[1], cfg.input_kind)


def make_rhs_tt(cfg: Config, n_xi: int):
    """c5 right-hand side: N(0,1) cores of ranks rhs_ranks, each core scaled to unit
    Frobenius norm (a data-only normalisation; R15)."""
    rng = np.random.default_rng([cfg.index, 2])
    u1, u2, u3 = random_tt(rng, cfg.n_x, n_xi, cfg.n_t, cfg.rhs_ranks[0], cfg.rhs_ranks[1], "gauss")
    return u1 / np.linalg.norm(u1), u2 / np.linalg.norm(u2), u3 / np.linalg.norm(u3)


def make_velocity_tt(cfg: Config, n_xi: int):
    """c6 velocity u~ for the convection operator N(u~): decaying cores of ranks velocity_ranks
    (the low-rank truncation T_eps_conv(u) of eq:eps_conv stands behind it),
    scaled so the wind has O(1) magnitude on the grid."""
    rng = np.random.default_rng([cfg.index, 3])
    u1, u2, u3 = random_tt(rng, cfg.n_x, n_xi, cfg.n_t, cfg.velocity_ranks[0],
                           cfg.velocity_ranks[1], "decay")
    return u1 * np.sqrt(cfg.n_x / 3.0), u2 / np.linalg.norm(u2), u3 * np.sqrt(cfg.n_t)
