"""Pins for the seeded inputs (synth/): gPC Galerkin matrices, FD stencils, term lists."""
import json
import math
import os

import numpy as np
import pytest

from oracle.gpc_quadrature import g_by_quadrature, gauss_legendre_nodes
from synth import fd, gpc
from synth.configs import CONFIGS
from synth.operator import build_operator

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_numbers.json")))


@pytest.mark.parametrize("m,p,n", [(2, 2, 6), (3, 3, 20), (4, 3, 35), (6, 3, 84), (8, 3, 165), (1, 0, 1)])
def test_n_xi_formula(m, p, n):
    # PAPER.md:518 n_xi = (m+d_psi)!/(m! d_psi!)
    assert gpc.n_xi(m, p) == n == len(gpc.multi_indices(m, p))


def test_n_xi_paper_value():
    assert gpc.n_xi(3, 3) == GOLD["n_xi_m3_p3"]["value"]


def test_total_dofs_paper_value():
    g = GOLD["total_dofs"]
    assert g["n_t"] * g["n_xi"] * (g["n_u"] + g["n_p"]) == g["value"]


@pytest.mark.parametrize("m,p", [(2, 2), (3, 3), (4, 3), (1, 4)])
def test_g_closed_form_matches_quadrature(m, p):
    """synth's closed form vs quadrature of the definition <xi_l psi_r psi_s>."""
    idx = gpc.multi_indices(m, p)
    gc = gpc.g_matrices(m, p)
    gq = g_by_quadrature(idx, m, p)
    for l in range(m + 1):
        assert np.max(np.abs(gc[l] - gq[l])) <= 2e-15 * max(1.0, np.max(np.abs(gq[l])))


@pytest.mark.parametrize("m,p", [(2, 2), (4, 3), (8, 3)])
def test_g_structure(m, p):
    gs = gpc.g_matrices(m, p)
    assert np.array_equal(gs[0], np.eye(gpc.n_xi(m, p)))
    for l in range(1, m + 1):
        assert np.array_equal(gs[l], gs[l].T)
        assert np.count_nonzero(gs[l]) == 2 * math.comb(m + p - 1, m)


def test_g1_entry_12():
    # SPEC.md:249 [G_1]_12 = <xi psi_1 psi_2> = 1 with psi_2 = xi (unit variance)
    assert gpc.g_matrices(2, 2)[1][0, 1] == pytest.approx(1.0, abs=1e-15)
    assert gpc.g_matrices(1, 2)[1][0, 1] == pytest.approx(1.0, abs=1e-15)


@pytest.mark.parametrize("p", [1, 2, 3, 5])
def test_g1_eigenvalues_are_scaled_gauss_nodes(p):
    """m=1: G_1 is the Jacobi matrix of the normalised Legendre recurrence in xi = sqrt3 x,
    so eig(G_1) = sqrt3 * roots(P_{p+1})  (Golub-Welsch)."""
    ev = np.sort(np.linalg.eigvalsh(gpc.g_matrices(1, p)[1]))
    ref = np.sort(math.sqrt(3.0) * gauss_legendre_nodes(p + 1))
    assert np.max(np.abs(ev - ref)) <= 1e-14


def test_fd_stencils_exact_on_polynomials():
    n = 12
    xs, ys, h = fd.grid_coords(n)
    u = xs * (1 - xs) * ys * (1 - ys)          # vanishes on the boundary
    lap = fd.laplacian(n) @ u
    assert np.allclose(lap, 2 * ys * (1 - ys) + 2 * xs * (1 - xs), atol=1e-12)
    v = xs * (1 - xs)
    v2 = ys * (1 - ys)
    assert np.allclose(fd.central_dx(n) @ v, 1 - 2 * xs, atol=1e-12)
    assert np.allclose(fd.central_dy(n) @ v2, 1 - 2 * ys, atol=1e-12)
    assert np.allclose(fd.forward_dx(n) @ v, 1 - 2 * xs - h, atol=1e-12)
    L = fd.laplacian(n).toarray()
    assert np.allclose(L, L.T) and np.min(np.linalg.eigvalsh(L)) > 0


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_operator_term_lists(name):
    cfg = CONFIGS[name]
    op = build_operator(cfg)
    assert op.T == cfg.n_terms == {"c1": 4, "c2": 6}[name]
    assert op.n_x == 3 * cfg.grid ** 2 and op.n_xi == gpc.n_xi(cfg.m, cfg.p)
    t0 = op.terms[0].T_dense()
    ref = (np.eye(cfg.n_t) - np.eye(cfg.n_t, k=-1)) / cfg.tau      # (I - C_{n_t})/tau
    assert np.allclose(t0, ref)
    for t in op.terms[1:]:
        assert np.array_equal(t.T_dense(), np.eye(cfg.n_t))
    for t in op.terms:
        assert t.K.indices.dtype == np.int32 and t.K.shape == (op.n_x, op.n_x)


def test_config_term_counts():
    # BASELINE.json: c3 has 9 terms, c4 has 14
    assert CONFIGS["c3"].n_terms == 9 and CONFIGS["c4"].n_terms == 14
