"""Pins of the CPU oracle (oracle/tt.py) against things other than itself:
explicit Kronecker matvecs, dense TT-SVD (Alg. 2), closed-form spectra, invariants."""
import json
import math
import os

import numpy as np
import pytest

from oracle import tt
from oracle.kron_dense import kron_matrix
from synth.configs import CONFIGS
from synth.operator import build_operator, random_operator, KronSumOp, Term, band_identity
from synth.tt import make_input_tt, random_tt
import scipy.sparse as sp

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_numbers.json")))


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def c1():
    cfg = CONFIGS["c1"]
    op = build_operator(cfg)
    x = make_input_tt(cfg, op.n_xi)
    return cfg, op, x


# ----------------------------------------------------------------------------- apply
def test_apply_matches_explicit_kron_c1(c1):
    cfg, op, x = c1
    y = tt.apply_op(op, x)
    assert tt.ranks(y) == (op.T * 4, op.T * 4)
    ref = kron_matrix(op) @ tt.vec(tt.full(x))
    assert rel(tt.vec(tt.full(y)), ref) <= 1e-14


@pytest.mark.parametrize("seed", range(6))
def test_apply_matches_explicit_kron_random(seed):
    rng = np.random.default_rng(seed)
    n_x, n_xi, n_t = rng.integers(2, 9, size=3)
    T = int(rng.integers(1, 5))
    op = random_operator(rng, int(n_x), int(n_xi), int(n_t), T)
    x = random_tt(rng, n_x, n_xi, n_t, int(rng.integers(1, 4)), int(rng.integers(1, 4)))
    y = tt.apply_op(op, x)
    ref = kron_matrix(op) @ tt.vec(tt.full(x))
    assert rel(tt.vec(tt.full(y)), ref) <= 1e-13


def test_apply_identity_operator(rng):
    n_x, n_xi, n_t = 7, 4, 5
    kl, ku, b = band_identity(n_t)
    op = KronSumOp(n_x, n_xi, n_t, [Term("id", kl, ku, b, np.eye(n_xi), sp.identity(n_x, format="csr"))])
    x = random_tt(rng, n_x, n_xi, n_t, 3, 2)
    y = tt.apply_op(op, x)
    assert tt.ranks(y) == (3, 2)
    assert np.array_equal(tt.full(y), tt.full(x))


def test_apply_linearity(rng):
    op = random_operator(rng, 6, 3, 4, 3)
    x = random_tt(rng, 6, 3, 4, 2, 3)
    y = random_tt(rng, 6, 3, 4, 3, 1)
    lhs = tt.full(tt.apply_op(op, tt.axpby(2.0, x, -0.5, y)))
    rhs = 2.0 * tt.full(tt.apply_op(op, x)) - 0.5 * tt.full(tt.apply_op(op, y))
    assert rel(lhs, rhs) <= 1e-13


# ----------------------------------------------------------------------------- round
@pytest.mark.parametrize("tol", [1e-10, 1e-3, 0.1, 0.3])
def test_round_equals_dense_ttsvd_on_c1_apply(c1, tol):
    _, op, x = c1
    y = tt.apply_op(op, x)
    yr, info = tt.round_tt(y, tol, return_info=True)
    d = tt.tt_svd_dense(tt.full(y), tol)
    assert tt.ranks(yr) == tt.ranks(d)
    assert rel(tt.full(yr), tt.full(d)) <= 1e-12
    assert info["norm"] == pytest.approx(np.linalg.norm(tt.full(y)), rel=1e-13)


@pytest.mark.parametrize("seed", range(40))
def test_round_error_bound_random(seed):
    """SPEC AC1-style: random TTs, modes <= 12, ranks <= 8: ||x~ - x|| <= eps ||x|| and
    equality with dense TT-SVD."""
    rng = np.random.default_rng(1000 + seed)
    n = rng.integers(1, 13, size=3)
    r1, r2 = rng.integers(1, 9, size=2)
    x = random_tt(rng, int(n[0]), int(n[1]), int(n[2]), int(r1), int(r2))
    eps = [1e-1, 1e-3, 1e-6][seed % 3]
    xr = tt.round_tt(x, eps)
    xf = tt.full(x)
    assert np.linalg.norm(tt.full(xr) - xf) <= eps * np.linalg.norm(xf) * (1 + 1e-12) + 1e-14
    d = tt.tt_svd_dense(xf, eps)
    assert tt.ranks(xr) == tt.ranks(d)
    assert rel(tt.full(xr), tt.full(d)) <= 1e-11
    k1, k2 = tt.ranks(xr)
    assert k1 <= min(n[0], n[1] * n[2]) and k2 <= min(n[0] * n[1], n[2])


def _diag_tt(rng, n_x, n_xi, n_t, sig):
    """X = sum_a sig_a u_a (x) q_a (x) w_a with orthonormal {u_a}, {q_a}, {w_a}:
    both unfoldings have singular values exactly sig."""
    r = len(sig)
    u1 = np.linalg.qr(rng.standard_normal((n_x, r)))[0]
    q = np.linalg.qr(rng.standard_normal((n_xi, r)))[0]
    w = np.linalg.qr(rng.standard_normal((n_t, r)))[0].T
    u2 = np.zeros((r, n_xi, r))
    for a in range(r):
        u2[a, :, a] = sig[a] * q[:, a]
    return u1, u2, w


@pytest.mark.parametrize("tol", [0.0, 1e-12, 1e-4, 2e-3, 0.05, 0.3])
def test_round_closed_form_spectrum(rng, tol):
    sig = np.array([1.0, 0.5, 0.25, 0.1, 1e-2, 1e-3, 1e-5, 1e-9])
    x = _diag_tt(rng, 20, 9, 11, sig)
    xr, info = tt.round_tt(x, tol, return_info=True)
    nrm = np.linalg.norm(sig)
    delta = tol * nrm / math.sqrt(2)
    # closed form of the tail rule
    r1 = next(r for r in range(1, 9) if np.linalg.norm(sig[r:]) <= delta) if tol > 0 else 8
    r2 = next(r for r in range(1, r1 + 1) if np.linalg.norm(sig[r:r1]) <= delta) if tol > 0 else r1
    assert tt.ranks(xr) == (r1, r2)
    assert np.max(np.abs(info["sigma1"][:8] - sig)) <= 1e-15 * 8
    err = np.linalg.norm(tt.full(xr) - tt.full(x))
    assert err == pytest.approx(math.sqrt(np.sum(sig[r2:] ** 2)), abs=1e-14)


def test_round_invariants_orthonormal_and_norm(c1):
    _, op, x = c1
    y = tt.apply_op(op, x)
    u1, u2, u3 = tt.round_tt(y, 1e-6)
    k1, k2 = u1.shape[1], u3.shape[0]
    assert np.max(np.abs(u1.T @ u1 - np.eye(k1))) <= 1e-13
    m2 = u2.reshape(-1, k2)
    assert np.max(np.abs(m2.T @ m2 - np.eye(k2))) <= 1e-13
    assert np.linalg.norm(u3) == pytest.approx(np.linalg.norm(tt.full(y)), rel=1e-12)


def test_round_rank_monotone_in_tol(c1):
    _, op, x = c1
    y = tt.apply_op(op, x)
    prev = (10 ** 9, 10 ** 9)
    for tol in [1e-14, 1e-10, 1e-6, 1e-3, 1e-2, 0.1, 0.3, 0.6]:
        r = tt.ranks(tt.round_tt(y, tol))
        assert r[0] <= prev[0] and r[1] <= prev[1]
        prev = r


def test_round_lossless_and_padding(rng):
    x = random_tt(rng, 9, 5, 7, 3, 4)
    x0 = tt.round_tt(x, 0.0)
    assert rel(tt.full(x0), tt.full(x)) <= 1e-13
    # zero padding to doubled ranks returns to the original ranks
    u1 = np.concatenate([x[0], np.zeros((9, 3))], axis=1)
    u2 = np.zeros((6, 5, 8)); u2[:3, :, :4] = x[1]
    u3 = np.concatenate([x[2], np.zeros((4, 7))], axis=0)
    xp = tt.round_tt((u1, u2, u3), 1e-14)
    assert tt.ranks(xp) == (3, 4)
    assert rel(tt.full(xp), tt.full(x)) <= 1e-13


def test_round_rmax_caps(c1):
    _, op, x = c1
    y = tt.apply_op(op, x)
    yr, info = tt.round_tt(y, 1e-12, rmax=3, return_info=True)
    assert tt.ranks(yr)[0] <= 3 and tt.ranks(yr)[1] <= 3


def test_round_zero_tensor_and_bad_tol(rng):
    z = (np.zeros((5, 2)), np.zeros((2, 3, 2)), np.zeros((2, 4)))
    zr = tt.round_tt(z, 1e-3)
    assert tt.ranks(zr) == (1, 1) and not np.any(tt.full(zr))
    with pytest.raises(ValueError):
        tt.round_tt(random_tt(rng, 3, 3, 3, 1, 1), -1.0)


def test_round_lowrank_structure_from_operator(c1):
    """Exact rank deficiency: K_k = nu_k L for the two KL terms, T_k = I for
    three terms -> numerical ranks at most 12 (space) and 8 (time)."""
    _, op, x = c1
    y = tt.apply_op(op, x)
    yr = tt.round_tt(y, 1e-12)
    assert tt.ranks(yr)[0] <= 12 and tt.ranks(yr)[1] <= 8


# ----------------------------------------------------------------------------- dot / axpby
@pytest.mark.parametrize("seed", range(8))
def test_dot_axpby_norm_dense(seed):
    rng = np.random.default_rng(50 + seed)
    n = [int(v) for v in rng.integers(1, 9, size=3)]
    x = random_tt(rng, *n, int(rng.integers(1, 5)), int(rng.integers(1, 5)))
    y = random_tt(rng, *n, int(rng.integers(1, 5)), int(rng.integers(1, 5)))
    xf, yf = tt.full(x), tt.full(y)
    assert tt.dot(x, y) == pytest.approx(float(np.sum(xf * yf)), rel=1e-12, abs=1e-12)
    assert tt.norm(x) == pytest.approx(np.linalg.norm(xf), rel=1e-12)
    z = tt.axpby(1.5, x, -2.0, y)
    assert tt.ranks(z) == (x[0].shape[1] + y[0].shape[1], x[2].shape[0] + y[2].shape[0])
    assert rel(tt.full(z), 1.5 * xf - 2.0 * yf) <= 1e-14


def test_add_negation_rounds_to_zero(rng):
    x = random_tt(rng, 8, 4, 6, 3, 3)
    z = tt.round_tt(tt.axpby(1.0, x, -1.0, x), 1e-12)
    assert tt.norm(z) <= 1e-12 * tt.norm(x)


def test_dot_disjoint_support_is_zero():
    a = (np.array([[1.0], [0.0]]), np.ones((1, 2, 1)), np.ones((1, 3)))
    b = (np.array([[0.0], [1.0]]), np.ones((1, 2, 1)), np.ones((1, 3)))
    assert tt.dot(a, b) == 0.0


def test_axpby_shape_mismatch(rng):
    with pytest.raises(ValueError):
        tt.axpby(1.0, random_tt(rng, 3, 3, 3, 1, 1), 1.0, random_tt(rng, 4, 3, 3, 1, 1))


def test_storage_ratio_paper_value():
    """ranks (13, 83) in the paper's (t, xi, x) order give 270748 stored
    entries vs 3829760 full velocity entries, ~7.1%."""
    g = GOLD["storage_ranks_paper_order"]
    x = (np.zeros((g["n_x"], g["kappa2"])), np.zeros((g["kappa2"], g["n_xi"], g["kappa1"])),
         np.zeros((g["kappa1"], g["n_t"])))
    assert tt.storage(x) == g["tt_storage"]
    assert g["n_t"] * g["n_xi"] * g["n_x"] == g["full_storage"]
    assert round(100 * g["tt_storage"] / g["full_storage"], 1) == g["ratio_percent_printed"]


# ----------------------------------------------------------------------------- rank rule
# The tail rule of PAPER.md:247-249 (Alg. 2 line 4, ||E||_F <= delta) with SPEC.md:109's tie
# rule ("keep every value equal to the last retained one") and BASELINE.json's rmax cap
# applied LAST: r = min(r_tie(r_delta), rmax).  Exact spectra with repeated values at the cut.
_SIG_TIE = np.array([1.0, 0.5, 0.5, 0.5, 0.1])   # tails: ||s[1:]|| = .8718, ||s[2:]|| = .7141,
                                                  #        ||s[3:]|| = .5099, ||s[4:]|| = .1


@pytest.mark.parametrize("delta,rmax,expect", [
    (0.6, 0, 4),     # r_delta = 3 (tail .5099 <= .6) -> tie s[3] == s[2] extends to 4
    (0.72, 0, 4),    # r_delta = 2 -> ties extend 2 -> 3 -> 4
    (0.9, 0, 1),     # r_delta = 1, s[1] = .5 != s[0]: no tie
    (0.05, 0, 5),    # nothing may be dropped
    (0.1, 0, 4),     # tail after 4 == delta exactly: kept (<=), s[4] != s[3]
    (0.6, 3, 3),     # rmax caps AFTER the tie loop: min(4, 3)
    (0.72, 2, 2),    # min(4, 2)
    (0.9, 3, 1),     # rmax larger than the rule: no effect
    (0.6, 9, 4),     # rmax beyond n
])
def test_rank_rule_ties_and_rmax_closed_form(delta, rmax, expect):
    assert tt.rank_rule(_SIG_TIE, delta, rmax) == expect


def test_rank_rule_tie_only_extends_over_equal_values():
    # a near-tie (1 ulp apart) is not a tie
    s = np.array([1.0, 0.5, np.nextafter(0.5, 0.0), 0.1])
    assert tt.rank_rule(s, math.sqrt(0.5 ** 2 + 0.01) + 1e-12, 0) == 2
    # a tie at the very end keeps everything
    s = np.array([1.0, 0.25, 0.25])
    assert tt.rank_rule(s, 0.3, 0) == 3
    # r >= 1 even for delta >= ||s|| and the empty spectrum
    assert tt.rank_rule(np.array([0.3, 0.2]), 10.0, 0) == 1
    assert tt.rank_rule(np.array([]), 1.0, 0) == 1


@pytest.mark.parametrize("rmax", [0, 2, 3])
def test_round_tie_spectrum_through_round_tt(rng, rmax):
    """round_tt on a TT whose unfoldings have EXACTLY repeated singular values.  Computed
    repeated values are equal only up to rounding, so the space rank is pinned up to the tie
    (3 or 4 without rmax, exactly rmax when it binds); the bond-1 discarded norm is the
    closed-form tail of the chosen rank, and the PAPER.md:252-258 bound holds when rmax does
    not bind (which vectors of a tied subspace are kept is not unique)."""
    sig = np.array([1.0, 0.5, 0.5, 0.5, 0.1])
    x = _diag_tt(rng, 30, 12, 9, sig)
    nrm = np.linalg.norm(sig)
    tol = 0.6 * math.sqrt(2) / nrm          # delta = 0.6 -> rank 4 (tie rule), or 3 if capped
    xr, info = tt.round_tt(x, tol, rmax=rmax, return_info=True)
    r = tt.ranks(xr)[0]
    assert r in ({3, 4} if rmax == 0 else {min(4, rmax)})
    assert info["discarded"][0] == pytest.approx(np.linalg.norm(sig[r:]), abs=1e-14)
    assert np.max(np.abs(info["sigma1"][:5] - sig)) <= 1e-14
    if rmax == 0:
        assert np.linalg.norm(tt.full(xr) - tt.full(x)) <= tol * nrm * (1 + 1e-12)
