"""Pin of the oracle GMRES cycle: at rounding tol ~ 0 it must reproduce dense GMRES on the
explicit Kronecker matrix (the idea of SPEC.md:401), implemented here independently."""
import dataclasses

import numpy as np
import pytest

from oracle import tt
from oracle.gmres import gmres_cycle
from oracle.kron_dense import kron_matrix
from synth.configs import CONFIGS
from synth.operator import build_operator
from synth.tt import make_rhs_tt


def dense_gmres_history(A, b, steps):
    n = b.size
    beta = np.linalg.norm(b)
    V = np.zeros((n, steps + 1))
    H = np.zeros((steps + 1, steps))
    V[:, 0] = b / beta
    hist = [beta]
    for k in range(steps):
        w = A @ V[:, k]
        for i in range(k + 1):
            H[i, k] = w @ V[:, i]
            w = w - H[i, k] * V[:, i]
        H[k + 1, k] = np.linalg.norm(w)
        V[:, k + 1] = w / H[k + 1, k]
        e1 = np.zeros(k + 2); e1[0] = beta
        y, *_ = np.linalg.lstsq(H[: k + 2, : k + 1], e1, rcond=None)
        hist.append(np.linalg.norm(e1 - H[: k + 2, : k + 1] @ y))
    return np.array(hist)


@pytest.fixture(scope="module")
def c1_small():
    cfg = CONFIGS["c1"]
    op = build_operator(cfg)
    b = make_rhs_tt(dataclasses.replace(cfg, rhs_ranks=(2, 2)), op.n_xi)
    return op, b


def test_gmres_cycle_equals_dense_gmres_at_tiny_tol(c1_small):
    op, b = c1_small
    steps = 8
    res = gmres_cycle(op, b, steps=steps, tol=1e-14)
    A = kron_matrix(op)
    ref = dense_gmres_history(A, tt.vec(tt.full(b)), steps)
    assert res["steps"] == steps
    assert np.max(np.abs(res["history"] - ref) / ref[0]) <= 1e-9


def test_gmres_history_nonincreasing(c1_small):
    op, b = c1_small
    res = gmres_cycle(op, b, steps=6, tol=1e-6)
    h = res["history"]
    assert np.all(np.diff(h) <= 1e-12 * h[0])
    # explicit residual of the returned z is consistent with the estimate up to truncation
    assert res["explicit"] <= h[-1] + 1e-4 * h[0]


def dense_restarted_gmres(A, b, restart, cycles):
    """Restarted GMRES(m) on the explicit matrix, x_0 = 0; explicit residual after each cycle."""
    x = np.zeros_like(b)
    res = [np.linalg.norm(b)]
    for _ in range(cycles):
        r = b - A @ x
        beta = np.linalg.norm(r)
        n = b.size
        V = np.zeros((n, restart + 1))
        H = np.zeros((restart + 1, restart))
        V[:, 0] = r / beta
        for k in range(restart):
            w = A @ V[:, k]
            for i in range(k + 1):
                H[i, k] = w @ V[:, i]
                w = w - H[i, k] * V[:, i]
            H[k + 1, k] = np.linalg.norm(w)
            V[:, k + 1] = w / H[k + 1, k]
        e1 = np.zeros(restart + 1)
        e1[0] = beta
        y, *_ = np.linalg.lstsq(H, e1, rcond=None)
        x = x + V[:, :restart] @ y
        res.append(np.linalg.norm(b - A @ x))
    return x, np.array(res)


def test_gmres_solve_equals_dense_restarted_gmres_at_tiny_tol(c1_small):
    """NEXT-2 pin: with truncation tol ~ 0 the restarted low-rank solver is restarted GMRES(m)."""
    from oracle.gmres import gmres_solve
    op, b = c1_small
    res = gmres_solve(op, b, restart=4, max_cycles=3, tol=1e-14, tol_gmres=0.0, eps_soln=1e-14)
    A = kron_matrix(op)
    xv, ref = dense_restarted_gmres(A, tt.vec(tt.full(b)), 4, 3)
    assert res["cycles"] == 3
    assert np.max(np.abs(res["explicit"] - ref) / ref[0]) <= 1e-9
    zv = tt.vec(tt.full(res["z"]))
    assert np.linalg.norm(zv - xv) <= 1e-8 * np.linalg.norm(xv)


def test_gmres_solve_stops_and_decreases(c1_small):
    from oracle.gmres import gmres_solve
    op, b = c1_small
    res = gmres_solve(op, b, restart=6, max_cycles=6, tol=1e-10, tol_gmres=1e-3)
    e = res["explicit"]
    assert e[-1] <= 1e-3 * tt.norm(b) * (1 + 1e-6) or res["cycles"] == 6
    assert np.all(np.diff(e) <= 1e-8 * e[0])  # restarted GMRES residuals never grow
