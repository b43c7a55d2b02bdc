"""NEXT-2 through the C ABI: the complete restarted low-rank GMRES of Alg. 3
 with the truncated solution update of eq:eps_soln,
tk_gmres_solve vs oracle.gmres.gmres_solve on the same seeded operator and right-hand side.

Bars: explicit residual norms per cycle within 1e-8 relative (to ||b||), same cycle and step
counts, the returned solution within 1e-8 (reconstructed, relative) — at truncation
tolerances where both sides take the same rank decisions (R5)."""
import dataclasses

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1906_06785_b200 as ttk  # noqa: E402
from oracle import tt as otT  # noqa: E402
from oracle.gmres import gmres_solve as o_solve  # noqa: E402
from synth.configs import CONFIGS  # noqa: E402
from synth.operator import build_operator  # noqa: E402
from synth.tt import make_rhs_tt  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    return ttk.default_context()


@pytest.mark.parametrize("restart,cycles,tol,tol_gmres,eps_soln", [
    (4, 3, 1e-10, 0.0, 1e-10),     # fixed number of restarts
    (6, 8, 1e-8, 1e-4, 1e-8),      # stops on the explicit residual
    (5, 3, 1e-8, 0.0, 1e-6),       # coarser solution update (eq:eps_soln)
])
def test_gmres_solve_parity_c1(restart, cycles, tol, tol_gmres, eps_soln, ctx):
    cfg = CONFIGS["c1"]
    op = build_operator(cfg)
    b = make_rhs_tt(dataclasses.replace(cfg, rhs_ranks=(2, 2)), op.n_xi)
    o = o_solve(op, b, restart=restart, max_cycles=cycles, tol=tol, tol_gmres=tol_gmres,
                eps_soln=eps_soln)
    g = ttk.gmres_solve(ttk.Operator.from_kronsum(op, ctx), ttk.TT.from_cores(*b), restart=restart,
                        max_cycles=cycles, tol=tol, tol_gmres=tol_gmres, eps_soln=eps_soln)
    bn = otT.norm(b)
    assert g["cycles"] == o["cycles"]
    assert np.max(np.abs(g["explicit"] - o["explicit"])) <= 1e-8 * bn
    for a, c in zip(g["ls"], o["ls"]):
        assert len(a) == len(c)
        assert np.max(np.abs(a - c)) <= 1e-8 * bn
    zo = otT.full(o["z"])
    zg = otT.full(g["z"].cores_numpy())
    assert np.linalg.norm(zg - zo) <= 1e-8 * np.linalg.norm(zo)


def test_gmres_solve_zero_rhs(ctx):
    cfg = CONFIGS["c1"]
    op = build_operator(cfg)
    b = make_rhs_tt(dataclasses.replace(cfg, rhs_ranks=(1, 1)), op.n_xi)
    b = (b[0] * 0.0, b[1], b[2])
    g = ttk.gmres_solve(ttk.Operator.from_kronsum(op, ctx), ttk.TT.from_cores(*b), restart=3,
                        max_cycles=2, tol=1e-8, tol_gmres=1e-6)
    assert g["cycles"] == 0
    assert np.all(g["z"].cores_numpy()[0] == 0.0)


def test_gmres_solve_parity_c5_operator(ctx):
    """The c5 operator (c2 sizes, 6 terms) and right-hand side, two restarts of 4 steps at the
    config's truncation tolerance: explicit residuals and the solution vs the oracle."""
    cfg = CONFIGS["c5"]
    op = build_operator(cfg)
    b = make_rhs_tt(cfg, op.n_xi)
    o = o_solve(op, b, restart=4, max_cycles=2, tol=cfg.tol, tol_gmres=0.0)
    g = ttk.gmres_solve(ttk.Operator.from_kronsum(op, ctx), ttk.TT.from_cores(*b), restart=4,
                        max_cycles=2, tol=cfg.tol, tol_gmres=0.0)
    bn = otT.norm(b)
    assert g["cycles"] == o["cycles"] == 2
    assert np.max(np.abs(g["explicit"] - o["explicit"])) <= 1e-8 * bn
    # the solution: ||z_g - z_o|| via the orthogonalised difference TT (too large to densify)
    d = otT.round_tt(otT.axpby(1.0, g["z"].cores_numpy(), -1.0, o["z"]), 0.0)
    assert np.linalg.norm(d[2]) <= 1e-8 * otT.norm(o["z"])
