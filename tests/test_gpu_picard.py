"""NEXT-4 through the C ABI: the inexact Picard iteration of Alg. 1
(eq:inexact_solve :536-538), tk_picard vs oracle/picard.py on the seeded
all-at-once stochastic Galerkin Navier-Stokes problem (configs c7, c8; R21).

Bars: the same number of Picard iterations and rank sequence, nonlinear residual norms within
1e-8 ||f|| per iteration, the solution within 1e-8 (reconstructed, relative).  At c8 (GPU
scale) the oracle recomputes the nonlinear residual of the GPU's solution from its own
operator (eq:ns_sys_all)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1906_06785_b200 as ttk  # noqa: E402
from oracle import tt as otT  # noqa: E402
from oracle.picard import picard as o_picard  # noqa: E402
from oracle.picard import residual, system_operator  # noqa: E402
from oracle.precond import MeanLSC as OLSC  # noqa: E402
from synth import gpc  # noqa: E402
from synth.configs import CONFIGS  # noqa: E402
from synth.operator import build_operator, convection_stencils, mean_blocks, picard_forcing  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    return ttk.default_context()


def problem(name, ctx):
    cfg = CONFIGS[name]
    op = build_operator(cfg)
    H = gpc.h_matrices(cfg.m, cfg.p)
    D, nv = convection_stencils(cfg.grid)
    f = picard_forcing(cfg, op.n_xi)
    g_op = ttk.Operator.from_kronsum(op, ctx)
    g_conv = ttk.Convection(op.n_x, op.n_xi, op.n_t, D, nv, np.array(H), ctx=ctx)
    return cfg, op, H, D, nv, f, g_op, g_conv


@pytest.mark.parametrize("with_prec", [False, True])
def test_picard_parity_c7(with_prec, ctx):
    cfg, op, H, D, nv, f, g_op, g_conv = problem("c7", ctx)
    kw = dict(tol_picard=1e-3, maxit=8, tol_gmres=1e-1, eps_gmres=cfg.tol, restart=20,
              max_cycles=5)
    o_prec = g_prec = None
    if with_prec:
        F0s, B = mean_blocks(cfg)
        o_prec = OLSC(F0s, B, cfg.tau, op.n_xi, op.n_t, tol=cfg.tol).apply
        g_prec = ttk.MeanLSC(F0s, B, cfg.tau, op.n_xi, op.n_t, tol=cfg.tol, grid=cfg.grid,
                             ctx=ctx)
    o = o_picard(op, H, D, nv, f, prec=o_prec, **kw)
    g = ttk.picard(g_op, g_conv, ttk.TT.from_cores(*f), prec=g_prec, **kw)
    fn = o["fnorm"]
    assert g["iterations"] == o["iterations"]
    assert [tuple(r) for r in g["ranks"]] == [tuple(r) for r in o["ranks"]]
    assert np.max(np.abs(g["residuals"] - np.array(o["residuals"]))) <= 1e-8 * fn
    zo = otT.full(o["z"])
    zg = otT.full(g["z"].cores_numpy())
    assert np.linalg.norm(zg - zo) <= 1e-8 * np.linalg.norm(zo)


def test_picard_c8_converges_and_solves_the_system(ctx):
    """c8 (16 x 16 grid, n_xi = 6, n_t = 8) with the mean-based preconditioner: the GPU
    iteration stops on the Picard test, contracts, and the oracle's own nonlinear residual of
    the returned solution agrees with the GPU's last one."""
    cfg, op, H, D, nv, f, g_op, g_conv = problem("c8", ctx)
    F0s, B = mean_blocks(cfg)
    P = ttk.MeanLSC(F0s, B, cfg.tau, op.n_xi, op.n_t, tol=cfg.tol, grid=cfg.grid, ctx=ctx)
    tol_picard = 1e-3
    g = ttk.picard(g_op, g_conv, ttk.TT.from_cores(*f), tol_picard=tol_picard, maxit=12,
                   tol_gmres=1e-1, eps_gmres=cfg.tol, restart=20, max_cycles=5, prec=P)
    fn = otT.norm(f)
    r = g["residuals"] / fn
    assert r[-1] <= tol_picard and np.all(r[:-1] > tol_picard)
    assert np.all(np.diff(r) < 0)
    z = g["z"].cores_numpy()
    L = system_operator(op, z, H, D, nv, cfg.tol)
    ro = otT.norm(residual(f, L, z, 0.0))
    assert abs(ro - g["residuals"][-1]) <= 2 * cfg.tol * fn
