"""NEXT-3 through the C ABI: the block-tridiagonal spatial solves, M^{-1} of
eq:11_prec, S_LSC,0^{-1} of eq:mean_lsc, the full P^{-1} of eq:prec (R20) and flexible
GMRES with P — GPU (tk_bt_*, tk_prec_*, tk_gmres_*_p) vs oracle/precond.py on the same seeded
inputs.  The oracle's solves are scipy SuperLU; the GPU's are block LU on DMMA.

Bars: spatial solves elementwise to 1e-11 of the largest entry (the factors' conditioning is
far below 1e3 at these sizes); anything that rounds is compared on the reconstructed tensor at
1e-10 relative (R7); GMRES histories to 1e-8 beta (the c5 bar)."""
import dataclasses
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import scipy.sparse as sp  # noqa: E402

import paper_1906_06785_b200 as ttk  # noqa: E402
from oracle import tt as otT  # noqa: E402
from oracle.gmres import gmres_cycle as o_cycle  # noqa: E402
from oracle.precond import MeanLSC as OLSC  # noqa: E402
from oracle.precond import restrict_rows, spatial_solve  # noqa: E402
from synth.configs import CONFIGS  # noqa: E402
from synth.operator import build_operator, mean_blocks  # noqa: E402
from synth.tt import make_rhs_tt, random_tt  # noqa: E402

from parity_util import tt_diff_rel  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
TINY = dataclasses.replace(CONFIGS["c1"], grid=3, m=1, p=2, n_t=4, tau=0.1, nus=(0.05, 0.01),
                           ranks=(2, 2))
CFGS = {"tiny": TINY, "c1": CONFIGS["c1"], "c2": CONFIGS["c2"]}


@pytest.fixture(scope="module")
def ctx():
    return ttk.default_context()


def setup(name, tol, ctx, **inner):
    cfg = CFGS[name]
    op = build_operator(cfg)
    F0s, B = mean_blocks(cfg)
    o = OLSC(F0s, B, cfg.tau, op.n_xi, op.n_t, tol=tol,
             inner={**dict(tol=1e-1, restart=10, max_cycles=3), **inner})
    g = ttk.MeanLSC(F0s, B, cfg.tau, op.n_xi, op.n_t, tol=tol, grid=cfg.grid,
                    tol_in=inner.get("tol", 1e-1), restart_in=inner.get("restart", 10),
                    max_cycles_in=inner.get("max_cycles", 3), ctx=ctx)
    return cfg, op, F0s, B, o, g


def close_cores(a, b, rel):
    for x, y in zip(a, b):
        assert x.shape == y.shape
        assert np.abs(x - y).max() <= rel * max(np.abs(y).max(), 1e-300)


@pytest.mark.parametrize("name", ["tiny", "c1", "c2"])
@pytest.mark.parametrize("which", ["velocity", "pressure"])
def test_block_tridiagonal_solve(name, which, ctx):
    """tk_bt_solve vs SuperLU on K_s = tau^-1 I + F0s (both velocity blocks) and on B B^T."""
    cfg = CFGS[name]
    op = build_operator(cfg)
    F0s, B = mean_blocks(cfg)
    N = cfg.grid
    nv = N * N
    rng = np.random.default_rng(11)
    x = random_tt(rng, op.n_x, op.n_xi, op.n_t, 5, 3)
    import scipy.sparse.linalg as spla
    if which == "velocity":
        K = (sp.identity(nv) / cfg.tau + F0s).tocsc()
        bt = ttk.BlockTridiag(F0s, N, N, shift=1.0 / cfg.tau, ctx=ctx)
        row0, reps = 0, 2
    else:
        K = (B @ B.T).tocsc()
        bt = ttk.BlockTridiag(B, N, N, gram=True, ctx=ctx)
        row0, reps = 2 * nv, 1
    ref = spatial_solve(x, spla.splu(K), row0, nv, reps=reps)
    got = bt.solve(ttk.TT.from_cores(*x), row0, reps).cores_numpy()
    close_cores(got, ref, 1e-11)
    assert np.array_equal(got[1], x[1]) and np.array_equal(got[2], x[2])


def test_block_tridiagonal_rejects_wide_band(ctx):
    """A coupling two block rows apart is outside the factorisation's structure: TK_EARG."""
    n, N = 12, 3
    A = sp.identity(n, format="csr") + sp.csr_matrix(([1.0], ([0], [7])), shape=(n, n))
    with pytest.raises(ttk.TkError) as e:
        ttk.BlockTridiag(A.tocsr(), n // N, N, ctx=ctx)
    assert e.value.code == ttk.TK_EARG


@pytest.mark.parametrize("name", ["tiny", "c1", "c2"])
def test_m_inv_parity(name, ctx):
    """M^{-1} of eq:11_prec: time cumulative sum + K_s^{-1} on both velocity blocks."""
    cfg, op, F0s, B, o, g = setup(name, 1e-10, ctx)
    rng = np.random.default_rng(12)
    x = random_tt(rng, op.n_x, op.n_xi, op.n_t, 4, 3)
    ref = o.m_inv(x)
    got = g.apply(ttk.TT.from_cores(*x), part=1).cores_numpy()
    close_cores(got, ref, 1e-11)


@pytest.mark.parametrize("name", ["tiny", "c1", "c2"])
def test_schur_inv_parity(name, ctx):
    """S_LSC,0^{-1} v_p of eq:mean_lsc (two pressure solves around B (F0 + C) B^T, rounded)."""
    cfg, op, F0s, B, o, g = setup(name, 1e-10, ctx)
    rng = np.random.default_rng(13)
    x = random_tt(rng, op.n_x, op.n_xi, op.n_t, 3, 3)
    nv2 = 2 * cfg.grid ** 2
    ref = o.schur_inv(restrict_rows(x, nv2, op.n_x))
    got = g.apply(ttk.TT.from_cores(*x), part=2)
    assert got.ranks == otT.ranks(ref)
    assert tt_diff_rel(got.cores_numpy(), ref) <= 1e-10


@pytest.mark.parametrize("name,tol", [("tiny", 1e-10), ("c1", 1e-10), ("c2", 1e-8)])
def test_prec_apply_parity(name, tol, ctx):
    """The full P^{-1} v (R20 steps 1-7, inner GMRES with M at tol_in = 1e-1).  c2 truncates at
    1e-8: at 1e-10 its final spectrum is quasi-continuous across delta and the ~30 roundings
    of the inner solve move the tail sums by more than the gaps (a tie, R5)."""
    cfg, op, F0s, B, o, g = setup(name, tol, ctx)
    b = make_rhs_tt(dataclasses.replace(cfg, rhs_ranks=(3, 3)), op.n_xi)
    ref = o.apply(b)
    got = g.apply(ttk.TT.from_cores(*b), part=0)
    assert got.ranks == otT.ranks(ref)
    assert tt_diff_rel(got.cores_numpy(), ref) <= 1e-10


@pytest.mark.parametrize("name,steps,tol", [("tiny", 5, 1e-10), ("c1", 6, 1e-6)])
def test_gmres_cycle_with_lsc_parity(name, steps, tol, ctx):
    """Flexible GMRES with the mean-based P (Alg. 3 line 4): least-squares history, steps and the
    explicit residual vs the oracle, to 1e-8 beta."""
    cfg, op, F0s, B, o, g = setup(name, tol, ctx)
    b = make_rhs_tt(dataclasses.replace(cfg, rhs_ranks=(4, 4)), op.n_xi)
    ro = o_cycle(op, b, steps=steps, tol=tol, prec=o.apply)
    rg = ttk.gmres_cycle(ttk.Operator.from_kronsum(op, ctx), ttk.TT.from_cores(*b), steps=steps,
                         tol=tol, prec=g)
    beta = ro["history"][0]
    assert rg["steps"] == ro["steps"]
    assert np.max(np.abs(rg["history"] - ro["history"])) <= 1e-8 * beta
    assert abs(rg["explicit"] - ro["explicit"]) <= 1e-8 * beta


def test_gmres_cycle_with_lsc_c5_golden(ctx):
    """c5's operator (the c2 operator family) with P = the mean-based LSC preconditioner: the GPU history vs
    the oracle history stored by tools/make_golden.py (oracle + synth only; ~8 CPU minutes)."""
    path = os.path.join(HERE, "golden", "c5p_gmres_oracle.json")
    gold = json.load(open(path))
    cfg = CONFIGS["c5"]
    op = build_operator(cfg)
    F0s, B = mean_blocks(cfg)
    b = make_rhs_tt(cfg, op.n_xi)
    g = ttk.MeanLSC(F0s, B, cfg.tau, op.n_xi, op.n_t, tol=gold["tol"], grid=cfg.grid, ctx=ctx)
    rg = ttk.gmres_cycle(ttk.Operator.from_kronsum(op, ctx), ttk.TT.from_cores(*b),
                         steps=gold["steps"], tol=gold["tol"], prec=g)
    h = np.array(gold["history"])
    assert rg["steps"] == gold["steps_done"]
    assert np.max(np.abs(rg["history"] - h)) <= 1e-8 * h[0]
    assert abs(rg["explicit"] - gold["explicit"]) <= 1e-8 * h[0]
