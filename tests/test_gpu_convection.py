"""NEXT-1 through the C ABI: the TT convection operator N(u) (eq:N_kron,
PAPER.md:324-329) built ON THE DEVICE by tk_op_convection from a device-resident velocity TT,
applied and rounded by libttk, vs the oracle's own eq:N_kron operator
(oracle.convection.convection_operator) on the same velocity cores.  The two sides share only
input data (the difference stencils and the H_l of synth/); each forms N(w), the chaos factors
and the diagonal time factors itself.  Plus: the eps_conv construction N(T_eps(u))
(eq:eps_conv) from a GPU-rounded velocity vs an oracle-rounded one, the
multi-chunk SpMM (> 16 spatial groups), and operator concatenation (F(u) = fixed + N(u)).

Bars as tests/test_gpu_parity.py: apply 1e-13 per core; round 1e-10 on the reconstructed
tensor, kept singular values 1e-10 s_1, equal ranks away from ties (R5).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1906_06785_b200 as ttk  # noqa: E402
from oracle import tt as otT  # noqa: E402
from oracle.convection import Operator as OOp, convection_operator  # noqa: E402
from synth import gpc  # noqa: E402
from synth.operator import convection_stencils, random_operator  # noqa: E402
from synth.tt import random_tt  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def ctx():
    return ttk.default_context()


def _case(seed, n, m, p, nt, uranks, xranks):
    rng = np.random.default_rng(seed)
    H = gpc.h_matrices(m, p)
    u = random_tt(rng, 3 * n * n, len(H), nt, *uranks)
    x = random_tt(rng, 3 * n * n, len(H), nt, *xranks)
    return H, u, x


def _conv(n, H, nt, ctx):
    D, n_v = convection_stencils(n)
    return ttk.Convection(3 * n_v, len(H), nt, D, n_v, np.stack(H), ctx), D, n_v


@pytest.mark.parametrize("uranks", [(1, 1), (3, 4), (5, 4), (8, 8), (17, 2), (4, 1)])
def test_convection_apply_parity(uranks, ctx):
    """1 .. 64 terms; (17, 2): two merged-SpMM chunks (16 + 1 spatial groups); (4, 1): the
    chunk's groups are its terms (identity output map)."""
    n, nt = 6, 5
    H, u, x = _case(11, n, 2, 2, nt, uranks, (3, 2))
    conv, D, n_v = _conv(n, H, nt, ctx)
    op_g = conv.operator(ttk.TT.from_cores(*u))
    assert op_g.T == uranks[0] * uranks[1]
    op_o = convection_operator(*u, H, D, n_v)
    y_o = otT.apply_op(op_o, x)
    y_g = ttk.tt_apply_op(op_g, ttk.TT.from_cores(*x)).cores_numpy()
    for a, b in zip(y_g, y_o):
        assert a.shape == b.shape
        assert rel(a, b) <= 1e-13
    with pytest.raises(ttk.TkError):   # no per-term CSR for a device-built operator
        op_g.set_spmm_kernel(1)


@pytest.mark.parametrize("tol", [1e-10, 1e-4])
def test_convection_apply_round_parity(tol, ctx):
    n, nt = 6, 6
    H, u, x = _case(12, n, 2, 2, nt, (3, 3), (3, 3))
    conv, D, n_v = _conv(n, H, nt, ctx)
    op_o = convection_operator(*u, H, D, n_v)
    y = otT.apply_op(op_o, x)
    o, info = otT.round_tt(y, tol, 0, return_info=True)
    g, ginfo = ttk.tt_apply_round(conv.operator(ttk.TT.from_cores(*u)), ttk.TT.from_cores(*x),
                                  tol, 0, want_info=True)
    assert ginfo.ranks == info["ranks"]
    k1 = ginfo.ranks[0]
    assert np.max(np.abs(ginfo.sigma1[:k1] - info["sigma1"][:k1])) <= 1e-10 * info["sigma1"][0]
    assert rel(otT.full(g.cores_numpy()), otT.full(o)) <= 1e-10


def test_convection_from_rounded_velocity(ctx):
    """eq:eps_conv: N(T_eps(u)) with the velocity rounded AND the operator built on the GPU vs
    both done by the oracle (the rounded cores differ by gauge, the operators must not)."""
    n, nt = 5, 4
    H, u, x = _case(13, n, 2, 2, nt, (2, 2), (2, 2))
    # a velocity of redundant rank (6, 6): u + u/2 + u/4 re-rounded to its true rank
    w = otT.axpby(1.0, otT.axpby(1.0, u, 0.5, u), 0.25, u)
    eps = 1e-8
    conv, D, n_v = _conv(n, H, nt, ctx)
    uo = otT.round_tt(w, eps, 0)
    ug = ttk.tt_round(ttk.TT.from_cores(*w), eps, 0, ctx)
    assert otT.ranks(uo) == ug.ranks == (2, 2)
    ref = otT.full(otT.apply_op(convection_operator(*uo, H, D, n_v), x))
    got = ttk.tt_apply_op(conv.operator(ug), ttk.TT.from_cores(*x)).cores_numpy()
    assert rel(otT.full(got), ref) <= 1e-12


@pytest.mark.parametrize("perterm_fixed", [False, True])
def test_concat_fixed_plus_convection(perterm_fixed, ctx):
    """tk_op_concat: A = A_fixed + N(u) (the Picard matrix shape), vs the oracle applying both
    term lists.  The fixed part alone keeps its per-term CSR, the concatenation cannot (the
    convection part has none), so it runs on the merged kernel."""
    n, nt = 5, 4
    H, u, x = _case(14, n, 2, 2, nt, (3, 2), (2, 3))
    rng = np.random.default_rng(5)
    fixed = random_operator(rng, 3 * n * n, len(H), nt, 4, density=0.05, max_band=1)
    conv, D, n_v = _conv(n, H, nt, ctx)
    gf = ttk.Operator.from_kronsum(fixed, ctx)
    if perterm_fixed:
        gf.set_spmm_kernel(1)
    gA = ttk.Operator.concat([gf, conv.operator(ttk.TT.from_cores(*u))])
    assert gA.T == 4 + 6
    oc = convection_operator(*u, H, D, n_v)
    oA = OOp(3 * n * n, len(H), nt, list(fixed.terms) + list(oc.terms))
    y_o = otT.apply_op(oA, x)
    y_g = ttk.tt_apply_op(gA, ttk.TT.from_cores(*x)).cores_numpy()
    for a, b in zip(y_g, y_o):
        assert rel(a, b) <= 1e-13
    # and the fused apply+round on the concatenation
    o, info = otT.round_tt(y_o, 1e-8, 0, return_info=True)
    g, ginfo = ttk.tt_apply_round(gA, ttk.TT.from_cores(*x), 1e-8, 0, want_info=True)
    assert ginfo.ranks == info["ranks"]
    assert rel(otT.full(g.cores_numpy()), otT.full(o)) <= 1e-10
