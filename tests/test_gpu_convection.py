"""NEXT-1 through the C ABI: the TT convection operator N(u) (eq:N_kron,
PAPER.md:324-329) as a Kronecker-sum descriptor (diagonal T_k, dense G_k = sum_l u2 H_l, CSR
N(u_a)), applied and rounded by libttk, vs the oracle on the same descriptor; and the
eps_conv construction N(T_eps(u)) (eq:eps_conv) from GPU-rounded velocity
cores vs from oracle-rounded ones (the cores differ by gauge, the operators must not).

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
from synth import gpc  # noqa: E402
from synth.operator import convection_operator  # noqa: E402
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


@pytest.mark.parametrize("uranks", [(1, 1), (3, 4), (5, 4)])  # 1, 12 (merged SpMM), 20 terms
def test_convection_apply_parity(uranks, ctx):
    H, u, x = _case(11, 6, 2, 2, 5, uranks, (3, 2))
    op = convection_operator(6, len(H), 5, H, *u)
    y_o = otT.apply_op(op, x)
    y_g = ttk.tt_apply_op(ttk.Operator.from_kronsum(op, ctx), ttk.TT.from_cores(*x)).cores_numpy()
    for a, b in zip(y_g, y_o):
        assert a.shape == b.shape
        assert rel(a, b) <= 1e-13


@pytest.mark.parametrize("tol", [1e-10, 1e-4])
def test_convection_apply_round_parity(tol, ctx):
    H, u, x = _case(12, 6, 2, 2, 6, (3, 3), (3, 3))
    op = convection_operator(6, len(H), 6, H, *u)
    y = otT.apply_op(op, x)
    o, info = otT.round_tt(y, tol, 0, return_info=True)
    g, ginfo = ttk.tt_apply_round(ttk.Operator.from_kronsum(op, ctx), ttk.TT.from_cores(*x), tol,
                                  0, want_info=True)
    assert ginfo.ranks == info["ranks"]
    k1 = ginfo.ranks[0]
    assert np.max(np.abs(ginfo.sigma1[:k1] - info["sigma1"][:k1])) <= 1e-10 * info["sigma1"][0]
    assert rel(otT.full(g.cores_numpy()), otT.full(o)) <= 1e-10


def test_convection_from_rounded_velocity(ctx):
    """eq:eps_conv: N(T_eps(u)) with the velocity rounded on the GPU vs by the oracle."""
    H, u, x = _case(13, 5, 2, 2, 4, (2, 2), (2, 2))
    # a velocity of redundant rank (6, 6): u + u/2 + u/4 re-rounded to its true rank
    w = otT.axpby(1.0, otT.axpby(1.0, u, 0.5, u), 0.25, u)
    eps = 1e-8
    uo = otT.round_tt(w, eps, 0)
    ug = ttk.tt_round(ttk.TT.from_cores(*w), eps, 0, ctx).cores_numpy()
    assert otT.ranks(uo) == tuple(ug[0].shape[1:2] + ug[2].shape[:1]) == (2, 2)
    ref = otT.full(otT.apply_op(convection_operator(5, len(H), 4, H, *uo), x))
    og = convection_operator(5, len(H), 4, H, *ug)
    got = ttk.tt_apply_op(ttk.Operator.from_kronsum(og, ctx), ttk.TT.from_cores(*x)).cores_numpy()
    assert rel(otT.full(got), ref) <= 1e-12
