"""Scheduling variants of the block-Jacobi eigensolver behind the bond SVDs (include/ttk.h
tk_ctx_set_jacobi_schedule): the dataflow schedule (pair CTAs and tile CTAs one round apart,
ordered by counters in global memory) performs the same rotations and the same tile products in
the same order as the grid-barrier schedule, so a rounding gives bitwise identical cores, ranks
and singular values under both; and both agree with the CPU oracle (oracle/tt.py round_tt)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1906_06785_b200 as ttk  # noqa: E402
from oracle import tt as otT  # noqa: E402
from parity_util import tt_diff_rel  # noqa: E402
from synth.configs import CONFIGS  # noqa: E402
from synth.operator import build_operator  # noqa: E402
from synth.tt import make_input_tt, random_tt  # noqa: E402


def _round_with(schedule, cores, tol, rmax):
    ctx = ttk.Context()
    ctx.set_jacobi_schedule(schedule)
    y = ttk.TT.from_cores(*[np.array(c) for c in cores])
    _, info = ttk.tt_round(y, tol, rmax, ctx=ctx, want_info=True)
    torch.cuda.synchronize()
    return y.ranks, [c.copy() for c in y.cores_numpy()], info


def _grown(name):
    cfg = CONFIGS[name]
    op = build_operator(cfg)
    x = make_input_tt(cfg, op.n_xi)
    return cfg, otT.apply_op(op, x)


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_flow_schedule_bitwise_equals_barrier_schedule(name):
    cfg, y = _grown(name)
    ra, ca, ia = _round_with(0, y, cfg.tol, cfg.rmax)
    rb, cb, ib = _round_with(1, y, cfg.tol, cfg.rmax)
    assert ra == rb
    for a, b in zip(ca, cb):
        assert np.array_equal(a, b)
    assert np.array_equal(np.asarray(ia.sigma1), np.asarray(ib.sigma1))
    assert np.array_equal(np.asarray(ia.sigma2), np.asarray(ib.sigma2))


@pytest.mark.parametrize("shape", [(3000, 7, 40, 100, 30), (1500, 5, 33, 150, 20), (5000, 3, 70, 260, 12)])
def test_flow_schedule_random_shapes(shape):
    """Bond sizes with 2, 3 and 5 block pairs (k = 100, 150, 260 -> n_pad 128, 192, 320), against
    the other schedule (bitwise) and the oracle (1e-10 on the reconstructed tensor)."""
    n_x, n_xi, n_t, r1, r2 = shape
    rng = np.random.default_rng(list(shape))
    x = random_tt(rng, n_x, n_xi, n_t, r1, r2)
    tol = 1e-9
    ra, ca, _ = _round_with(0, x, tol, 0)
    rb, cb, _ = _round_with(1, x, tol, 0)
    assert ra == rb
    for a, b in zip(ca, cb):
        assert np.array_equal(a, b)
    ref = otT.round_tt(x, tol, 0)
    assert rb == (ref[0].shape[1], ref[2].shape[0])
    assert tt_diff_rel(cb, ref) <= 1e-10


def test_schedule_argument_error():
    ctx = ttk.Context()
    with pytest.raises(ttk.TkError):
        ctx.set_jacobi_schedule(3)


@pytest.mark.parametrize("feed,schedule", [(0, 0), (0, 1), (1, 0)])
def test_non_default_feed_and_schedule_match_the_oracle(feed, schedule):
    """The non-default combinations (cp.async GEMM feed, grid-barrier Jacobi) through the whole
    fused apply+round at c2 against the CPU oracle: ranks, kept singular values (1e-10 s_1) and
    the reconstructed tensor (1e-10)."""
    cfg = CONFIGS["c2"]
    op = build_operator(cfg)
    x = make_input_tt(cfg, op.n_xi)
    ctx = ttk.Context()
    ctx.set_gemm_feed(feed)
    ctx.set_jacobi_schedule(schedule)
    gop = ttk.Operator.from_kronsum(op, ctx)
    y, info = ttk.tt_apply_round(gop, ttk.TT.from_cores(*x), cfg.tol, cfg.rmax, want_info=True)
    torch.cuda.synchronize()
    ref, rinfo = otT.round_tt(otT.apply_op(op, x), cfg.tol, cfg.rmax, return_info=True)
    assert y.ranks == (ref[0].shape[1], ref[2].shape[0])
    s1 = np.asarray(info.sigma1)[: y.ranks[0]]
    assert np.abs(s1 - np.asarray(rinfo["sigma1"])[: y.ranks[0]]).max() <= 1e-10 * s1[0]
    assert tt_diff_rel(y.cores_numpy(), ref) <= 1e-10
