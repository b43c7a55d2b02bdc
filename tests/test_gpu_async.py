"""The asynchronous boundary of SURVEY.md 8(b) (include/ttk.h tk_ctx_set_async / tk_sync_ranks,
tk_round_workspace_bytes): queued roundings return before the GPU finishes, give the same
result as the synchronous path, are stream-ordered with later work on the context stream, and
report their errors at tk_sync_ranks; the scratch bound holds against the measured peak."""
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1906_06785_b200 as ttk  # noqa: E402
from oracle import tt as otT  # noqa: E402
from synth.configs import CONFIGS  # noqa: E402
from synth.operator import build_operator  # noqa: E402
from synth.tt import make_input_tt, random_tt  # noqa: E402


def c3_grown():
    cfg = CONFIGS["c3"]
    op = build_operator(cfg)
    x = make_input_tt(cfg, op.n_xi)
    return cfg, op, x


def test_async_round_returns_early_and_matches_sync():
    cfg, op, x = c3_grown()
    ctx_s = ttk.Context()
    gop = ttk.Operator.from_kronsum(op, ctx_s)
    xg = ttk.TT.from_cores(*x)
    y = ttk.tt_apply_op(gop, xg)
    ya = ttk.TT.from_cores(*[torch.as_tensor(c) for c in (y.U1, y.U2, y.U3)])
    torch.cuda.synchronize()
    ttk.tt_round(y, cfg.tol, cfg.rmax, ctx=ctx_s)  # warm-up of the synchronous path
    y = ttk.TT.from_cores(*[torch.as_tensor(c) for c in (ya.U1, ya.U2, ya.U3)])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ttk.tt_round(y, cfg.tol, cfg.rmax, ctx=ctx_s)
    t_sync = time.perf_counter() - t0
    torch.cuda.synchronize()

    ctx_a = ttk.Context()
    if not ctx_a.set_async(True):
        pytest.skip("no stream memory operations on this driver: async mode unavailable")
    for _ in range(2):
        z = ttk.TT.from_cores(*[torch.as_tensor(c) for c in (ya.U1, ya.U2, ya.U3)])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ttk.tt_round(z, cfg.tol, cfg.rmax, ctx=ctx_a)
        t_async = time.perf_counter() - t0
        # stream order: a copy enqueued right away on the context stream sees the rounded core
        snap = z.b1.clone()
        ctx_a.sync()
    assert t_async < 0.25 * t_sync, (t_async, t_sync)
    assert z.ranks == y.ranks
    for a, b in zip(z.cores_numpy(), y.cores_numpy()):
        assert np.array_equal(a, b)  # same kernels in the same order: bitwise
    torch.cuda.synchronize()
    assert torch.equal(snap[: z.n_x * z.r1], z.b1[: z.n_x * z.r1])
    ctx_a.set_async(False)


def test_async_chained_roundings_and_apply_round():
    """Two queued roundings of the same TT (the second reads the first's published ranks) and
    a queued fused apply+round, then a dot on the context stream."""
    cfg = CONFIGS["c1"]
    op = build_operator(cfg)
    x = make_input_tt(cfg, op.n_xi)
    ctx = ttk.Context()
    gop = ttk.Operator.from_kronsum(op, ctx)
    ref = otT.round_tt(otT.round_tt(otT.apply_op(op, x), 1e-10), 1e-3)
    ref2 = otT.round_tt(otT.apply_op(op, x), 1e-8, 6)
    if not ctx.set_async(True):
        pytest.skip("async mode unavailable")
    y = ttk.tt_apply_op(gop, ttk.TT.from_cores(*x))
    ttk.tt_round(y, 1e-10, ctx=ctx)
    ttk.tt_round(y, 1e-3, ctx=ctx)
    w = ttk.tt_apply_round(gop, ttk.TT.from_cores(*x), 1e-8, 6)
    ctx.sync()
    assert y.ranks == otT.ranks(ref)
    a, b = otT.full(y.cores_numpy()), otT.full(ref)
    assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(b)
    assert w.ranks == otT.ranks(ref2)
    d = ttk.tt_dot(w, w, ctx=ctx).item()
    assert abs(d - otT.dot(ref2, ref2)) <= 1e-10 * abs(d)
    ctx.set_async(False)


def test_async_error_is_reported_at_sync():
    rng = np.random.default_rng(3)
    x = ttk.TT.from_cores(*random_tt(rng, 30, 4, 5, 3, 3))
    ctx = ttk.Context()
    if not ctx.set_async(True):
        pytest.skip("async mode unavailable")
    ttk.tt_round(x, -1.0, ctx=ctx)  # queued: validated by the worker
    with pytest.raises(ttk.TkError) as e:
        ctx.sync()
    assert e.value.code == ttk.TK_EARG
    ttk.tt_round(x, 1e-8, ctx=ctx)  # the context is usable afterwards
    ctx.sync()
    assert x.ranks == (3, 3)
    ctx.set_async(False)


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_round_workspace_bound(name):
    """tk_round_workspace_bytes >= the measured scratch peak of tk_round and tk_apply_round."""
    cfg = CONFIGS[name]
    op = build_operator(cfg)
    x = make_input_tt(cfg, op.n_xi)
    ctx = ttk.Context()
    gop = ttk.Operator.from_kronsum(op, ctx)
    xg = ttk.TT.from_cores(*x)
    R1, R2 = op.T * xg.r1, op.T * xg.r2
    bound = ttk.round_workspace_bytes(op.n_x, op.n_xi, op.n_t, R1, R2)
    y = ttk.tt_apply_op(gop, xg)
    ctx.scratch_high_water(reset=True)
    ttk.tt_round(y, cfg.tol, cfg.rmax, ctx=ctx)
    peak_round = ctx.scratch_high_water(reset=True)
    ttk.tt_apply_round(gop, xg, cfg.tol, cfg.rmax)
    peak_fused = ctx.scratch_high_water()
    assert 0 < peak_round <= bound, (peak_round, bound)
    assert 0 < peak_fused <= bound, (peak_fused, bound)


@pytest.mark.parametrize("seed", range(6))
def test_round_workspace_bound_random(seed):
    rng = np.random.default_rng(900 + seed)
    n = [int(v) for v in rng.integers(2, 60, size=3)]
    r1, r2 = [int(v) for v in rng.integers(1, 200, size=2)]
    x = ttk.TT.from_cores(*random_tt(rng, *n, r1, r2))
    ctx = ttk.Context()
    ctx.scratch_high_water(reset=True)
    ttk.tt_round(x, 1e-8, ctx=ctx)
    assert ctx.scratch_high_water() <= ttk.round_workspace_bytes(*n, r1, r2)


def _wait_idle(stream, seconds=10.0):
    t0 = time.perf_counter()
    while not stream.query():
        if time.perf_counter() - t0 > seconds:
            return False
        time.sleep(0.001)
    return True


@pytest.mark.parametrize("use_async", [False, True])
def test_copy_window_gate(use_async):
    """tk_ctx_gate_stream: work on a gated stream waits (on the device) for the most recently
    submitted rounding of the context to reach its DMMA-bound phase and is released by it — also
    when that rounding fails; with nothing submitted, or in synchronous mode, the stream is not
    delayed."""
    cfg = CONFIGS["c3"]
    op = build_operator(cfg)
    x = make_input_tt(cfg, op.n_xi)
    ctx = ttk.Context()
    if use_async and not ctx.set_async(True):
        pytest.skip("no stream memory operations on this driver")
    gop = ttk.Operator.from_kronsum(op, ctx)
    xg = ttk.TT.from_cores(*x)
    side = torch.cuda.Stream()
    src = torch.arange(1 << 20, dtype=torch.float64, device="cuda")
    dst = torch.zeros_like(src)
    torch.cuda.synchronize()
    # nothing submitted yet: the gate is open
    if not ctx.gate_stream(side):
        pytest.skip("driver cannot gate streams")
    with torch.cuda.stream(side):
        dst.copy_(src, non_blocking=True)
    assert _wait_idle(side) and torch.equal(dst, src)
    # a submitted rounding: the copy completes, and never before the rounding was submitted
    for _ in range(2):
        dst.zero_()
        torch.cuda.synchronize()
        y = ttk.tt_apply_round(gop, xg, cfg.tol, cfg.rmax)
        assert ctx.gate_stream(side)
        with torch.cuda.stream(side):
            dst.copy_(src, non_blocking=True)
        ctx.sync()
        assert _wait_idle(side)
        assert torch.equal(dst, src)
    ref = otT.round_tt(otT.apply_op(op, x), cfg.tol, cfg.rmax)
    assert y.ranks == (ref[0].shape[1], ref[2].shape[0])
    # a rounding that fails validation still releases the stream
    dst.zero_()
    torch.cuda.synchronize()
    bad = ttk.TT.from_cores(*random_tt(np.random.default_rng(1), 11, 3, 4, 2, 2))
    with pytest.raises(ttk.TkError):
        ttk.tt_apply_round(gop, bad, cfg.tol, cfg.rmax)
        assert ctx.gate_stream(side)
        with torch.cuda.stream(side):
            dst.copy_(src, non_blocking=True)
        ctx.sync()
    if not use_async:  # (synchronous mode raised before the gate was requested)
        assert ctx.gate_stream(side)
        with torch.cuda.stream(side):
            dst.copy_(src, non_blocking=True)
    assert _wait_idle(side)
    assert torch.equal(dst, src)
