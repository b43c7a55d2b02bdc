"""tk_gemm (include/ttk.h): the dense fp64 contraction of the path on the DMMA pipe, with both
operand feeds (TMA tensor tiles / cp.async), against the definition C = alpha op(A) op(B) + beta C
evaluated on the CPU in fp64 (NumPy matmul: the plain definition, not the GPU path).

Shapes span several 64 x 64 x 16 tiles with ragged M, N and K tails, all four operand
orientations, padded leading dimensions, the symmetric-Gram mode and split-K (small output,
long K).  Tolerance: |C_gpu - C_ref| <= 8 eps K max|A| max|B| (a K-term fp64 dot product in any
summation order is within K eps sum|a_i b_i| of the exact value; both sides are, hence 2 K eps,
and the factor 8 leaves room for alpha/beta rounding)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1906_06785_b200 as ttk  # noqa: E402

EPS = np.finfo(np.float64).eps


def _operand(rng, rows, cols, ld):
    """rows x cols values inside a rows x ld row-major buffer (the padding is NaN: must not be read
    into any result)."""
    buf = np.full((rows, ld), np.nan)
    buf[:, :cols] = rng.standard_normal((rows, cols))
    return buf


def _run(ctx, M, N, K, ta, tb, pad, rng, alpha=1.0, beta=0.0, sym=False):
    if sym:
        # symmetric Gram: B^T A == A^T B needs the same operand on both sides
        assert ta and not tb and M == N
        A = B = _operand(rng, K, M, M + pad)
    lda = (M if ta else K) + pad
    ldb = (K if tb else N) + pad
    if not sym:
        A = _operand(rng, K if ta else M, M if ta else K, lda)
        B = _operand(rng, N if tb else K, K if tb else N, ldb)
    opA = (A[:, :M].T if ta else A[:, :K])
    opB = (B[:, :K].T if tb else B[:, :N])
    ldc = N + pad
    C0 = rng.standard_normal((M, ldc))
    ref = alpha * (opA @ opB) + (beta * C0[:, :N] if beta != 0.0 else 0.0)
    dA = torch.as_tensor(A, device="cuda")
    dB = dA if sym else torch.as_tensor(B, device="cuda")
    dC = torch.as_tensor(C0, device="cuda").clone()
    ctx.gemm(dA, dB, dC, M, N, K, trans_a=ta, trans_b=tb, alpha=alpha, beta=beta, lda=lda, ldb=ldb,
             ldc=ldc, sym=sym)
    torch.cuda.synchronize()
    out = dC.cpu().numpy()
    tol = 8 * EPS * max(K, 1) * max(np.abs(opA).max(), 1.0) * max(np.abs(opB).max(), 1.0) * max(abs(alpha), 1.0)
    err = np.abs(out[:, :N] - ref).max()
    assert np.isfinite(out[:, :N]).all()
    assert err <= tol, (err, tol)
    # the padding columns of C are untouched
    assert np.array_equal(out[:, N:], C0[:, N:])
    return out[:, :N]


SHAPES = [
    # M, N, K  — heavy enough (2MNK >= 2e8) for the TMA feed, even leading dimensions (TMA
    # eligible), ragged tails in every dimension
    (1000, 330, 1202),
    (4098, 130, 258),
    (518, 642, 402),
]


@pytest.mark.parametrize("feed", [1, 0])
@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False), (True, True)])
@pytest.mark.parametrize("M,N,K", SHAPES)
def test_gemm_all_layouts(feed, ta, tb, M, N, K):
    rng = np.random.default_rng([M, N, K, int(ta), int(tb)])
    ctx = ttk.Context()
    ctx.set_gemm_feed(feed)
    _run(ctx, M, N, K, ta, tb, pad=6, rng=rng, alpha=0.75)


@pytest.mark.parametrize("feed", [1, 0])
@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False), (True, True)])
def test_gemm_n80_tile(feed, ta, tb):
    """N = 80 j with a tall M (the c4 reconstruction shape class): the 64 x 80 TMA tile / the
    128 x 80 cp.async tile, ragged M and K."""
    rng = np.random.default_rng([80, int(ta), int(tb)])
    ctx = ttk.Context()
    ctx.set_gemm_feed(feed)
    _run(ctx, 75802, 160, 322, ta, tb, pad=2, rng=rng, alpha=1.25)


@pytest.mark.parametrize("feed", [1, 0])
def test_gemm_split_k_and_gram(feed):
    """Small output with a long K (split-K partials + fixed-order reduction), symmetric mode."""
    rng = np.random.default_rng(7)
    ctx = ttk.Context()
    ctx.set_gemm_feed(feed)
    # W^T W of a tall W (transA, K-major both): the rounding's Gram
    g1 = _run(ctx, 200, 200, 70001, True, False, pad=0, rng=rng, sym=True)
    assert np.array_equal(g1, g1.T)  # mirrored exactly
    g2 = _run(ctx, 136, 136, 50003, True, False, pad=2, rng=rng, sym=False)
    assert g2.shape == (136, 136)
    # the TT dot's W1 = X1^T Y1 (different operands)
    _run(ctx, 90, 130, 65537, True, False, pad=4, rng=rng)


@pytest.mark.parametrize("feed", [1, 0])
def test_gemm_beta_odd_ld_and_small(feed):
    """beta != 0, odd leading dimensions / misaligned views (cp.async fallback) and tiny sizes give
    the same answers whatever the feed setting."""
    rng = np.random.default_rng(11)
    ctx = ttk.Context()
    ctx.set_gemm_feed(feed)
    _run(ctx, 700, 300, 600, False, False, pad=3, rng=rng, alpha=-1.5, beta=0.5)
    _run(ctx, 700, 301, 601, False, True, pad=1, rng=rng)
    _run(ctx, 5, 3, 2, False, False, pad=0, rng=rng)
    _run(ctx, 64, 64, 16, True, True, pad=0, rng=rng)


def test_gemm_feeds_agree_and_reproducible():
    """Both feeds compute the same sums (different fixed order): they agree to rounding, and each
    is bitwise reproducible run to run."""
    rng = np.random.default_rng(3)
    M, N, K = 3000, 640, 896
    A = torch.as_tensor(rng.standard_normal((M, K)), device="cuda")
    B = torch.as_tensor(rng.standard_normal((K, N)), device="cuda")
    outs = {}
    for feed in (0, 1):
        ctx = ttk.Context()
        ctx.set_gemm_feed(feed)
        C1 = torch.empty((M, N), dtype=torch.float64, device="cuda")
        C2 = torch.empty_like(C1)
        ctx.gemm(A, B, C1, M, N, K)
        ctx.gemm(A, B, C2, M, N, K)
        torch.cuda.synchronize()
        assert torch.equal(C1, C2)
        outs[feed] = C1.cpu().numpy()
    ref = A.cpu().numpy() @ B.cpu().numpy()
    for feed in (0, 1):
        assert np.abs(outs[feed] - ref).max() <= 8 * EPS * K * 25
    assert np.abs(outs[0] - outs[1]).max() <= 8 * EPS * K * 25


def test_gemm_argument_errors():
    ctx = ttk.Context()
    A = torch.zeros((4, 4), dtype=torch.float64, device="cuda")
    with pytest.raises(ttk.TkError):
        ctx.gemm(A, A, A, 4, 3, 4, sym=True)  # sym needs M == N
    with pytest.raises(ttk.TkError):
        ctx.set_gemm_feed(7)


def test_round_bitwise_reproducible_with_tma_feed():
    """Regression: the TMA-fed reconstruction GEMM runs on the low-priority side stream while the
    bond-2 chain runs at high priority; without the cross-proxy fence before a stage is released
    to the TMA a few warp tiles of U1 came out wrong (run-to-run differences of 1e-2).  Rounding
    the same c3 TT repeatedly must give bitwise identical cores."""
    from synth.configs import CONFIGS
    from synth.operator import build_operator
    from synth.tt import make_input_tt

    cfg = CONFIGS["c3"]
    op = build_operator(cfg)
    x = make_input_tt(cfg, op.n_xi)
    ctx = ttk.Context()
    ctx.set_gemm_feed(1)
    gop = ttk.Operator.from_kronsum(op, ctx)
    y0 = ttk.tt_apply_op(gop, ttk.TT.from_cores(*x))
    base = [torch.as_tensor(c).clone() for c in (y0.U1, y0.U2, y0.U3)]
    outs = []
    for _ in range(6):
        y = ttk.TT.from_cores(*[b.clone() for b in base])
        torch.cuda.synchronize()
        ttk.tt_round(y, cfg.tol, cfg.rmax, ctx=ctx)
        torch.cuda.synchronize()
        outs.append((y.ranks, [c.copy() for c in y.cores_numpy()]))
    for ranks, cores in outs[1:]:
        assert ranks == outs[0][0]
        for a, b in zip(cores, outs[0][1]):
            assert np.array_equal(a, b)
